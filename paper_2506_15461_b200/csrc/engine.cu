// Engine core: parameter groups, the iteration driver, replicas and the
// recovery path.  Block arithmetic lives in mlp_block.cu / llama_block.cu.
#include <dlfcn.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>
#include <string>

#include "engine.h"
#include "host_logic.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace ckf {

static bool step_debug() {  // CKF_STEP_DEBUG=1: per-step host / device split on stderr
  static const bool on = [] {
    const char* v = std::getenv("CKF_STEP_DEBUG");
    return v && v[0] == '1';
  }();
  return on;
}

long& launch_counter() {
  static long n = 0;
  return n;
}

std::vector<Range> even_partition(size_t layers, size_t stages) {
  // model.cpp:63-73: contiguous, the first (L mod s) stages take one extra layer
  std::vector<Range> out;
  size_t next = 1;
  for (size_t i = 0; i < stages; ++i) {
    const size_t cnt = layers / stages + (i < layers % stages ? 1 : 0);
    out.push_back({next, next + cnt - 1});
    next += cnt;
  }
  return out;
}

// ------------------------------------------------------------------ NCCL (dlopen)
// Resolved at runtime so the library does not pin one libnccl: inside a torch
// process this binds to the NCCL torch already loaded.
namespace {
struct NcclApi {
  using Uid = struct { char b[128]; };
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, Uid, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*CommSplit)(void*, int, int, void**, void*) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<int (*)(void**, int, NcclApi::Uid, int)>(dlsym(h, "ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
      api.Send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclSend"));
      api.Recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclRecv"));
      api.AllReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
          dlsym(h, "ncclAllReduce"));
      api.CommSplit = reinterpret_cast<int (*)(void*, int, int, void**, void*)>(dlsym(h, "ncclCommSplit"));
      api.AllGather =
          reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(dlsym(h, "ncclAllGather"));
      api.GroupStart = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupStart"));
      api.GroupEnd = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupEnd"));
      api.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.AllReduce;
    }
  }
  if (!api.ok) raise(7, "libnccl.so.2 not loadable (multi-GPU placement needs NCCL)");
  return api;
}
void nccl_check(int r, const char* what) {
  if (r != 0) raise(7, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}
}  // namespace

int nccl_unique_id(void* out, size_t cap) {
  if (cap < 128) raise(1, "unique id buffer must hold 128 bytes");
  nccl_check(nccl().GetUniqueId(out), "ncclGetUniqueId");
  return 128;
}

// ------------------------------------------------------------------ lifecycle
Engine::Engine(const ckf_model_desc& in) {
  d_.block = in.block;
  d_.prec = in.precision;
  d_.act = in.activation;
  d_.task = in.task;
  d_.in = in.input_dim;
  d_.hid = in.hidden_dim;
  d_.d = in.model_dim;
  d_.out = in.output_dim;
  d_.L = in.num_layers;
  d_.s = in.num_stages;
  d_.heads = in.n_heads ? in.n_heads : 1;
  d_.T = in.seq_len ? in.seq_len : 1;
  d_.max_rows = in.max_rows ? in.max_rows : 256;
  if (const char* g = std::getenv("CKF_MB_GROUP")) group_cap_ = std::max(0, std::atoi(g));
  if (const char* g = std::getenv("CKF_GRAPHS")) graphs_ = g[0] != '0';
  d_.device = in.device;
  if (d_.block != CKF_BLOCK_MLP && d_.block != CKF_BLOCK_LLAMA) raise(1, "unknown block kind");
  if (d_.prec < CKF_FP64 || d_.prec > CKF_BF16) raise(1, "unknown precision");
  if (d_.block == CKF_BLOCK_MLP && d_.prec == CKF_BF16) raise(1, "the residual-MLP parity block runs in fp64 or fp32");
  if (d_.in == 0 || d_.hid == 0 || d_.d == 0 || d_.out == 0 || d_.L == 0)
    raise(1, "model dimensions and layer count must be positive");
  if (d_.s < 1 || d_.s > d_.L) raise(1, "num_stages must lie in [1, num_layers]");
  if (in.partition) {
    for (size_t i = 0; i < d_.s; ++i) d_.part.push_back({in.partition[2 * i], in.partition[2 * i + 1]});
  } else {
    d_.part = even_partition(d_.L, d_.s);
  }
  size_t expect = 1;  // model.cpp:88-94
  for (auto& r : d_.part) {
    if (r.first != expect || r.last < r.first || r.last > d_.L)
      raise(1, "partition ranges must be contiguous, ordered and cover [1, num_layers]");
    expect = r.last + 1;
  }
  if (expect != d_.L + 1) raise(1, "partition does not cover all layers");
  if (d_.task == CKF_TASK_CLASSIFICATION && d_.out < 2) raise(1, "classification requires output_dim >= 2");

  CKF_CUDA(cudaSetDevice(d_.device));
  CKF_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  // side streams of the plan-driven pipeline (stage transfers) and of the data-parallel all-reduce
  CKF_CUDA(cudaStreamCreateWithFlags(&sst_, cudaStreamNonBlocking));
  CKF_CUDA(cudaStreamCreateWithFlags(&rst_, cudaStreamNonBlocking));
  CKF_CUDA(cudaStreamCreateWithFlags(&dst_, cudaStreamNonBlocking));
  CKF_CUDA(cudaMalloc(&red_.partials, ReduceScratch::kMaxReduceBlocks * sizeof(double)));
  CKF_CUDA(cudaMalloc(&scal_, 4096 * sizeof(double)));
  CKF_CUDA(cudaMemset(scal_, 0, 4096 * sizeof(double)));
  CKF_CUDA(cudaEventCreate(&ev0_));
  CKF_CUDA(cudaEventCreate(&ev1_));
  CKF_CUDA(cudaEventCreate(&sb_ev_));
  CKF_CUDA(cudaEventCreate(&sg_ev_));
  CKF_CUDA(cudaEventCreateWithFlags(&se_ev_, cudaEventBlockingSync));  // the step's final wait yields the CPU

  if (d_.block == CKF_BLOCK_LLAMA && d_.prec == CKF_FP64)
    raise(1, "the LLaMA block runs in bf16 (tensor cores) or fp32 (parity mode); fp64 parity is the MLP block's");
  impl_ = d_.block == CKF_BLOCK_MLP  ? make_mlp_block(this)
          : d_.prec == CKF_FP32      ? make_llama_f32_block(this)
                                     : make_llama_block(this);
  const bool lowp = d_.prec == CKF_BF16;
  stages_.resize(d_.s);
  for (size_t i = 0; i < d_.s; ++i) alloc_group(stages_[i], impl_->stage_params(static_cast<int>(i + 1)), lowp);
  alloc_group(embed_, impl_->embed_params(), lowp);
  alloc_group(deembed_, impl_->deembed_params(), lowp);
}

Engine::~Engine() {
  cudaSetDevice(d_.device);
  if (st_) cudaStreamSynchronize(st_);
  impl_.reset();
  for (auto& g : stages_) free_group(g);
  free_group(embed_);
  free_group(deembed_);
  cudaFree(rep_embed_);
  cudaFree(rep_deembed_);
  for (void* p : ws_) cudaFree(p);
  cudaFree(red_.partials);
  cudaFree(scal_);
  for (cudaStream_t x : {sst_, rst_, dst_})
    if (x) cudaStreamSynchronize(x);
  for (auto& l : links_)
    if (l.second && nccl().CommDestroy) nccl().CommDestroy(l.second);
  for (cudaEvent_t ev : pev_) cudaEventDestroy(ev);
  if (dp_comm_ && nccl().CommDestroy) nccl().CommDestroy(dp_comm_);
  if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
  if (gexec_) cudaGraphExecDestroy(gexec_);
  for (void* p : rc_replica_) cudaFree(p);
  for (auto& p : peer_)
    for (void* q : {p.w, p.m, p.v})
      if (q) cudaIpcCloseMemHandle(q);
  for (void* q : peer_mbox_)
    if (q) cudaIpcCloseMemHandle(q);
  for (uint64_t* q : peer_flags_)
    if (q) cudaIpcCloseMemHandle(q);
  cudaFree(mbox_);
  cudaFree(flags_);
  for (auto& c : ckpt_) cudaFree(c.buf);
  for (cudaEvent_t ev : kev_) cudaEventDestroy(ev);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (sb_ev_) cudaEventDestroy(sb_ev_);
  if (sg_ev_) cudaEventDestroy(sg_ev_);
  if (se_ev_) cudaEventDestroy(se_ev_);
  if (st_) cudaStreamDestroy(st_);
  for (cudaStream_t x : {sst_, rst_, dst_})
    if (x) cudaStreamDestroy(x);
}

void Engine::alloc_group(ParamGroup& g, size_t n, bool lowp) {
  g.n = n;
  const size_t b = n * master_bytes();
  if (!g.owned || n == 0) return;
  CKF_CUDA(cudaMalloc(&g.w, b));
  CKF_CUDA(cudaMalloc(&g.g, b));
  CKF_CUDA(cudaMalloc(&g.m, b));
  CKF_CUDA(cudaMalloc(&g.v, b));
  CKF_CUDA(cudaMemsetAsync(g.g, 0, b, st_));
  CKF_CUDA(cudaMemsetAsync(g.m, 0, b, st_));
  CKF_CUDA(cudaMemsetAsync(g.v, 0, b, st_));
  if (lowp) CKF_CUDA(cudaMalloc(&g.wlp, n * sizeof(__nv_bfloat16)));
}

void Engine::free_group(ParamGroup& g) {
  cudaFree(g.w);
  cudaFree(g.g);
  cudaFree(g.m);
  cudaFree(g.v);
  cudaFree(g.wlp);
  g.w = g.g = g.m = g.v = nullptr;
  g.wlp = nullptr;
}

void* Engine::ws(size_t bytes, int slot) {
  if (slot >= static_cast<int>(ws_.size())) {
    ws_.resize(static_cast<size_t>(slot) + 1, nullptr);
    ws_size_.resize(static_cast<size_t>(slot) + 1, 0);
  }
  if (ws_size_[static_cast<size_t>(slot)] < bytes) {
    CKF_CUDA(cudaStreamSynchronize(st_));
    cudaFree(ws_[static_cast<size_t>(slot)]);
    const size_t want = std::max<size_t>(bytes, 256);
    CKF_CUDA(cudaMalloc(&ws_[static_cast<size_t>(slot)], want));
    ++alloc_epoch();
    ws_size_[static_cast<size_t>(slot)] = want;
  }
  return ws_[static_cast<size_t>(slot)];
}

std::vector<ParamGroup*> Engine::owned_groups() {
  std::vector<ParamGroup*> v;
  for (auto& g : stages_)
    if (g.owned && g.n) v.push_back(&g);
  for (ParamGroup* g : {&embed_, &deembed_})
    if (g->owned && g->n) v.push_back(g);
  return v;
}

// ------------------------------------------------------------------ kernel timing
void Engine::kt_enable(bool on) {
  CKF_CUDA(cudaStreamSynchronize(st_));
  kt_on_ = on;
  kev_used_ = 0;
  krec_.clear();
  for (auto& k : kstat_) k = KStat{};
}

void Engine::kt_begin() {
  if (!kt_on_) return;
  if (kev_used_ + 2 > kev_.size()) {
    // grow the pool; a long step can tag a few thousand launches
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t ev;
      CKF_CUDA(cudaEventCreate(&ev));
      kev_.push_back(ev);
    }
  }
  CKF_CUDA(cudaEventRecord(kev_[kev_used_], st_));
}

void Engine::kt_end(int cls, double flops, double bytes) {
  if (!kt_on_) return;
  CKF_CUDA(cudaEventRecord(kev_[kev_used_ + 1], st_));
  kev_used_ += 2;
  krec_.push_back({cls, flops, bytes});
}

void Engine::kt_collect() {
  if (!kt_on_) return;
  for (size_t i = 0; i < krec_.size(); ++i) {
    float ms = 0.f;
    CKF_CUDA(cudaEventElapsedTime(&ms, kev_[2 * i], kev_[2 * i + 1]));
    KStat& k = kstat_[krec_[i].cls];
    k.ms += ms;
    k.flops += krec_[i].flops;
    k.bytes += krec_[i].bytes;
    ++k.launches;
  }
  krec_.clear();
  kev_used_ = 0;
}

// ------------------------------------------------------------------ placement
void Engine::set_placement(int nranks, int rank, const int* stage_rank, int replicas) {
  if (nranks < 1 || rank < 0 || rank >= nranks) raise(1, "invalid rank / world size");
  if (replicas < 1 || nranks % replicas) raise(1, "world size must be a multiple of the replica count");
  const int P = nranks / replicas;  // pipeline ranks per replica
  for (size_t i = 0; i < d_.s; ++i)
    if (stage_rank[i] < 0 || stage_rank[i] >= P) raise(1, "stage placed on a pipeline rank outside the replica");
  replicas_ = replicas;
  replica_ = rank / P;
  // global owner of each stage inside this rank's replica: ranks [replica * P, replica * P + P)
  stage_rank_.resize(d_.s);
  for (size_t i = 0; i < d_.s; ++i) stage_rank_[i] = replica_ * P + stage_rank[i];
  rank_ = rank;
  nranks_ = nranks;
  if (nranks > 1) schedule_ = impl_->supports_plan() ? 2 : 1;  // 1F1B where the block runs plan ops
  // release buffers of stages this rank does not own
  for (size_t i = 0; i < d_.s; ++i) {
    stages_[i].owned = stage_rank_[i] == rank_;
    if (!stages_[i].owned) free_group(stages_[i]);
  }
  embed_.owned = owner_of_embed() == rank_;
  deembed_.owned = owner_of_deembed() == rank_;
  if (!embed_.owned) free_group(embed_);
  if (!deembed_.owned) free_group(deembed_);
}

void Engine::attach_comm(const void* uid, int nranks, int rank, const int* stage_rank, int replicas) {
  set_placement(nranks, rank, stage_rank, replicas);
  if (nranks > 1) {
    const int P = nranks / replicas;
    NcclApi::Uid u;
    std::memcpy(u.b, uid, 128);
    CKF_CUDA(cudaSetDevice(d_.device));
    nccl_check(nccl().CommInitRank(&comm_, nranks, u, rank), "ncclCommInitRank");
    if (replicas > 1) {
      // data-parallel group: the same pipeline rank of every replica
      if (!nccl().CommSplit) raise(7, "ncclCommSplit unavailable (NCCL >= 2.18 needed for replicas)");
      nccl_check(nccl().CommSplit(comm_, rank % P, replica_, &dp_comm_, nullptr), "ncclCommSplit");
    }
  }
}

// One communicator per DIRECTED stage link of the pipeline (the links the standard and the
// CheckFree+ swapped routes use under this placement): on every rank a link's communicator is
// driven by exactly one stream (the source's send stream / the destination's recv stream).
// Created on the first NCCL-transport plan iteration -- every rank reaches it in the same
// iteration, and ncclCommSplit is collective over the world, so every rank walks the same list.
void Engine::ensure_links() {
  if (links_ready_ || nranks_ <= 1 || !comm_) return;
  links_ready_ = true;  // (a rank on no link still took part in every split)
  if (!nccl().CommSplit) raise(7, "ncclCommSplit unavailable (NCCL >= 2.18 needed for the stage links)");
  const int P = nranks_ / replicas_;
  if (P <= 1) return;
  std::vector<int> sr(d_.s);
  for (size_t i = 0; i < d_.s; ++i) sr[i] = stage_rank_[i] - replica_ * P;
  std::vector<std::pair<int, int>> want;
  for (int sw = 0; sw < (d_.s >= 4 ? 2 : 1); ++sw) {
    const std::vector<int> o = host::build_schedule(2, sw == 1, static_cast<int>(d_.s));
    for (const auto& op : host::pipeline_plan(static_cast<int>(d_.s), 2, o, sr, 1))
      if (op.kind == host::PlanOp::kXfer) want.push_back({op.rank, op.arg});
  }
  std::sort(want.begin(), want.end());
  want.erase(std::unique(want.begin(), want.end()), want.end());
  const int me = rank_ % P;
  for (size_t i = 0; i < want.size(); ++i) {
    const auto [a, b] = want[i];
    const bool in = me == a || me == b;
    void* c = nullptr;
    // color = link index x replicas + replica (each replica its own 2-rank communicator); the
    // source gets key 0
    nccl_check(nccl().CommSplit(comm_, in ? static_cast<int>(i) * replicas_ + replica_ : -1 /*NCCL_SPLIT_NOCOLOR*/,
                                me == a ? 0 : 1, &c, nullptr),
               "ncclCommSplit (stage link)");
    if (in) links_.push_back({{replica_ * P + a, replica_ * P + b}, c});
  }
}

void* Engine::link_comm(int src, int dst) {
  for (auto& l : links_)
    if (l.first.first == src && l.first.second == dst) return l.second;
  raise(7, "no communicator for stage link " + std::to_string(src) + " -> " + std::to_string(dst));
}

cudaEvent_t Engine::plan_event() {
  if (pev_used_ == pev_.size()) {
    cudaEvent_t ev;
    CKF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    pev_.push_back(ev);
  }
  return pev_[pev_used_++];
}

void Engine::enable_peer_transport(int max_m) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (max_m < 1) raise(1, "peer transport: max microbatches must be positive");
  if (d_.block != CKF_BLOCK_LLAMA || !impl_->supports_plan())
    raise(1, "peer transport carries the plan-driven (LLaMA) pipeline's stage transfers");
  if (mbox_) {
    cudaFree(mbox_);
    cudaFree(flags_);
  }
  mbox_m_ = max_m;
  mbox_slot_ = (d_.max_rows * d_.d * sizeof(float) + 255) / 256 * 256;
  CKF_CUDA(cudaMalloc(&mbox_, 2 * static_cast<size_t>(max_m) * mbox_slot_));
  CKF_CUDA(cudaMalloc(&flags_, 2 * static_cast<size_t>(max_m) * sizeof(uint64_t)));
  CKF_CUDA(cudaMemset(flags_, 0, 2 * static_cast<size_t>(max_m) * sizeof(uint64_t)));
  plan_epoch_ = 0;
}

void* Engine::mailbox(int k, int phase) const {
  if (!mbox_) return nullptr;
  if (k < 0 || k >= mbox_m_) raise(1, "peer transport: microbatch beyond the mailbox (enable it with more)");
  return static_cast<char*>(mbox_) + (static_cast<size_t>(k) * 2 + static_cast<size_t>(phase)) * mbox_slot_;
}

host::PlanCost Engine::plan_cost() const {
  host::PlanCost cost;
  for (size_t i = 0; i < d_.s; ++i) cost.stage.push_back(static_cast<double>(d_.part[i].count()));
  if (d_.block == CKF_BLOCK_LLAMA) {
    const double layer = 4.0 * d_.d * d_.d + 3.0 * d_.d * d_.hid + 2.0 * d_.d * d_.T;  // per token, fwd
    cost.head = static_cast<double>(d_.d) * static_cast<double>(d_.out) / layer;
  }
  return cost;
}

void Engine::grad_bucket_ready(void* g, size_t n) {
  if (replicas_ <= 1 || !dp_comm_ || n == 0) return;
  // this bucket's sum over the replicas on the data-parallel stream, behind the GEMMs that
  // produced it; the optimizer step waits for the stream (run_iteration)
  cudaEvent_t ev = plan_event();
  CKF_CUDA(cudaEventRecord(ev, st_));
  CKF_CUDA(cudaStreamWaitEvent(dst_, ev, 0));
  nccl_check(nccl().AllReduce(g, g, n, fp64() ? /*ncclFloat64*/ 8 : /*ncclFloat32*/ 7, /*ncclSum*/ 0, dp_comm_, dst_),
             "ncclAllReduce (data-parallel bucket)");
  dp_pending_ = true;
}

// Plan-driven iteration (schedule 2): every rank walks the SAME global op order
// (host::pipeline_plan, 1F1B) and executes its own share -- compute ops on the engine stream,
// sends on the send stream behind an event of the producing op, receives on the recv stream with
// the consuming op waiting on their event.  Each microbatch's buffers are private to it for the
// iteration, so the only cross-stream hazards are a buffer received back after this rank sent it
// (the recv waits for that send) and the end of the step (the engine stream joins both side
// streams).  With a virtual placement (hop log) on one GPU every op runs here and a transfer is
// a pointer hand-off.
void Engine::run_plan(const int* orders, int m, const char* x, size_t mb, size_t xrow) {
  const int s = static_cast<int>(d_.s);
  const bool virt = log_hops_;
  std::vector<int> placement(d_.s, 0);
  for (size_t i = 0; i < d_.s; ++i) placement[i] = virt ? vrank_[i] : owner_of_stage(static_cast<int>(i + 1));
  const host::PlanCost cost = plan_cost();
  const std::vector<int> ov(orders, orders + static_cast<size_t>(m) * d_.s);
  const int slots = host::plan_inflight_limit(m, placement);
  const auto plan = host::pipeline_plan(s, m, ov, placement, 2, &cost, slots);
  impl_->plan_begin(m, mb, slots, x);
  std::vector<cudaEvent_t> pending(static_cast<size_t>(m) * 2, nullptr);  // recv landed (per mb, phase)
  std::vector<cudaEvent_t> sent(static_cast<size_t>(m) * 2, nullptr);     // last send of the buffer
  bool any_send = false, any_recv = false;
  (void)xrow;
  const bool peer = !virt && peer_transport();
  if (!virt && !peer) ensure_links();
  if (peer && static_cast<int>(peer_mbox_.size()) != nranks_) raise(1, "peer transport: IPC exchange missing");
  if (peer && m > mbox_m_) raise(1, "peer transport: more microbatches than the mailbox holds");
  ++plan_epoch_;
  if (peer && plan_epoch_ >= (1ull << 55)) raise(1, "peer transport: epoch overflow");
  std::vector<std::vector<uint32_t>> arrivals(static_cast<size_t>(std::max(nranks_, 1)),
                                               std::vector<uint32_t>(static_cast<size_t>(m) * 2, 0));
  static const char* kNames[] = {"ckf.plan.embed_fwd", "ckf.plan.stage_fwd", "ckf.plan.xfer", "ckf.plan.head",
                                 "ckf.plan.stage_bwd", "ckf.plan.embed_bwd"};
  for (const auto& op : plan) {
    const int k = op.mb;
    if (!virt && op.kind != host::PlanOp::kXfer && op.rank != rank_) continue;
    NvtxRange nv(kNames[op.kind]);
    if (op.kind == host::PlanOp::kXfer) {
      size_t bytes = 0;
      void* b = impl_->plan_buffer(k, op.aux, &bytes);
      if (virt) {
        hop_log_.push_back(op.rank);
        hop_log_.push_back(op.arg);
        hop_log_.push_back(static_cast<long>(bytes));
        if (op.aux == 1) impl_->plan_received(k, 1);  // the receiving side's bf16(dh) refresh
        continue;
      }
      const size_t slot = static_cast<size_t>(k) * 2 + static_cast<size_t>(op.aux);
      if (peer) {
        // peer-memory transport: the sender's copy engine writes straight into the receiver's
        // mailbox over NVLink, then a one-thread kernel raises the receiver's flag (release);
        // the receiver's recv stream spins on it (acquire).  Flag value = iteration epoch and the
        // arrival count of this (microbatch, phase) at that rank -- every rank walks the whole
        // plan, so both sides count the same.
        const uint64_t val = (plan_epoch_ << 8) | static_cast<uint64_t>(++arrivals[static_cast<size_t>(op.arg)][slot]);
        if (op.rank == rank_) {
          if (op.arg >= static_cast<int>(peer_mbox_.size()) || !peer_mbox_[static_cast<size_t>(op.arg)])
            raise(1, "peer transport: rank " + std::to_string(op.arg) + "'s mailbox is not mapped (IPC exchange)");
          cudaEvent_t ev = plan_event();
          CKF_CUDA(cudaEventRecord(ev, st_));
          CKF_CUDA(cudaStreamWaitEvent(sst_, ev, 0));
          char* dstp = static_cast<char*>(peer_mbox_[static_cast<size_t>(op.arg)]) + slot * mbox_slot_;
          CKF_CUDA(cudaMemcpyAsync(dstp, b, bytes, cudaMemcpyDeviceToDevice, sst_));
          k::flag_signal(peer_flags_[static_cast<size_t>(op.arg)] + slot, val, sst_);
          any_send = true;
        } else if (op.arg == rank_) {
          k::flag_wait(flags_ + slot, val, rst_);
          cudaEvent_t ev = plan_event();
          CKF_CUDA(cudaEventRecord(ev, rst_));
          pending[slot] = ev;
          any_recv = true;
        }
        continue;
      }
      if (op.rank == rank_) {  // send behind the producing op
        cudaEvent_t ev = plan_event();
        CKF_CUDA(cudaEventRecord(ev, st_));
        CKF_CUDA(cudaStreamWaitEvent(sst_, ev, 0));
        nccl_check(nccl().Send(b, bytes, /*ncclInt8*/ 0, 1, link_comm(op.rank, op.arg), sst_), "ncclSend (stage link)");
        cudaEvent_t done = plan_event();
        CKF_CUDA(cudaEventRecord(done, sst_));
        sent[slot] = done;
        any_send = true;
      } else if (op.arg == rank_) {  // receive; the consuming op waits on it
        if (sent[slot]) CKF_CUDA(cudaStreamWaitEvent(rst_, sent[slot], 0));
        nccl_check(nccl().Recv(b, bytes, /*ncclInt8*/ 0, 0, link_comm(op.rank, op.arg), rst_), "ncclRecv (stage link)");
        cudaEvent_t ev = plan_event();
        CKF_CUDA(cudaEventRecord(ev, rst_));
        pending[slot] = ev;
        any_recv = true;
      }
      continue;
    }
    if (!virt && op.rank != rank_) continue;
    for (int ph = 0; ph < 2; ++ph) {
      cudaEvent_t& ev = pending[static_cast<size_t>(k) * 2 + static_cast<size_t>(ph)];
      if (!ev) continue;
      CKF_CUDA(cudaStreamWaitEvent(st_, ev, 0));
      ev = nullptr;
      if (ph == 1) impl_->plan_received(k, 1);
    }
    const int* o = orders + static_cast<size_t>(k) * d_.s;
    impl_->plan_op(op.kind, k, op.arg, o, scal_ + k);
  }
  // the step's end joins the side streams (sends done reading, every receive consumed)
  for (auto [flag, str] : {std::make_pair(any_send, sst_), std::make_pair(any_recv, rst_)}) {
    if (!flag) continue;
    cudaEvent_t ev = plan_event();
    CKF_CUDA(cudaEventRecord(ev, str));
    CKF_CUDA(cudaStreamWaitEvent(st_, ev, 0));
  }
  (void)x;
  (void)s;
}

// ------------------------------------------------------------------ peer (IPC) mappings
namespace {
struct IpcEntry {
  int32_t rank, replica, sid, kind;  // kind 0 = w, 1 = m, 2 = v
  uint64_t bytes;
  cudaIpcMemHandle_t h;
};
}  // namespace

size_t Engine::ipc_export(void* buf, size_t cap) {
  CKF_CUDA(cudaSetDevice(d_.device));
  std::vector<IpcEntry> v;
  for (size_t i = 0; i < d_.s; ++i) {
    ParamGroup& g = stages_[i];
    if (!g.owned || g.n == 0) continue;
    void* bufs[3] = {g.w, g.m, g.v};
    for (int k = 0; k < 3; ++k) {
      IpcEntry e{};
      e.rank = rank_;
      e.replica = replica_;
      e.sid = static_cast<int32_t>(i + 1);
      e.kind = k;
      e.bytes = g.n * master_bytes();
      CKF_CUDA(cudaIpcGetMemHandle(&e.h, bufs[k]));
      v.push_back(e);
    }
  }
  if (mbox_) {  // peer transport: mailbox and flags
    void* bufs[2] = {mbox_, flags_};
    const uint64_t sizes[2] = {2ull * static_cast<uint64_t>(mbox_m_) * mbox_slot_,
                               2ull * static_cast<uint64_t>(mbox_m_) * sizeof(uint64_t)};
    for (int k = 0; k < 2; ++k) {
      IpcEntry e{};
      e.rank = rank_;
      e.replica = replica_;
      e.sid = 0;
      e.kind = 3 + k;
      e.bytes = sizes[k];
      CKF_CUDA(cudaIpcGetMemHandle(&e.h, bufs[k]));
      v.push_back(e);
    }
  }
  const size_t need = v.size() * sizeof(IpcEntry);
  if (need > cap) raise(1, "IPC export buffer too small (" + std::to_string(need) + " bytes needed)");
  if (need) std::memcpy(buf, v.data(), need);
  return need;
}

void Engine::ipc_import(const void* buf, size_t len) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (len % sizeof(IpcEntry)) raise(1, "malformed IPC blob");
  if (peer_.size() != d_.s) peer_.assign(d_.s, PeerStage{});
  const auto* e = static_cast<const IpcEntry*>(buf);
  for (size_t i = 0; i < len / sizeof(IpcEntry); ++i) {
    const IpcEntry& x = e[i];
    if (x.rank == rank_ || x.replica != replica_) continue;  // own stages / other replicas' copies
    if (x.kind == 3 || x.kind == 4) {  // a peer's transport mailbox / flags
      if (x.rank < 0 || x.rank >= nranks_) raise(1, "malformed IPC entry (rank)");
      if (peer_mbox_.size() != static_cast<size_t>(nranks_)) {
        peer_mbox_.assign(static_cast<size_t>(nranks_), nullptr);
        peer_flags_.assign(static_cast<size_t>(nranks_), nullptr);
      }
      void** slot = x.kind == 3 ? &peer_mbox_[static_cast<size_t>(x.rank)]
                                : reinterpret_cast<void**>(&peer_flags_[static_cast<size_t>(x.rank)]);
      if (!*slot) CKF_CUDA(cudaIpcOpenMemHandle(slot, x.h, cudaIpcMemLazyEnablePeerAccess));
      continue;
    }
    if (x.sid < 1 || x.sid > static_cast<int>(d_.s) || x.kind < 0 || x.kind > 2) raise(1, "malformed IPC entry");
    ParamGroup& g = stages_[static_cast<size_t>(x.sid - 1)];
    if (g.owned) continue;
    if (x.bytes != g.n * master_bytes()) raise(1, "IPC entry size differs from the stage's size");
    void** slot = x.kind == 0 ? &peer_[x.sid - 1].w : x.kind == 1 ? &peer_[x.sid - 1].m : &peer_[x.sid - 1].v;
    if (*slot) continue;
    CKF_CUDA(cudaIpcOpenMemHandle(slot, x.h, cudaIpcMemLazyEnablePeerAccess));
  }
  peer_ready_ = true;
  for (size_t i = 0; i < d_.s; ++i)
    if (!stages_[i].owned && !(peer_[i].w && peer_[i].m && peer_[i].v)) peer_ready_ = false;
}

void Engine::hop(void* buf, size_t bytes, int src, int dst) {
  if (src == dst || bytes == 0) return;
  NvtxRange nv("ckf.hop");
  if (rank_ == src) nccl_check(nccl().Send(buf, bytes, /*ncclInt8*/ 0, dst, comm_, st_), "ncclSend");
  if (rank_ == dst) nccl_check(nccl().Recv(buf, bytes, /*ncclInt8*/ 0, src, comm_, st_), "ncclRecv");
}

bool Engine::move(void* buf, size_t bytes, int from_code, int to_code) {
  if (log_hops_) {
    auto vo = [&](int c) {
      const int sid = c <= 0 ? 1 : c > static_cast<int>(d_.s) ? static_cast<int>(d_.s) : c;
      return vrank_[static_cast<size_t>(sid - 1)];
    };
    if (vo(from_code) != vo(to_code)) {
      hop_log_.push_back(vo(from_code));
      hop_log_.push_back(vo(to_code));
      hop_log_.push_back(static_cast<long>(bytes));
    }
  }
  const int src = owner_of_code(from_code), dst = owner_of_code(to_code);
  if (src == dst) return false;
  hop(buf, bytes, src, dst);
  return rank_ == dst;
}

void Engine::hop_log_enable(int nranks, const int* vrank) {
  hop_log_.clear();
  log_hops_ = vrank != nullptr && nranks > 0;
  if (!log_hops_) return;
  vrank_.assign(vrank, vrank + d_.s);
  for (int r : vrank_)
    if (r < 0 || r >= nranks) raise(1, "virtual placement names a rank outside the world");
}

// ------------------------------------------------------------------ init
void Engine::init(uint64_t seed, double lr) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (lr <= 0.0) raise(1, "learning rate must be positive");
  for (size_t i = 0; i < d_.s; ++i) {
    ParamGroup& g = stages_[i];
    g.step = 0;
    g.omega = 0.0;
    g.lr = lr;
    if (!g.owned) continue;
    impl_->init_stage(static_cast<int>(i + 1), seed, g.w);
    CKF_CUDA(cudaMemsetAsync(g.g, 0, g.n * master_bytes(), st_));
    CKF_CUDA(cudaMemsetAsync(g.m, 0, g.n * master_bytes(), st_));
    CKF_CUDA(cudaMemsetAsync(g.v, 0, g.n * master_bytes(), st_));
    if (g.wlp) k::convert(static_cast<const float*>(g.w), g.wlp, g.n, st_);
  }
  impl_->init_edges(seed, embed_.owned ? embed_.w : nullptr, deembed_.owned ? deembed_.w : nullptr);
  for (ParamGroup* g : {&embed_, &deembed_}) {
    g->step = 0;
    g->lr = lr;
    if (!g->owned) continue;
    CKF_CUDA(cudaMemsetAsync(g->g, 0, g->n * master_bytes(), st_));
    CKF_CUDA(cudaMemsetAsync(g->m, 0, g->n * master_bytes(), st_));
    CKF_CUDA(cudaMemsetAsync(g->v, 0, g->n * master_bytes(), st_));
    if (g->wlp) k::convert(static_cast<const float*>(g->w), g->wlp, g->n, st_);
  }
  edge_lr = lr;
  replica_staleness_ = -1;
  CKF_CUDA(cudaStreamSynchronize(st_));
}

// ------------------------------------------------------------------ iteration
namespace {
void validate_order(const int* order, size_t s) {
  std::vector<bool> seen(s, false);  // model.cpp:201-209
  for (size_t i = 0; i < s; ++i) {
    const int sid = order[i];
    if (sid < 1 || static_cast<size_t>(sid) > s || seen[static_cast<size_t>(sid - 1)])
      raise(1, "stage order must be a permutation of [1..num_stages]");
    seen[static_cast<size_t>(sid - 1)] = true;
  }
}
}  // namespace

void Engine::adam_group(ParamGroup& g, double lr, double gscale, double* omega_dev) {
  ++g.step;  // on every rank: optimizer scalars stay replicated
  if (!g.owned || g.n == 0) return;
  // bias corrections with std::pow on the host, exactly kernels_serial.cpp:135-136
  const double bc1 = 1.0 - std::pow(0.9, static_cast<double>(g.step));
  const double bc2 = 1.0 - std::pow(0.999, static_cast<double>(g.step));
  kt_begin();
  if (fp64())
    k::adam(static_cast<double*>(g.w), static_cast<double*>(g.m), static_cast<double*>(g.v),
            static_cast<double*>(g.g), g.wlp, g.n, lr, bc1, bc2, gscale, true, omega_dev, red_, st_);
  else
    k::adam(static_cast<float*>(g.w), static_cast<float*>(g.m), static_cast<float*>(g.v), static_cast<float*>(g.g),
            g.wlp, g.n, lr, bc1, bc2, gscale, true, omega_dev, red_, st_);
  // g, w, m, v read; w, m, v, g(zeroed) written; + bf16 shadow
  kt_end(KC_ADAM, 0.0, static_cast<double>(g.n) * (8.0 * master_bytes() + (g.wlp ? 2.0 : 0.0)));
}

// Largest fused group (in microbatches of mb_rows) whose activations fit in half
// of the HBM still free after the block's pending reservations; fitted once per
// microbatch size so the choice (and hence the numerics) is stable across iterations.
int Engine::fused_group_size(int m, size_t mb_rows) {
  if (m < 2 || group_cap_ == 1) return 1;
  const size_t bpt = impl_->group_bytes_per_token();
  if (!bpt) return 1;
  const size_t tok = mb_rows * (d_.block == CKF_BLOCK_LLAMA ? d_.T : 1);
  int fit = 0;
  for (const auto& e : group_fit_)
    if (e.first == tok) fit = e.second;
  if (!fit) {
    size_t fr = 0, tot = 0;
    CKF_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t res = impl_->reserved_bytes();
    const size_t budget = fr > res ? (fr - res) / 2 : 0;
    fit = static_cast<int>(std::min<size_t>(64, budget / std::max<size_t>(1, bpt * tok)));
    fit = std::max(fit, 1);
    group_fit_.emplace_back(tok, fit);
  }
  int g = std::min(fit, m);
  if (group_cap_ > 0) g = std::min(g, group_cap_);
  return g;
}

void Engine::run_iteration(const int* orders, int m, const void* x, const void* y, size_t rows, bool on_device,
                           long iteration, double* loss, double* omegas) {
  NvtxRange nv_it("ckf.run_iteration");
  CKF_CUDA(cudaSetDevice(d_.device));
  if (m < 1) raise(1, "microbatch count must be positive");
  if (rows == 0 || rows % static_cast<size_t>(m) != 0)
    raise(1, "batch size must be divisible by the microbatch count");  // pipeline.cpp:62-63
  if (m > 2000) raise(1, "at most 2000 microbatches per iteration");
  for (int k = 0; k < m; ++k) validate_order(orders + static_cast<size_t>(k) * d_.s, d_.s);
  for (auto& g : stages_)
    if (g.lr <= 0.0) raise(1, "learning rate must be positive");
  const size_t mb = rows / static_cast<size_t>(m);
  // device-timeline bracket of the step: first device op (input H2D when from the host)
  // .. result D2H; read back by last_step_ms()
  CKF_CUDA(cudaEventRecord(sb_ev_, st_));
  const auto host_t0 = std::chrono::steady_clock::now();
  auto host_tg = host_t0;

  const size_t xcols = d_.block == CKF_BLOCK_MLP ? d_.in : d_.T + 1;
  const size_t xelt = d_.block == CKF_BLOCK_MLP ? master_bytes() : sizeof(int);
  const size_t ycols = d_.block == CKF_BLOCK_MLP ? (d_.task == CKF_TASK_REGRESSION ? d_.out : 1) : 0;
  const size_t yelt = d_.task == CKF_TASK_REGRESSION ? master_bytes() : sizeof(int);

  const char* xd = static_cast<const char*>(x);
  const char* yd = static_cast<const char*>(y);
  if (!on_device) {
    impl_->eng = this;
    void* xb = ws(rows * xcols * xelt, 0);
    if (d_.block == CKF_BLOCK_MLP) {
      // host inputs arrive as fp64 (the reference's Matrix); convert to the master dtype
      void* tmp = ws(rows * std::max(xcols, ycols) * sizeof(double), 2);
      CKF_CUDA(cudaMemcpyAsync(tmp, x, rows * xcols * sizeof(double), cudaMemcpyHostToDevice, st_));
      if (fp64())
        CKF_CUDA(cudaMemcpyAsync(xb, tmp, rows * xcols * 8, cudaMemcpyDeviceToDevice, st_));
      else
        k::convert(static_cast<const double*>(tmp), static_cast<float*>(xb), rows * xcols, st_);
      void* yb = ws(rows * ycols * yelt, 1);
      if (d_.task == CKF_TASK_REGRESSION) {
        CKF_CUDA(cudaMemcpyAsync(tmp, y, rows * ycols * sizeof(double), cudaMemcpyHostToDevice, st_));
        if (fp64())
          CKF_CUDA(cudaMemcpyAsync(yb, tmp, rows * ycols * 8, cudaMemcpyDeviceToDevice, st_));
        else
          k::convert(static_cast<const double*>(tmp), static_cast<float*>(yb), rows * ycols, st_);
      } else {
        std::vector<int> lab(rows);
        const double* yh = static_cast<const double*>(y);
        for (size_t i = 0; i < rows; ++i) {
          const double l = yh[i];
          if (l < 0 || l >= static_cast<double>(d_.out)) raise(1, "label out of range for output_dim");
          lab[i] = static_cast<int>(l);
        }
        CKF_CUDA(cudaMemcpyAsync(yb, lab.data(), rows * sizeof(int), cudaMemcpyHostToDevice, st_));
        CKF_CUDA(cudaStreamSynchronize(st_));
      }
      yd = static_cast<const char*>(yb);
    } else {
      CKF_CUDA(cudaMemcpyAsync(xb, x, rows * xcols * xelt, cudaMemcpyHostToDevice, st_));
    }
    xd = static_cast<const char*>(xb);
  }

  auto xk = [&](int k) { return xd + static_cast<size_t>(k) * mb * xcols * xelt; };
  auto yk = [&](int k) { return yd ? yd + static_cast<size_t>(k) * mb * ycols * yelt : nullptr; };
  auto ok = [&](int k) { return orders + static_cast<size_t>(k) * d_.s; };
  impl_->begin_iteration(m, mb);
  pev_used_ = 0;
  dp_pending_ = false;
  size_t nloss = static_cast<size_t>(m);
  bool flushed = false;
  // fusion needs every stage on this rank, the sequential schedule, and no virtual placement
  // (hop logging emulates a partitioned pipeline's transfers on one GPU)
  bool resident = schedule_ == 0 && !log_hops_;
  for (size_t i = 0; i < d_.s; ++i) resident = resident && mine(owner_of_stage(static_cast<int>(i + 1)));
  const int gsz = resident ? fused_group_size(m, mb) : 1;
  if (gsz > 1) {
    // All stages resident: microbatches sharing an execution order run as one
    // fused forward + backward (GEMM M = group tokens instead of one microbatch).
    // Same arithmetic as the reference's loop (pipeline.cpp:66-81): every token's
    // loss gradient is still scaled by 1/(microbatch tokens), the weight gradients
    // are summed over all tokens by the deferred W pass, and each group reports
    // the sum of its members' mean losses.  Groups keep microbatch-index order
    // within an order class; a class of non-contiguous microbatches (CheckFree+
    // swapped_half) has its token rows gathered first.
    std::vector<std::vector<int>> cls;
    for (int k = 0; k < m; ++k) {
      size_t c = 0;
      for (; c < cls.size(); ++c)
        if (std::equal(ok(k), ok(k) + d_.s, ok(cls[c][0]))) break;
      if (c == cls.size()) cls.emplace_back();
      cls[c].push_back(k);
    }
    std::vector<std::vector<int>> groups;
    for (const auto& c : cls)
      for (size_t i = 0; i < c.size(); i += static_cast<size_t>(gsz))
        groups.emplace_back(c.begin() + static_cast<long>(i),
                            c.begin() + static_cast<long>(std::min(c.size(), i + static_cast<size_t>(gsz))));
    const size_t xrow = mb * xcols * xelt;
    auto body = [&]() {
    impl_->loss_rows = mb;
    int woff = 0;
    for (size_t j = 0; j < groups.size(); ++j) {
      const auto& g = groups[j];
      const char* xg = xk(g[0]);
      bool contiguous = true;
      for (size_t i = 1; i < g.size(); ++i) contiguous = contiguous && g[i] == g[0] + static_cast<int>(i);
      if (!contiguous) {
        char* gb = static_cast<char*>(ws(g.size() * xrow, 3));
        for (size_t i = 0; i < g.size(); ++i)
          CKF_CUDA(cudaMemcpyAsync(gb + i * xrow, xk(g[i]), xrow, cudaMemcpyDeviceToDevice, st_));
        xg = gb;
      }
      impl_->wk = woff;
      {
        NvtxRange nv("ckf.group.fwd");
        impl_->mb_forward(0, ok(g[0]), xg, nullptr, g.size() * mb, true, scal_ + j);
      }
      {
        NvtxRange nv("ckf.group.bwd");
        impl_->mb_backward(0, ok(g[0]), xg, g.size() * mb);
      }
      if (redundant_) impl_->redundant_forward(ok(g[0]), xg, g.size() * mb);
      woff += static_cast<int>(g.size());
    }
    impl_->loss_rows = 0;
    NvtxRange nv("ckf.wgrad_pass");
    impl_->flush_grads();
    };
    // The fused step is a fixed launch sequence: after one eager pass with the same shape,
    // inputs and buffers, it is captured once as a CUDA graph and replayed (one launch per
    // iteration instead of ~300; Adam stays outside because its scalars change every step).
    // Any workspace reallocation (alloc_epoch) or a different order / group layout re-captures.
    const bool want_graph = graphs_ && !kt_on_;
    std::vector<long> key;
    if (want_graph) {
      key = {m, static_cast<long>(mb), static_cast<long>(reinterpret_cast<intptr_t>(xd)), gsz, alloc_epoch(),
             impl_->state_token(), redundant_ ? 1L : 0L};
      for (int k = 0; k < m; ++k) key.insert(key.end(), ok(k), ok(k) + d_.s);
    }
    if (step_debug()) {
      host_tg = std::chrono::steady_clock::now();
      CKF_CUDA(cudaEventRecord(sg_ev_, st_));
    }
    if (want_graph && gexec_ && key == gkey_) {
      CKF_CUDA(cudaGraphLaunch(gexec_, st_));
      launch_counter() += graph_kernels_;  // the replayed kernel nodes are this iteration's launches
    } else if (want_graph && key == gseen_) {
      if (gexec_) {
        cudaGraphExecDestroy(gexec_);
        gexec_ = nullptr;
      }
      cudaGraph_t graph = nullptr;
      const long n0 = launch_counter();
      CKF_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
      try {
        body();
      } catch (...) {
        cudaStreamEndCapture(st_, &graph);
        if (graph) cudaGraphDestroy(graph);
        graphs_ = false;
        throw;
      }
      CKF_CUDA(cudaStreamEndCapture(st_, &graph));
      graph_kernels_ = launch_counter() - n0;  // kernels captured (not executed during capture)
      CKF_CUDA(cudaGraphInstantiate(&gexec_, graph, 0));
      CKF_CUDA(cudaGraphUpload(gexec_, st_));  // device-side setup now, not on the first replay
      CKF_CUDA(cudaGraphDestroy(graph));
      gkey_ = key;
      gkey_[4] = alloc_epoch();  // (capture allocates nothing; kept exact anyway)
      CKF_CUDA(cudaGraphLaunch(gexec_, st_));
    } else {
      body();
      if (want_graph) gseen_ = key;
    }
    flushed = true;
    nloss = groups.size();
  } else if (schedule_ == 2 && impl_->supports_plan()) {
    run_plan(orders, m, xd, mb, mb * xcols * xelt);  // 1F1B over the placement (host::pipeline_plan)
  } else if (schedule_ == 0) {
    for (int k = 0; k < m; ++k) {
      impl_->microbatch(k, ok(k), xk(k), yk(k), mb, true, scal_ + k);
      if (redundant_) impl_->redundant_forward(ok(k), xk(k), mb);
    }
  } else {
    // GPipe: all forwards, then all backwards in microbatch order (per-stage accumulation
    // order is the reference's, pipeline.cpp:66-81); hops are issued in one global order
    // on every rank, so NCCL send/recv pair up without deadlock
    for (int k = 0; k < m; ++k) {
      impl_->wk = k;
      impl_->mb_forward(k, ok(k), xk(k), yk(k), mb, true, scal_ + k);
    }
    for (int k = 0; k < m; ++k) {
      impl_->wk = k;
      impl_->mb_backward(k, ok(k), xk(k), mb);
    }
  }
  if (!flushed) impl_->flush_grads();
  // data parallelism: sum every owned group's gradient over the replicas (each replica ran
  // its own m microbatches of the global batch), then Adam with 1/(m*R).  The stage groups were
  // all-reduced layer by layer on the data-parallel stream while the remaining weight-gradient
  // GEMMs ran (grad_bucket_ready); the edge groups (and everything, when the weight gradients
  // were not deferred) follow here; the optimizer waits for the stream.
  if (replicas_ > 1) {
    cudaEvent_t ev = plan_event();
    CKF_CUDA(cudaEventRecord(ev, st_));
    CKF_CUDA(cudaStreamWaitEvent(dst_, ev, 0));
    for (ParamGroup* g : owned_groups()) {
      const bool edge = g == &embed_ || g == &deembed_;
      if (dp_pending_ && !edge) continue;
      nccl_check(nccl().AllReduce(g->g, g->g, g->n, fp64() ? /*ncclFloat64*/ 8 : /*ncclFloat32*/ 7, /*ncclSum*/ 0,
                                  dp_comm_, dst_),
                 "ncclAllReduce (data parallel)");
    }
    cudaEvent_t done = plan_event();
    CKF_CUDA(cudaEventRecord(done, dst_));
    CKF_CUDA(cudaStreamWaitEvent(st_, done, 0));
    dp_pending_ = false;
  }
  // mean loss in microbatch order, then *1/m (model.cpp:299-312, pipeline.cpp:82-83)
  std::vector<double> losses(nloss);
  const double inv = 1.0 / (static_cast<double>(m) * replicas_);
  NvtxRange nv_adam("ckf.adam_omega");
  for (size_t i = 0; i < d_.s; ++i) adam_group(stages_[i], stages_[i].lr, inv, scal_ + 2048 + i);
  adam_group(embed_, edge_lr, inv, scal_ + 3000);
  adam_group(deembed_, edge_lr, inv, scal_ + 3001);
  if (redundant_) {  // post-step refresh of every stage's hot copy
    if (rc_replica_.size() != d_.s) rc_replica_.assign(d_.s, nullptr);
    for (size_t i = 0; i < d_.s; ++i) {
      ParamGroup& g = stages_[i];
      if (!g.owned || g.n == 0) continue;
      if (!rc_replica_[i]) CKF_CUDA(cudaMalloc(&rc_replica_[i], g.n * master_bytes()));
      kt_begin();
      CKF_CUDA(cudaMemcpyAsync(rc_replica_[i], g.w, g.n * master_bytes(), cudaMemcpyDeviceToDevice, st_));
      kt_end(KC_RECOVER, 0.0, 2.0 * g.n * master_bytes());
    }
  }
  if (auto_replicas_) refresh_edge_replicas();  // CheckFree+ (trainer.cpp:83-84), inside the step
  std::vector<double> om(d_.s);
  CKF_CUDA(cudaMemcpyAsync(losses.data(), scal_, nloss * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaMemcpyAsync(om.data(), scal_ + 2048, d_.s * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaEventRecord(se_ev_, st_));
  // Block (not spin) until the step is done: a ~50 ms spin per step burns a whole core of
  // the host's CPU quota, and quota throttling later stalls the launching thread for tens
  // of ms right when the next step must be enqueued.
  CKF_CUDA(cudaEventSynchronize(se_ev_));
  if (step_debug()) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, sb_ev_, sg_ev_);
    cudaEventElapsedTime(&b, sg_ev_, se_ev_);
    const double host = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    const double hg = std::chrono::duration<double, std::milli>(host_tg - host_t0).count();
    std::fprintf(stderr, "step_debug start->graph %.3f ms graph->end %.3f ms host %.3f ms host-start->graph %.3f ms\n", a,
                 b, host, hg);
  }
  kt_collect();
  double total = 0.0;
  for (double l : losses) total += l;
  total *= inv;  // this replica's share of the global mean loss
  if (nranks_ > 1 && comm_) {
    // every rank learns every stage's omega (the recovery reads its neighbours') and the loss
    // (placement without a communicator -- the peer-transport tests -- returns this rank's own)
    std::vector<double> v(d_.s + 1, 0.0);
    for (size_t i = 0; i < d_.s; ++i) v[i] = stages_[i].owned && replica_ == 0 ? om[i] : 0.0;
    v[d_.s] = mine(owner_of_deembed()) ? total : 0.0;
    double* dv = scal_ + 3100;
    CKF_CUDA(cudaMemcpyAsync(dv, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, st_));
    nccl_check(nccl().AllReduce(dv, dv, v.size(), /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm_, st_), "ncclAllReduce");
    CKF_CUDA(cudaMemcpyAsync(v.data(), dv, v.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
    CKF_CUDA(cudaStreamSynchronize(st_));
    for (size_t i = 0; i < d_.s; ++i) om[i] = v[i];
    total = v[d_.s];
  }
  bool finite = std::isfinite(total);
  for (size_t i = 0; i < d_.s; ++i) {
    if (!stages_[i].owned && nranks_ == 1) continue;
    stages_[i].omega = om[i];
    if (!std::isfinite(om[i])) finite = false;
  }
  if (!finite) raise(2, "non-finite gradient or activation", iteration);
  if (loss) *loss = total;
  if (omegas)
    for (size_t i = 0; i < d_.s; ++i) omegas[i] = stages_[i].omega;
}

// ------------------------------------------------------------------ checkpointing baseline
void Engine::checkpoint_save(long iteration) {
  CKF_CUDA(cudaSetDevice(d_.device));
  const size_t ng = d_.s + 2;
  if (ckpt_.size() != ng) ckpt_.assign(ng, CkptGroup{});
  auto grp = [&](size_t i) -> ParamGroup& { return i < d_.s ? stages_[i] : i == d_.s ? embed_ : deembed_; };
  for (size_t i = 0; i < ng; ++i) {
    ParamGroup& g = grp(i);
    CkptGroup& c = ckpt_[i];
    c.step = g.step;
    c.omega = g.omega;
    c.lr = g.lr;
    if (!g.owned || g.n == 0) continue;
    const size_t b = g.n * master_bytes();
    const size_t need = 3 * b + (g.wlp ? g.n * sizeof(__nv_bfloat16) : 0);
    if (c.bytes < need) {
      cudaFree(c.buf);
      CKF_CUDA(cudaMalloc(&c.buf, need));
      c.bytes = need;
    }
    char* p = static_cast<char*>(c.buf);
    CKF_CUDA(cudaMemcpyAsync(p, g.w, b, cudaMemcpyDeviceToDevice, st_));
    CKF_CUDA(cudaMemcpyAsync(p + b, g.m, b, cudaMemcpyDeviceToDevice, st_));
    CKF_CUDA(cudaMemcpyAsync(p + 2 * b, g.v, b, cudaMemcpyDeviceToDevice, st_));
    if (g.wlp) CKF_CUDA(cudaMemcpyAsync(p + 3 * b, g.wlp, g.n * sizeof(__nv_bfloat16), cudaMemcpyDeviceToDevice, st_));
  }
  ckpt_edge_lr_ = edge_lr;
  ckpt_iter_ = iteration;
  ckpt_valid_ = true;
  CKF_CUDA(cudaStreamSynchronize(st_));
}

long Engine::checkpoint_restore(const int* stages, int n_stages, double* red, float* ms) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (!ckpt_valid_) raise(1, "no checkpoint to restore");
  auto grp = [&](size_t i) -> ParamGroup& { return i < d_.s ? stages_[i] : i == d_.s ? embed_ : deembed_; };
  CKF_CUDA(cudaEventRecord(ev0_, st_));
  for (int k = 0; k < n_stages; ++k) {  // reduction error of the failed stages (trainer.cpp:179-189)
    const int sid = stages[k];
    if (sid < 1 || sid > static_cast<int>(d_.s)) raise(1, "stage id out of range");
    ParamGroup& g = stages_[static_cast<size_t>(sid - 1)];
    if (!red || !g.owned || g.n == 0) continue;
    if (fp64())
      k::sum_sq_diff(static_cast<const double*>(g.w), static_cast<const double*>(ckpt_[sid - 1].buf), g.n,
                     scal_ + 3200 + k, red_, st_);
    else
      k::sum_sq_diff(static_cast<const float*>(g.w), static_cast<const float*>(ckpt_[sid - 1].buf), g.n,
                     scal_ + 3200 + k, red_, st_);
  }
  for (size_t i = 0; i < ckpt_.size(); ++i) {
    ParamGroup& g = grp(i);
    const CkptGroup& c = ckpt_[i];
    g.step = c.step;
    g.omega = c.omega;
    g.lr = c.lr;
    if (!g.owned || g.n == 0) continue;
    const size_t b = g.n * master_bytes();
    const char* p = static_cast<const char*>(c.buf);
    CKF_CUDA(cudaMemcpyAsync(g.w, p, b, cudaMemcpyDeviceToDevice, st_));
    CKF_CUDA(cudaMemcpyAsync(g.m, p + b, b, cudaMemcpyDeviceToDevice, st_));
    CKF_CUDA(cudaMemcpyAsync(g.v, p + 2 * b, b, cudaMemcpyDeviceToDevice, st_));
    if (g.wlp) CKF_CUDA(cudaMemcpyAsync(g.wlp, p + 3 * b, g.n * sizeof(__nv_bfloat16), cudaMemcpyDeviceToDevice, st_));
    CKF_CUDA(cudaMemsetAsync(g.g, 0, b, st_));
  }
  edge_lr = ckpt_edge_lr_;
  CKF_CUDA(cudaEventRecord(ev1_, st_));
  std::vector<double> r(static_cast<size_t>(std::max(n_stages, 0)), 0.0);
  if (red && n_stages > 0)
    CKF_CUDA(cudaMemcpyAsync(r.data(), scal_ + 3200, r.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaStreamSynchronize(st_));
  float t = 0.f;
  CKF_CUDA(cudaEventElapsedTime(&t, ev0_, ev1_));
  if (nranks_ > 1 && comm_) {
    // multi-rank: each failed stage's reduction error comes from its owner (replica 0); the
    // restore time is the slowest rank's
    std::vector<double> v(r.size() + 1, 0.0);
    for (int k = 0; k < n_stages; ++k) {
      const int sid = stages[k];
      v[static_cast<size_t>(k)] = replica_ == 0 && stages_[static_cast<size_t>(sid - 1)].owned ? r[static_cast<size_t>(k)] : 0.0;
    }
    const auto all = allreduce_host(v);
    for (size_t k = 0; k < r.size(); ++k) r[k] = all[k];
    std::vector<double> tv(static_cast<size_t>(nranks_), 0.0);
    tv[static_cast<size_t>(rank_)] = t;
    const auto ts = allreduce_host(tv);
    for (double x : ts) t = std::max(t, static_cast<float>(x));
  }
  if (red)
    for (int k = 0; k < n_stages; ++k) red[k] = r[static_cast<size_t>(k)];
  if (ms) *ms = t;
  return ckpt_iter_;
}

float Engine::last_step_ms() {
  CKF_CUDA(cudaEventSynchronize(se_ev_));
  float ms = 0.f;
  CKF_CUDA(cudaEventElapsedTime(&ms, sb_ev_, se_ev_));
  return ms;
}

void Engine::upload(const void* x, const void* y, size_t rows, const void** xd, const void** yd) {
  const size_t xcols = d_.block == CKF_BLOCK_MLP ? d_.in : d_.T + 1;
  if (d_.block == CKF_BLOCK_LLAMA) {
    void* xb = ws(rows * xcols * sizeof(int), 0);
    CKF_CUDA(cudaMemcpyAsync(xb, x, rows * xcols * sizeof(int), cudaMemcpyHostToDevice, st_));
    *xd = xb;
    *yd = nullptr;
    return;
  }
  const size_t ycols = d_.task == CKF_TASK_REGRESSION ? d_.out : 1;
  void* tmp = ws(rows * std::max(xcols, ycols) * sizeof(double), 2);
  void* xb = ws(rows * xcols * master_bytes(), 0);
  CKF_CUDA(cudaMemcpyAsync(tmp, x, rows * xcols * 8, cudaMemcpyHostToDevice, st_));
  if (fp64())
    CKF_CUDA(cudaMemcpyAsync(xb, tmp, rows * xcols * 8, cudaMemcpyDeviceToDevice, st_));
  else
    k::convert(static_cast<const double*>(tmp), static_cast<float*>(xb), rows * xcols, st_);
  void* yb = ws(rows * ycols * (d_.task == CKF_TASK_REGRESSION ? master_bytes() : 4), 1);
  if (d_.task == CKF_TASK_REGRESSION) {
    CKF_CUDA(cudaMemcpyAsync(tmp, y, rows * ycols * 8, cudaMemcpyHostToDevice, st_));
    if (fp64())
      CKF_CUDA(cudaMemcpyAsync(yb, tmp, rows * ycols * 8, cudaMemcpyDeviceToDevice, st_));
    else
      k::convert(static_cast<const double*>(tmp), static_cast<float*>(yb), rows * ycols, st_);
  } else {
    std::vector<int> lab(rows);
    for (size_t i = 0; i < rows; ++i) {
      const double l = static_cast<const double*>(y)[i];
      if (l < 0 || l >= static_cast<double>(d_.out)) raise(1, "label out of range for output_dim");
      lab[i] = static_cast<int>(l);
    }
    CKF_CUDA(cudaMemcpyAsync(yb, lab.data(), rows * 4, cudaMemcpyHostToDevice, st_));
    CKF_CUDA(cudaStreamSynchronize(st_));
  }
  *xd = xb;
  *yd = yb;
}

double Engine::eval_loss(const int* order, const void* x, const void* y, size_t rows, bool on_device) {
  CKF_CUDA(cudaSetDevice(d_.device));
  validate_order(order, d_.s);
  if (rows == 0) raise(1, "empty batch");
  if (!on_device) upload(x, y, rows, &x, &y);
  double l = 0.0;
  if (d_.block == CKF_BLOCK_LLAMA && rows * d_.T > d_.max_rows) {
    // token-mean over equal-weight chunks of at most max_rows tokens
    const size_t cr = std::max<size_t>(1, d_.max_rows / d_.T);
    const int* xi = static_cast<const int*>(x);
    std::vector<std::pair<size_t, size_t>> chunks;
    for (size_t r0 = 0; r0 < rows; r0 += cr) chunks.push_back({r0, std::min(cr, rows - r0)});
    if (chunks.size() > 64) raise(1, "evaluation batch too large for the engine's max_rows");
    for (size_t i = 0; i < chunks.size(); ++i)
      impl_->microbatch(0, order, xi + chunks[i].first * (d_.T + 1), nullptr, chunks[i].second, false, scal_ + 4010 + i);
    std::vector<double> ls(chunks.size());
    CKF_CUDA(cudaMemcpyAsync(ls.data(), scal_ + 4010, ls.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
    CKF_CUDA(cudaStreamSynchronize(st_));
    for (size_t i = 0; i < chunks.size(); ++i) l += ls[i] * static_cast<double>(chunks[i].second);
    return share_from_head(l / static_cast<double>(rows));
  }
  impl_->microbatch(0, order, x, y, rows, false, scal_ + 4000);
  CKF_CUDA(cudaMemcpyAsync(&l, scal_ + 4000, sizeof(double), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaStreamSynchronize(st_));
  return share_from_head(l);
}

// Multi-rank: the loss exists on the de-embedding owner only; every rank returns replica 0's value.
double Engine::share_from_head(double v) {
  if (nranks_ <= 1 || !comm_) return v;
  const double mine_v = mine(owner_of_deembed()) && replica_ == 0 ? v : 0.0;
  return allreduce_host({mine_v})[0];
}

std::vector<double> Engine::allreduce_host(const std::vector<double>& v) {
  double* dv = scal_ + 3700;
  if (v.size() > 200) raise(1, "allreduce_host: at most 200 values");
  CKF_CUDA(cudaMemcpyAsync(dv, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, st_));
  nccl_check(nccl().AllReduce(dv, dv, v.size(), /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm_, st_), "ncclAllReduce");
  std::vector<double> out(v.size());
  CKF_CUDA(cudaMemcpyAsync(out.data(), dv, v.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaStreamSynchronize(st_));
  return out;
}

// Peer mappings for recovery over NVLink: every rank's IPC blob (ipc_export) all-gathered over
// the world communicator, then imported (stages of the same replica this rank does not own).
void Engine::exchange_peers() {
  if (nranks_ <= 1 || !comm_) return;
  if (!nccl().AllGather) raise(7, "ncclAllGather unavailable");
  constexpr size_t kBlob = 1 << 14;
  std::vector<char> mine_b(kBlob + 8, 0);
  const size_t n = ipc_export(mine_b.data() + 8, kBlob);
  std::memcpy(mine_b.data(), &n, 8);
  char* dev = static_cast<char*>(ws((kBlob + 8) * static_cast<size_t>(nranks_ + 1), 70));
  CKF_CUDA(cudaMemcpyAsync(dev, mine_b.data(), kBlob + 8, cudaMemcpyHostToDevice, st_));
  nccl_check(nccl().AllGather(dev, dev + kBlob + 8, kBlob + 8, /*ncclInt8*/ 0, comm_, st_), "ncclAllGather (IPC)");
  std::vector<char> all((kBlob + 8) * static_cast<size_t>(nranks_));
  CKF_CUDA(cudaMemcpyAsync(all.data(), dev + kBlob + 8, all.size(), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaStreamSynchronize(st_));
  std::vector<char> cat;
  for (int r = 0; r < nranks_; ++r) {
    const char* b = all.data() + static_cast<size_t>(r) * (kBlob + 8);
    size_t len = 0;
    std::memcpy(&len, b, 8);
    cat.insert(cat.end(), b + 8, b + 8 + len);
  }
  ipc_import(cat.data(), cat.size());
}

double Engine::accumulate(const int* order, const void* x, const void* y, size_t rows, bool on_device) {
  CKF_CUDA(cudaSetDevice(d_.device));
  validate_order(order, d_.s);
  if (rows == 0) raise(1, "empty batch");
  if (!on_device) upload(x, y, rows, &x, &y);
  impl_->begin_iteration(1, rows);
  impl_->microbatch(0, order, x, y, rows, true, scal_ + 4001);
  impl_->flush_grads();
  double l = 0.0;
  CKF_CUDA(cudaMemcpyAsync(&l, scal_ + 4001, sizeof(double), cudaMemcpyDeviceToHost, st_));
  CKF_CUDA(cudaStreamSynchronize(st_));
  kt_collect();
  return l;
}

void Engine::zero_grad() {
  CKF_CUDA(cudaSetDevice(d_.device));
  for (auto& g : stages_)
    if (g.owned && g.n) CKF_CUDA(cudaMemsetAsync(g.g, 0, g.n * master_bytes(), st_));
  for (ParamGroup* g : {&embed_, &deembed_})
    if (g->owned && g->n) CKF_CUDA(cudaMemsetAsync(g->g, 0, g->n * master_bytes(), st_));
  CKF_CUDA(cudaStreamSynchronize(st_));
}

void Engine::export_grad(ParamGroup& g, double* out) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (!g.owned) raise(3, "parameter group is not resident on this rank");
  if (fp64()) {
    CKF_CUDA(cudaMemcpyAsync(out, g.g, g.n * 8, cudaMemcpyDeviceToHost, st_));
  } else {
    double* tmp = static_cast<double*>(ws(g.n * 8, 3));
    k::convert(static_cast<const float*>(g.g), tmp, g.n, st_);
    CKF_CUDA(cudaMemcpyAsync(out, tmp, g.n * 8, cudaMemcpyDeviceToHost, st_));
  }
  CKF_CUDA(cudaStreamSynchronize(st_));
}

void Engine::predict_device(const int* order, const void* x_dev, size_t rows, void* pred_dev) {
  validate_order(order, d_.s);
  impl_->predict(order, x_dev, rows, pred_dev);
}

void Engine::predict(const int* order, const double* x_host, size_t rows, double* pred_host) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (d_.block != CKF_BLOCK_MLP) raise(1, "predict is defined for the residual-MLP block");
  validate_order(order, d_.s);
  void* tmp = ws(rows * std::max(d_.in, d_.out) * 8, 2);
  void* xb = ws(rows * d_.in * master_bytes(), 0);
  void* pb = ws(rows * d_.out * master_bytes(), 1);
  CKF_CUDA(cudaMemcpyAsync(tmp, x_host, rows * d_.in * 8, cudaMemcpyHostToDevice, st_));
  if (fp64())
    CKF_CUDA(cudaMemcpyAsync(xb, tmp, rows * d_.in * 8, cudaMemcpyDeviceToDevice, st_));
  else
    k::convert(static_cast<const double*>(tmp), static_cast<float*>(xb), rows * d_.in, st_);
  impl_->predict(order, xb, rows, pb);
  if (fp64()) {
    CKF_CUDA(cudaMemcpyAsync(pred_host, pb, rows * d_.out * 8, cudaMemcpyDeviceToHost, st_));
  } else {
    k::convert(static_cast<const float*>(pb), static_cast<double*>(tmp), rows * d_.out, st_);
    CKF_CUDA(cudaMemcpyAsync(pred_host, tmp, rows * d_.out * 8, cudaMemcpyDeviceToHost, st_));
  }
  CKF_CUDA(cudaStreamSynchronize(st_));
}

// ------------------------------------------------------------------ replicas
void Engine::refresh_edge_replicas() {
  // recovery.cpp:80-84: replica := (E, E^-1); held by the GPUs of stages 2 and s-1
  CKF_CUDA(cudaSetDevice(d_.device));
  const int hold_e = owner_of_stage(d_.s >= 2 ? 2 : 1);
  const int hold_d = owner_of_stage(d_.s >= 2 ? static_cast<int>(d_.s) - 1 : 1);
  const size_t be = embed_.n * master_bytes(), bd = deembed_.n * master_bytes();
  if (mine(hold_e) && !rep_embed_) CKF_CUDA(cudaMalloc(&rep_embed_, be));
  if (mine(hold_d) && !rep_deembed_) CKF_CUDA(cudaMalloc(&rep_deembed_, bd));
  if (mine(owner_of_embed()) && mine(hold_e))
    CKF_CUDA(cudaMemcpyAsync(rep_embed_, embed_.w, be, cudaMemcpyDeviceToDevice, st_));
  else
    hop(mine(owner_of_embed()) ? embed_.w : rep_embed_, be, owner_of_embed(), hold_e);
  if (mine(owner_of_deembed()) && mine(hold_d))
    CKF_CUDA(cudaMemcpyAsync(rep_deembed_, deembed_.w, bd, cudaMemcpyDeviceToDevice, st_));
  else
    hop(mine(owner_of_deembed()) ? deembed_.w : rep_deembed_, bd, owner_of_deembed(), hold_d);
  replica_staleness_ = 0;
}

void Engine::kill_stage(int sid) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (sid < 1 || static_cast<size_t>(sid) > d_.s) raise(1, "stage id out of range");
  ParamGroup& g = stage(sid);
  auto poison = [&](ParamGroup& p) {
    if (!p.owned) return;
    if (fp64()) {
      for (void* b : {p.w, p.m, p.v}) k::poison(static_cast<double*>(b), p.n, st_);
    } else {
      for (void* b : {p.w, p.m, p.v}) k::poison(static_cast<float*>(b), p.n, st_);
    }
    if (p.wlp) k::fill(p.wlp, NAN, p.n, st_);
  };
  poison(g);
  // the edge layers live on the GPUs of stages 1 and s (cost_model.cpp:264-268)
  if (sid == 1) poison(embed_);
  if (static_cast<size_t>(sid) == d_.s) poison(deembed_);
}

// ------------------------------------------------------------------ recovery
ckf_recovery_report Engine::recover_stage(int sid, int mode, int moments, double lr_bump, uint64_t reinit_seed,
                                          bool want_red) {
  NvtxRange nv_rec("ckf.recover_stage");
  CKF_CUDA(cudaSetDevice(d_.device));
  const int s = static_cast<int>(d_.s);
  if (sid < 1 || sid > s) raise(1, "stage id out of range");
  if (lr_bump <= 0.0) raise(1, "lr_bump must be positive");
  ckf_recovery_report rep{0, 0.0, 0.0};
  ParamGroup& f = stage(sid);
  const bool edge = sid == 1 || sid == s;
  if (edge && mode != CKF_REC_EDGE)
    raise(5, std::string("stage ") + std::to_string(sid) +
                 " is a first/last stage: only the CheckFree+ edge copy can recover it (single neighbour)");
  if (!edge && mode == CKF_REC_EDGE) raise(1, "edge recovery applies to the first and last stage only");
  if (mode == CKF_REC_EDGE && replica_staleness_ != 0)
    raise(1, "edge replica is stale; refresh must precede recovery");  // recovery.cpp:98
  if (f.lr <= 0.0) raise(1, "learning rate must be positive");
  if (mode < CKF_REC_CHECKFREE || mode > CKF_REC_EDGE) raise(1, "unknown recovery mode");

  const size_t mb = master_bytes();
  const size_t bytes = f.n * mb;
  const int F = owner_of_stage(sid);  // the replacement GPU of the failed stage
  const bool local = mine(F);
  ParamGroup* nbp = mode == CKF_REC_EDGE ? &stage(sid == 1 ? 2 : s - 1) : (sid > 1 ? &stage(sid - 1) : nullptr);
  ParamGroup* nxp = mode != CKF_REC_EDGE && sid < s ? &stage(sid + 1) : nullptr;
  const bool avg = moments == CKF_MOM_AVERAGED && (mode == CKF_REC_CHECKFREE || mode == CKF_REC_EDGE);

  // latency = kill-to-ready on the replacement GPU: the clock starts BEFORE any neighbour
  // transfer, so a multi-GPU recovery's pull (or peer reads inside the kernel) is counted
  if (local) CKF_CUDA(cudaEventRecord(ev0_, st_));
  // ---- bring the neighbour state this recovery reads onto F (peer pulls over NCCL;
  //      a no-op when everything is resident, e.g. on one GPU)
  std::vector<std::pair<void**, void*>> borrowed;  // (slot, temp) to undo
  auto pull = [&](void** slot, int src, size_t nbytes, int ws_slot) {
    if (src == F) return;
    void* tmp = local ? ws(nbytes, ws_slot) : nullptr;
    if (local) {
      borrowed.push_back({slot, *slot});
      *slot = tmp;
    }
    hop(local ? tmp : *slot, nbytes, src, F);
  };
  // neighbours mapped from peer HBM (ipc_import): the recovery kernel reads them in place
  auto peer_of = [&](ParamGroup* g) -> PeerStage* {
    if (!g || g->owned || peer_.empty()) return nullptr;
    PeerStage& p = peer_[static_cast<size_t>(g - stages_.data())];
    return p.w ? &p : nullptr;
  };
  auto borrow_peer = [&](ParamGroup* g) {
    PeerStage* p = peer_of(g);
    if (!p || !local) return false;
    for (auto [slot, src] : {std::make_pair(&g->w, p->w), std::make_pair(&g->m, p->m), std::make_pair(&g->v, p->v)}) {
      borrowed.push_back({slot, *slot});
      *slot = src;
    }
    return true;
  };
  // every rank imported every peer blob (ipc_import), so all ranks agree on peer_ready_ and
  // the neighbours' owners skip the NCCL sends the replacement GPU no longer posts
  if (peer_ready_) {
    borrow_peer(nbp);
    borrow_peer(nxp);
  }
  if (nranks_ > 1) {
    const bool need_prev = mode != CKF_REC_RANDOM && !peer_ready_;
    if (nbp && need_prev) {
      const int src = owner_of_stage(mode == CKF_REC_EDGE ? (sid == 1 ? 2 : s - 1) : sid - 1);
      pull(&nbp->w, src, bytes, 60);
      if (avg) {
        pull(&nbp->m, src, bytes, 61);
        pull(&nbp->v, src, bytes, 62);
      }
    }
    if (nxp && !peer_ready_ && (mode == CKF_REC_CHECKFREE || mode == CKF_REC_UNIFORM)) {
      const int src = owner_of_stage(sid + 1);
      pull(&nxp->w, src, bytes, 63);
      if (avg) {
        pull(&nxp->m, src, bytes, 64);
        pull(&nxp->v, src, bytes, 65);
      }
    }
    if (mode == CKF_REC_EDGE) {  // the replica lives on the neighbour's GPU (recovery.cpp:80-84)
      void** rep = sid == 1 ? &rep_embed_ : &rep_deembed_;
      const size_t rb = (sid == 1 ? embed_.n : deembed_.n) * mb;
      pull(rep, owner_of_stage(sid == 1 ? 2 : s - 1), rb, 66);
    }
  }

  double* red_dev = want_red ? scal_ + 3500 : nullptr;
  long new_step = 0;
  bool fused = false;
  if (mode == CKF_REC_EDGE) {
    ParamGroup& nb = *nbp;
    ParamGroup& eg = sid == 1 ? embed_ : deembed_;
    if (local) {
      if (want_red) {
        if (fp64())
          k::sum_sq_diff(static_cast<const double*>(f.w), static_cast<const double*>(nb.w), f.n, red_dev, red_, st_);
        else
          k::sum_sq_diff(static_cast<const float*>(f.w), static_cast<const float*>(nb.w), f.n, red_dev, red_, st_);
      }
      CKF_CUDA(cudaMemcpyAsync(f.w, nb.w, bytes, cudaMemcpyDeviceToDevice, st_));
      CKF_CUDA(cudaMemcpyAsync(eg.w, sid == 1 ? rep_embed_ : rep_deembed_, eg.n * mb, cudaMemcpyDeviceToDevice, st_));
      CKF_CUDA(cudaMemsetAsync(eg.m, 0, eg.n * mb, st_));  // that edge's Adam state resets (trainer.cpp:218-224)
      CKF_CUDA(cudaMemsetAsync(eg.v, 0, eg.n * mb, st_));
      CKF_CUDA(cudaMemsetAsync(eg.g, 0, eg.n * mb, st_));
      if (eg.wlp) k::convert(static_cast<const float*>(eg.w), eg.wlp, eg.n, st_);
      if (avg) {  // single neighbour: copy, like the weights (trainer.cpp:225-226)
        CKF_CUDA(cudaMemcpyAsync(f.m, nb.m, bytes, cudaMemcpyDeviceToDevice, st_));
        CKF_CUDA(cudaMemcpyAsync(f.v, nb.v, bytes, cudaMemcpyDeviceToDevice, st_));
      } else {
        CKF_CUDA(cudaMemsetAsync(f.m, 0, bytes, st_));
        CKF_CUDA(cudaMemsetAsync(f.v, 0, bytes, st_));
      }
    }
    eg.step = 0;
    new_step = avg ? nb.step : 0;
  } else {
    ParamGroup& p = *nbp;
    ParamGroup& n = *nxp;
    double op = p.omega, on = n.omega;
    if (op < 0.0 || on < 0.0) raise(1, "gradient norms must be nonnegative");
    if (mode == CKF_REC_CHECKFREE) {
      if (op + on == 0.0) rep.degenerate = 1;  // recovery.cpp:63-68
    } else if (mode == CKF_REC_UNIFORM) {
      op = on = 1.0;
    } else if (mode == CKF_REC_COPY_PREV) {
      op = 1.0;
      on = 0.0;
    }
    if (local) {
      if (mode == CKF_REC_RANDOM) {
        void* tmp = want_red ? ws(bytes, 3) : nullptr;
        if (want_red) CKF_CUDA(cudaMemcpyAsync(tmp, f.w, bytes, cudaMemcpyDeviceToDevice, st_));
        impl_->init_stage(sid, reinit_seed, f.w);
        if (want_red) {
          if (fp64())
            k::sum_sq_diff(static_cast<const double*>(tmp), static_cast<const double*>(f.w), f.n, red_dev, red_, st_);
          else
            k::sum_sq_diff(static_cast<const float*>(tmp), static_cast<const float*>(f.w), f.n, red_dev, red_, st_);
        }
      } else if (mode == CKF_REC_COPY_PREV) {
        if (want_red) {
          if (fp64())
            k::sum_sq_diff(static_cast<const double*>(f.w), static_cast<const double*>(p.w), f.n, red_dev, red_, st_);
          else
            k::sum_sq_diff(static_cast<const float*>(f.w), static_cast<const float*>(p.w), f.n, red_dev, red_, st_);
        }
        CKF_CUDA(cudaMemcpyAsync(f.w, p.w, bytes, cudaMemcpyDeviceToDevice, st_));
      } else {
        // CheckFree / uniform average: ONE streaming pass makes the stage ready -- weights
        // (recovery.cpp:57-73), moments Fresh or omega-weighted (trainer.cpp:263-269), gradient
        // accumulator zeroed, bf16 shadow, and ||old - new||^2 from the same read of the old W.
        // The neighbour pointers may be peer mappings of another GPU's HBM.
        kt_begin();
        auto run = [&](auto* tag) {
          using T = std::remove_pointer_t<decltype(tag)>;
          k::StageRecovery<T> r;
          r.wp = static_cast<const T*>(p.w);
          r.wn = static_cast<const T*>(n.w);
          r.w = static_cast<T*>(f.w);
          r.m = static_cast<T*>(f.m);
          r.v = static_cast<T*>(f.v);
          r.g = static_cast<T*>(f.g);
          r.wlp = f.wlp;
          r.n = f.n;
          r.op = op;
          r.on = on;
          r.averaged = avg;
          if (avg) {
            r.mp = static_cast<const T*>(p.m);
            r.mn = static_cast<const T*>(n.m);
            r.vp = static_cast<const T*>(p.v);
            r.vn = static_cast<const T*>(n.v);
            r.mop = p.omega;
            r.mon = n.omega;
          }
          r.old_sq = red_dev;
          k::recover_stage(r, red_, st_);
        };
        if (fp64())
          run(static_cast<double*>(nullptr));
        else
          run(static_cast<float*>(nullptr));
        fused = true;
        const double pb = static_cast<double>(master_bytes());
        kt_end(KC_RECOVER, 0.0,
               static_cast<double>(f.n) * (pb * (6.0 + (avg ? 4.0 : 0.0) + (want_red ? 1.0 : 0.0)) + (f.wlp ? 2.0 : 0.0)));
      }
      if (!fused) {
        if (avg) {
          // omega-weighted moments (trainer.cpp:263-269)
          const double wp = p.omega, wn = n.omega;
          if (fp64()) {
            k::weighted_or_uniform(static_cast<const double*>(p.m), static_cast<const double*>(n.m),
                                   static_cast<double*>(f.m), f.n, wp, wn, st_);
            k::weighted_or_uniform(static_cast<const double*>(p.v), static_cast<const double*>(n.v),
                                   static_cast<double*>(f.v), f.n, wp, wn, st_);
          } else {
            k::weighted_or_uniform(static_cast<const float*>(p.m), static_cast<const float*>(n.m),
                                   static_cast<float*>(f.m), f.n, wp, wn, st_);
            k::weighted_or_uniform(static_cast<const float*>(p.v), static_cast<const float*>(n.v),
                                   static_cast<float*>(f.v), f.n, wp, wn, st_);
          }
        } else {
          CKF_CUDA(cudaMemsetAsync(f.m, 0, bytes, st_));
          CKF_CUDA(cudaMemsetAsync(f.v, 0, bytes, st_));
        }
      }
    }
    new_step = avg ? std::min(p.step, n.step) : 0;
  }
  if (local) {
    if (!fused) {
      CKF_CUDA(cudaMemsetAsync(f.g, 0, bytes, st_));
      if (f.wlp) k::convert(static_cast<const float*>(f.w), f.wlp, f.n, st_);
    }
    CKF_CUDA(cudaEventRecord(ev1_, st_));
  }
  f.step = new_step;
  f.lr = lr_bump * f.lr;  // bump_lr (recovery.cpp:75-78), failed stage only
  f.omega = 0.0;          // trainer.cpp:276
  if (local && want_red)
    CKF_CUDA(cudaMemcpyAsync(&rep.reduction_error, red_dev, sizeof(double), cudaMemcpyDeviceToHost, st_));
  if (peer_ready_ && comm_) {
    // the neighbours' owners must not update the weights the replacement GPU reads in place
    // until its recovery kernel is done: an all-reduce enqueued behind it is the barrier
    nccl_check(nccl().AllReduce(scal_ + 3600, scal_ + 3600, 1, /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm_, st_),
               "ncclAllReduce (recovery barrier)");
  }
  CKF_CUDA(cudaStreamSynchronize(st_));
  kt_collect();
  for (auto it = borrowed.rbegin(); it != borrowed.rend(); ++it) *it->first = it->second;
  if (local) {
    float ms = 0.f;
    CKF_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
    rep.latency_ms = ms;
  }
  if (nranks_ > 1 && comm_) {  // every rank reports the replacement GPU's numbers (replica 0)
    const bool src = local && replica_ == 0;
    const auto v = allreduce_host({src ? rep.reduction_error : 0.0, src ? rep.latency_ms : 0.0});
    rep.reduction_error = v[0];
    rep.latency_ms = v[1];
  }
  return rep;
}

// ------------------------------------------------------------------ state exchange
void Engine::export_group(ParamGroup& g, double* w, double* m, double* v) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (!g.owned) raise(3, "parameter group is not resident on this rank");
  void* srcs[3] = {g.w, g.m, g.v};
  double* dsts[3] = {w, m, v};
  for (int i = 0; i < 3; ++i) {
    if (!dsts[i]) continue;
    if (fp64()) {
      CKF_CUDA(cudaMemcpyAsync(dsts[i], srcs[i], g.n * 8, cudaMemcpyDeviceToHost, st_));
    } else {
      double* tmp = static_cast<double*>(ws(g.n * 8, 3));
      k::convert(static_cast<const float*>(srcs[i]), tmp, g.n, st_);
      CKF_CUDA(cudaMemcpyAsync(dsts[i], tmp, g.n * 8, cudaMemcpyDeviceToHost, st_));
    }
    CKF_CUDA(cudaStreamSynchronize(st_));
  }
}

void Engine::import_group(ParamGroup& g, const double* w, const double* m, const double* v) {
  CKF_CUDA(cudaSetDevice(d_.device));
  if (!g.owned) raise(3, "parameter group is not resident on this rank");
  void* dsts[3] = {g.w, g.m, g.v};
  const double* srcs[3] = {w, m, v};
  for (int i = 0; i < 3; ++i) {
    if (!srcs[i]) continue;
    if (fp64()) {
      CKF_CUDA(cudaMemcpyAsync(dsts[i], srcs[i], g.n * 8, cudaMemcpyHostToDevice, st_));
    } else {
      double* tmp = static_cast<double*>(ws(g.n * 8, 3));
      CKF_CUDA(cudaMemcpyAsync(tmp, srcs[i], g.n * 8, cudaMemcpyHostToDevice, st_));
      k::convert(tmp, static_cast<float*>(dsts[i]), g.n, st_);
    }
    CKF_CUDA(cudaStreamSynchronize(st_));
  }
  if (w && g.wlp) k::convert(static_cast<const float*>(g.w), g.wlp, g.n, st_);
  CKF_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace ckf
