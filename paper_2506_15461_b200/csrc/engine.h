// Device-resident CheckFree / CheckFree+ engine (internal C++; exported only
// through include/ckf.h).
//
// One Engine per GPU.  It owns the master weights, gradient accumulators and
// Adam moments of the stages placed on its GPU (plus the edge layers when it
// hosts stage 1 / stage s), runs pipeline::run_iteration semantics
// (src/pipeline.cpp:58-95) and the recovery path (src/recovery.cpp:57-126,
// src/trainer.cpp:196-282).  Stage activations cross GPUs over NCCL
// send/recv when the placement spans ranks.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/ckf.h"
#include "common.cuh"
#include "host_logic.h"
#include "kernels.h"

#include <nvtx3/nvToolsExt.h>

namespace ckf {

// NVTX range over a scope (iteration, microbatch group, plan op, transfer, recovery, optimizer):
// nsys / ncu --nvtx timelines show the pipeline structure.  Header-only NVTX3; a no-op unless a
// tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Range {
  size_t first = 0, last = 0;  // 1-based inclusive (model.hpp:24-28)
  size_t count() const { return last - first + 1; }
};

struct Desc {
  int block = CKF_BLOCK_MLP;
  int prec = CKF_FP64;
  int act = CKF_ACT_TANH;
  int task = CKF_TASK_REGRESSION;
  size_t in = 16, hid = 64, d = 32, out = 16, L = 8, s = 4, heads = 1, T = 1, max_rows = 256;
  int device = 0;
  std::vector<Range> part;
};

// Flat buffers of one parameter group (a stage or an edge layer).  The
// master copy `w` has the engine's master dtype (fp64 in FP64 mode, fp32
// otherwise); `wlp` is the bf16 shadow the tensor-core GEMMs read.
struct ParamGroup {
  size_t n = 0;
  bool owned = true;
  void* w = nullptr;
  void* g = nullptr;
  void* m = nullptr;
  void* v = nullptr;
  __nv_bfloat16* wlp = nullptr;
  long step = 0;
  double omega = 0.0;
  double lr = 3e-4;
};

class Engine;

// Per-class kernel timing (bench.py's roofline evidence): when enabled, each
// tagged launch is bracketed by CUDA events on the engine stream and its
// algorithmic FLOPs / bytes are recorded; collect() folds them after a sync.
enum KClass { KC_GEMM = 0, KC_ATTN = 1, KC_ADAM = 2, KC_RECOVER = 3, KC_NORM = 4, KC_LOSS = 5, KC_COMM = 6, KC_N = 7 };
struct KStat {
  double ms = 0.0, flops = 0.0, bytes = 0.0;
  long launches = 0;
};

// Block-specific arithmetic (residual MLP of model.hpp:55-60, or LLaMA).
struct BlockImpl {
  explicit BlockImpl(Engine* e) : eng(e) {}
  virtual ~BlockImpl() = default;
  virtual size_t stage_params(int sid) const = 0;
  virtual size_t embed_params() const = 0;
  virtual size_t deembed_params() const = 0;
  // Fills master weights on the device (init_model streams, model.cpp:159-197).
  virtual void init_stage(int sid, uint64_t seed, void* w) = 0;
  virtual void init_edges(uint64_t seed, void* embed, void* deembed) = 0;
  // Forward of microbatch slot `mb` along `order`: embedding, the owned
  // stages' layers, and on the de-embedding owner the head: loss into
  // *loss_dev (device double) and, when train, the head backward leaving
  // dL/dh_final in the slot.  Activations are cached per (slot, applied layer).
  virtual void mb_forward(int mb, const int* order, const void* x, const void* y, size_t rows, bool train,
                          double* loss_dev) = 0;
  // Backward of slot `mb`: owned layers in reverse applied order (gradients
  // accumulate into the groups' g buffers), then the embedding.
  virtual void mb_backward(int mb, const int* order, const void* x, size_t rows) = 0;
  // the reference's per-microbatch order: forward then backward (model.cpp:211-378);
  // k = the microbatch's position in the iteration (activation slot 0 is reused)
  void microbatch(int k, const int* order, const void* x, const void* y, size_t rows, bool train, double* loss_dev) {
    wk = k;
    mb_forward(0, order, x, y, rows, train, loss_dev);
    if (train) mb_backward(0, order, x, rows);
  }
  // An iteration of m microbatches of `rows` each begins / its backward phase is
  // over: blocks that defer work to the end of the backward phase (the LLaMA
  // block's weight-gradient GEMMs) flush it here, before DP all-reduce and Adam.
  virtual void begin_iteration(int m, size_t rows) {
    (void)m;
    (void)rows;
  }
  virtual void flush_grads() {}
  // Device bytes one token of a fused microbatch group keeps live from its
  // forward to its backward (activation cache over every resident layer, head
  // logits, scratch).  0 = the block does not fuse microbatches.
  virtual size_t group_bytes_per_token() const { return 0; }
  // device bytes the block will still allocate this iteration (e.g. deferred-gradient inputs)
  virtual size_t reserved_bytes() const { return 0; }
  // redundant-computation baseline: one extra forward of every stage's layers for this microbatch
  virtual void redundant_forward(const int* order, const void* x, size_t rows) {
    (void)order;
    (void)x;
    (void)rows;
    raise(1, "redundant computation is implemented for the LLaMA bf16 block");
  }
  // block state that changes the launch sequence of an iteration (part of the CUDA-graph key)
  virtual long state_token() const { return 0; }
  // ---- plan-driven execution (schedule 2, 1F1B): the engine walks the global op order of
  // host::pipeline_plan and hands this rank's ops to the block one at a time; transfers are the
  // engine's (send / recv streams).  Microbatch k keeps its own residual-stream and gradient
  // buffers for the whole iteration; activation caches rotate over `slots` microbatches (the
  // plan keeps at most that many in flight per rank).
  virtual bool supports_plan() const { return false; }
  virtual void plan_begin(int m, size_t rows, int slots, const void* x) {
    (void)m;
    (void)rows;
    (void)slots;
    (void)x;
  }
  // kind: host::PlanOp kind (embed fwd, stage fwd, head, stage bwd, embed bwd); sid for stage ops
  virtual void plan_op(int kind, int k, int sid, const int* order, double* loss_dev) {
    (void)kind;
    (void)k;
    (void)sid;
    (void)order;
    (void)loss_dev;
  }
  // the buffer a transfer of microbatch k carries (phase 0: residual stream h, 1: its gradient dh)
  virtual void* plan_buffer(int k, int phase, size_t* bytes) {
    (void)k;
    (void)phase;
    *bytes = 0;
    return nullptr;
  }
  // a transfer of microbatch k landed on this rank (compute-stream ordered)
  virtual void plan_received(int k, int phase) {
    (void)k;
    (void)phase;
  }
  int wk = 0;  // position of the current microbatch within the iteration (in microbatches)
  // Rows of ONE microbatch when a call carries a fused group of several (the
  // loss and its gradient stay per-microbatch means, pipeline.cpp:66-83); 0 = rows.
  size_t loss_rows = 0;
  // Predictions of forward(order, x) (MLP) into a device buffer of rows*out.
  virtual void predict(const int* order, const void* x, size_t rows, void* pred) = 0;
  Engine* eng;
};

class Engine {
 public:
  explicit Engine(const ckf_model_desc& d);
  ~Engine();

  const Desc& desc() const { return d_; }
  bool fp64() const { return d_.prec == CKF_FP64; }
  size_t master_bytes() const { return fp64() ? 8 : 4; }
  cudaStream_t stream() const { return st_; }
  ReduceScratch& scratch() { return red_; }

  void init(uint64_t seed, double lr);
  void run_iteration(const int* orders, int m, const void* x, const void* y, size_t rows, bool on_device,
                     long iteration, double* loss, double* omegas);
  double eval_loss(const int* order, const void* x, const void* y, size_t rows, bool on_device);
  // one microbatch forward + backward accumulating into the gradient buffers (no Adam)
  double accumulate(const int* order, const void* x, const void* y, size_t rows, bool on_device);
  void zero_grad();
  void export_grad(ParamGroup& g, double* out);
  void predict(const int* order, const double* x_host, size_t rows, double* pred_host);
  // device-side variants used by the trainer's data path
  void predict_device(const int* order, const void* x_dev, size_t rows, void* pred_dev);

  void refresh_edge_replicas();
  // Checkpointing baseline (recovery.hpp:88-108, checkpoint.cpp:70-83): a deep copy of every
  // owned group's weights, Adam moments, bf16 shadow and scalars kept in HBM (device-to-device,
  // no host round trip).  restore returns the snapshot's model iteration; *red (optional, per
  // stage id 1..s) receives ||W_now - W_snapshot||^2 for the listed stages before the rollback.
  void checkpoint_save(long iteration);
  long checkpoint_restore(const int* stages, int n_stages, double* red, float* ms);
  bool has_checkpoint() const { return ckpt_valid_; }
  void kill_stage(int sid);
  ckf_recovery_report recover_stage(int sid, int mode, int moments, double lr_bump, uint64_t reinit_seed,
                                    bool want_reduction_error);

  void export_group(ParamGroup& g, double* w, double* m, double* v);
  void import_group(ParamGroup& g, const double* w, const double* m, const double* v);

  ParamGroup& stage(int sid) { return stages_.at(static_cast<size_t>(sid - 1)); }
  ParamGroup& embed() { return embed_; }
  ParamGroup& deembed() { return deembed_; }
  double edge_lr = 3e-4;

  // placement (multi-GPU): rank owning each stage; edges follow stages 1 and s
  int rank() const { return rank_; }
  int owner_of_stage(int sid) const { return stage_rank_.empty() ? 0 : stage_rank_[static_cast<size_t>(sid - 1)]; }
  int owner_of_embed() const { return owner_of_stage(1); }
  int owner_of_deembed() const { return owner_of_stage(static_cast<int>(d_.s)); }
  bool mine(int owner) const { return owner == rank_; }
  // nranks = replicas x P pipeline ranks; rank r is pipeline rank r % P of replica r / P;
  // stage_rank[s-1] names the pipeline rank (0..P-1) holding stage s in every replica
  void attach_comm(const void* uid, int nranks, int rank, const int* stage_rank, int replicas = 1);
  // placement without a communicator (attach_comm = this + NCCL init)
  void set_placement(int nranks, int rank, const int* stage_rank, int replicas = 1);
  // peer recovery: CUDA IPC handles of the owned stages' w / m / v; import maps the other
  // ranks' stages (same replica) so recover_stage reads neighbours straight from peer HBM
  size_t ipc_export(void* buf, size_t cap);
  void ipc_import(const void* buf, size_t len);
  // collective: all-gathers every rank's IPC blob over NCCL and imports them
  void exchange_peers();
  // Peer-memory stage transport for the plan-driven pipeline: a mailbox of 2 x max_m microbatch
  // buffers (residual stream / its gradient, max_rows x d fp32 each) and 2 x max_m flags, both
  // exported with the IPC blob; transfers then copy straight into the receiver's mailbox (peer
  // HBM) and signal its flag instead of going through NCCL.  Enable on every rank BEFORE the
  // IPC exchange.
  void enable_peer_transport(int max_m);
  bool peer_transport() const { return mbox_ != nullptr; }
  // this rank's mailbox slot of microbatch k (phase 0: h, 1: dh); null without the transport
  void* mailbox(int k, int phase) const;
  // costs the 1F1B plan is simulated with: forward time units per stage (its layer count) and the
  // head (LM head + loss + head backward) relative to one layer's forward FLOPs
  host::PlanCost plan_cost() const;
  // collective helpers over the world communicator (host doubles, summed)
  std::vector<double> allreduce_host(const std::vector<double>& v);
  double share_from_head(double v);
  int replicas() const { return replicas_; }
  int replica() const { return replica_; }
  std::vector<ParamGroup*> owned_groups();
  // 0 = sequential (forward+backward per microbatch, one live activation cache);
  // 1 = GPipe (all forwards, then all backwards in microbatch order: the ranks of
  //     a multi-GPU pipeline overlap; per-stage accumulation order is unchanged)
  // 2 = 1F1B (plan-driven, host::pipeline_plan): per rank at most P microbatches in flight,
  //     transfers on dedicated send / recv streams with one NCCL communicator per directed
  //     link, overlapped with compute; per-stage accumulation still in microbatch order
  void set_schedule(int mode) {
    if (mode < 0 || mode > 2) raise(1, "schedule must be 0 (sequential), 1 (gpipe) or 2 (1f1b)");
    schedule_ = mode;
  }
  int schedule() const { return schedule_; }
  // Microbatch fusion when every stage is resident on this rank (no stage hops):
  // microbatches that share an execution order run as ONE forward + backward of
  // up to group_cap microbatches (0 = as many as HBM allows, 1 = off).
  void set_group_cap(int cap) { group_cap_ = cap < 0 ? 0 : cap; }
  void set_graphs(bool on) { graphs_ = on; }
  // Redundant-computation baseline, measured: every stage's forward runs a second time per
  // microbatch (the downstream node's hot copy) and every stage's master weights are copied to
  // its replica after the optimizer step (the post-step weight refresh of cost_model.cpp:271-279).
  void set_redundant(bool on) { redundant_ = on; }
  // CheckFree+: refresh the edge replicas at the end of every run_iteration (trainer.cpp:83-84)
  void set_edge_replicas(bool on) { auto_replicas_ = on; }
  // device time (ms) of the last run_iteration: first device op .. loss / omega D2H
  float last_step_ms();
  int group_cap() const { return group_cap_; }
  // move `bytes` of `buf` from rank src to rank dst (NCCL send/recv on the engine stream)
  void hop(void* buf, size_t bytes, int src, int dst);
  // Stage-boundary transfer between pipeline positions (codes: 0 = embedding,
  // 1..s = stage, s+1 = de-embedding).  Returns true on the rank that received
  // data from another rank.  Logged against the virtual placement when enabled.
  bool move(void* buf, size_t bytes, int from_code, int to_code);
  int owner_of_code(int code) const {
    return code <= 0 ? owner_of_embed() : code > static_cast<int>(d_.s) ? owner_of_deembed() : owner_of_stage(code);
  }
  // hop log (multi-GPU placement check on one GPU): records (src, dst, bytes) of every
  // transfer the virtual placement `vrank` (stage -> rank) would perform
  void hop_log_enable(int nranks, const int* vrank);
  const std::vector<long>& hop_log() const { return hop_log_; }

  // kernel timing (KClass)
  void kt_enable(bool on);
  bool kt_on() const { return kt_on_; }
  void kt_begin();
  void kt_end(int cls, double flops, double bytes);
  void kt_collect();  // stream must be synchronised
  const KStat& kt_stat(int cls) const { return kstat_[cls]; }

  // device workspace (grows on demand, reused across calls)
  void* ws(size_t bytes, int slot);
  double* dev_scalars() { return scal_; }  // small device double array (losses, omegas)

 private:
  void alloc_group(ParamGroup& g, size_t n, bool lowp);
  void free_group(ParamGroup& g);
  void adam_group(ParamGroup& g, double lr, double gscale, double* omega_dev);
  // uploads host inputs (fp64 rows / int32 tokens) into device buffers; returns device x, y
  void upload(const void* x, const void* y, size_t rows, const void** xd, const void** yd);

  Desc d_;
  cudaStream_t st_ = nullptr;
  ReduceScratch red_;
  std::vector<ParamGroup> stages_;
  ParamGroup embed_, deembed_;
  void* rep_embed_ = nullptr;   // CheckFree+ replica of E held by stage 2's GPU
  void* rep_deembed_ = nullptr; // replica of E^-1 held by stage s-1's GPU
  long replica_staleness_ = -1; // recovery.hpp:57-61
  std::unique_ptr<BlockImpl> impl_;
  std::vector<void*> ws_;
  std::vector<size_t> ws_size_;
  double* scal_ = nullptr;
  int rank_ = 0, nranks_ = 1;
  int schedule_ = 0;
  int group_cap_ = 0;
  // CUDA graph of the fused (all stages resident) step: key = shape, inputs, orders, alloc epoch
  bool graphs_ = true;
  cudaGraphExec_t gexec_ = nullptr;
  std::vector<long> gkey_, gseen_;
  long graph_kernels_ = 0;  // kernel launches inside the captured graph
  bool redundant_ = false;
  bool auto_replicas_ = false;
  std::vector<void*> rc_replica_;  // per stage: the hot copy's master weights
  std::vector<std::pair<size_t, int>> group_fit_;  // (microbatch tokens, fitted group size)
  int fused_group_size(int m, size_t mb_rows);
  int replicas_ = 1, replica_ = 0;
  void* dp_comm_ = nullptr;  // ncclComm_t over the same pipeline rank of every replica
  bool log_hops_ = false;
  std::vector<int> vrank_;
  std::vector<long> hop_log_;
  std::vector<int> stage_rank_;
  // plan-driven (1F1B) executor: side streams, per-link communicators, event pool
  void run_plan(const int* orders, int m, const char* x, size_t mb, size_t xrow);
  void* link_comm(int src, int dst);
  void ensure_links();
  bool links_ready_ = false;
  cudaEvent_t plan_event();
  cudaStream_t sst_ = nullptr, rst_ = nullptr, dst_ = nullptr;  // send, recv, data-parallel streams
  std::vector<std::pair<std::pair<int, int>, void*>> links_;    // (src, dst) -> ncclComm_t
  std::vector<cudaEvent_t> pev_;
  size_t pev_used_ = 0;
 public:
  // data-parallel gradient bucket ready (block calls it as each layer's weight gradients finish):
  // the all-reduce of the replicas' sums runs on the data-parallel stream, overlapped with the
  // remaining weight-gradient GEMMs
  void grad_bucket_ready(void* g, size_t n);
 private:
  bool dp_pending_ = false;
  struct PeerStage {
    void *w = nullptr, *m = nullptr, *v = nullptr;
  };
  std::vector<PeerStage> peer_;
  // peer transport: own mailbox / flags, and every other rank's (IPC-mapped), by global rank
  void* mbox_ = nullptr;
  uint64_t* flags_ = nullptr;
  int mbox_m_ = 0;
  size_t mbox_slot_ = 0;  // bytes per microbatch buffer
  std::vector<void*> peer_mbox_;
  std::vector<uint64_t*> peer_flags_;
  uint64_t plan_epoch_ = 0;
  bool peer_ready_ = false;  // every stage this rank does not own is mapped  // per stage id - 1: IPC mappings of stages owned by other ranks
  void* comm_ = nullptr;  // ncclComm_t
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  cudaEvent_t sb_ev_ = nullptr, se_ev_ = nullptr;  // run_iteration device-timeline bracket
  cudaEvent_t sg_ev_ = nullptr;  // CKF_STEP_DEBUG: just before the fused step's graph / body
  struct CkptGroup {
    void* buf = nullptr;  // [w | m | v] master dtype, then the bf16 shadow
    size_t bytes = 0;
    long step = 0;
    double omega = 0.0, lr = 0.0;
  };
  std::vector<CkptGroup> ckpt_;  // stages 1..s, then embed, deembed
  double ckpt_edge_lr_ = 0.0;
  long ckpt_iter_ = 0;
  bool ckpt_valid_ = false;
  bool kt_on_ = false;
  std::vector<cudaEvent_t> kev_;
  size_t kev_used_ = 0;
  struct KRec {
    int cls;
    double flops, bytes;
  };
  std::vector<KRec> krec_;
  KStat kstat_[KC_N];
  friend struct MlpBlock;
  friend struct LlamaBlock;
};

std::unique_ptr<BlockImpl> make_mlp_block(Engine* e);
std::unique_ptr<BlockImpl> make_llama_block(Engine* e);
std::unique_ptr<BlockImpl> make_llama_f32_block(Engine* e);  // fp32 parity mode (llama_f32.cu)

std::vector<Range> even_partition(size_t layers, size_t stages);

// The failure-injected trainer (trainer.cu).  cm (optional): this process's place in a
// multi-GPU run -- NCCL unique id, world size, rank, data-parallel replicas.
struct TrainerComm {
  const void* uid = nullptr;
  int nranks = 1, rank = 0, replicas = 1;
};
std::string run_experiment(const std::string& kv, const std::string& trace_text, uint64_t seed,
                           const std::string& dir, const TrainerComm* cm = nullptr);

}  // namespace ckf
