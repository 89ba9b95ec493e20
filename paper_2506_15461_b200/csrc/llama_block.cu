// LLaMA-style stage block on the bf16 throughput path:
//   h  = E[tok]                                           (embedding, edge group 0)
//   per layer:  h += Wo  . attn(rope(RMSNorm(h; g1) Wqkv))
//               h += Wd  . swiglu(RMSNorm(h; g2) Wgu)
//   logits = RMSNorm(h; gF) E_inv ; loss = mean CE        (de-embedding, edge group 1)
// Stage GEMMs run on the tcgen05 kernel (gemm_tc.cu), attention on the flash
// kernels (attention.cu), everything else on llama_kernels.cu.  The residual
// stream, gradients, norms and Adam master weights are fp32; GEMM operands
// and cached activations are bf16.
//
// It follows the reference's structure exactly where one exists
// (/root/reference/proj/src/model.cpp:211-378): stages applied in the
// microbatch's execution order with a per-applied-block activation cache,
// gradients accumulated straight into the stage accumulators (GEMM epilogue
// += instead of Gradients::accumulate, model.cpp:299-305), canonical flat
// stage layout = blocks in order (model.cpp:117-125).  Per-layer flat layout:
//   [g1 (d) | Wqkv (d x 3d) | Wo (d x d) | g2 (d) | Wgu (d x 2f) | Wd (f x d)]
// edge groups: E [V x d];  [gF (d) | E_inv (d x V)].  Weights row-major
// [fan_in x fan_out] like the reference (model.cpp:27-33).
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "engine.h"
#include "gemm_tc.h"
#include "llama_kernels.h"

namespace ckf {

using llama::bf16;

namespace {

struct Off {
  size_t g1, wqkv, wo, g2, wgu, wd, total;
};
Off layer_offsets(size_t d, size_t f) {
  Off o;
  o.g1 = 0;
  o.wqkv = d;
  o.wo = o.wqkv + 3 * d * d;
  o.g2 = o.wo + d * d;
  o.wgu = o.g2 + d;
  o.wd = o.wgu + 2 * d * f;
  o.total = o.wd + f * d;
  return o;
}

}  // namespace

struct LlamaBlock final : BlockImpl {
  explicit LlamaBlock(Engine* e) : BlockImpl(e) {
    const Desc& D = eng->desc();
    d = D.d;
    f = D.hid;
    V = D.out;
    H = D.heads;
    T = D.T;
    hd = d / H;
    off = layer_offsets(d, f);
    if (D.in != D.out) raise(1, "LLaMA block: input_dim and output_dim are both the vocabulary size");
    if (d % 128 || d > 4096) raise(1, "LLaMA block: model_dim must be a multiple of 128 (<= 4096)");
    if (d % H || (hd != 64 && hd != 128)) raise(1, "LLaMA block: head_dim = model_dim / n_heads must be 64 or 128");
    if (T % 64) raise(1, "LLaMA block: seq_len must be a multiple of 64");
    if (f % 64) raise(1, "LLaMA block: ffn width must be a multiple of 64");
    if (V % 8) raise(1, "LLaMA block: vocabulary size must be a multiple of 8");
    if (D.prec != CKF_BF16)
      raise(1, "LLaMA block runs on the bf16 tensor-core path (the fp32/fp64 parity precisions use the residual-MLP "
               "block)");
  }

  size_t d, f, V, H, T, hd;
  Off off;

  size_t stage_params(int sid) const override {
    return eng->desc().part[static_cast<size_t>(sid - 1)].count() * off.total;
  }
  size_t embed_params() const override { return V * d; }
  size_t deembed_params() const override { return d + d * V; }

  void sample(float* w, size_t n, size_t fan_in, size_t fan_out, uint64_t key) {
    const double a = std::sqrt(6.0 / static_cast<double>(fan_in + fan_out));  // model.cpp:27-33
    k::uniform(w, n, key, -a, a, 0, eng->stream());
  }

  // init streams: the reference's tag scheme (model.cpp:24-25) extended per matrix:
  //   Wqkv(l) = derive_key(seed, 2l, 1), Wo(l) = (2l, 2), Wgu(l) = (2l+1, 1), Wd(l) = (2l+1, 2);
  //   E = derive_key(seed, 0), E_inv = derive_key(seed, 1); RMSNorm gains = 1.
  void init_stage(int sid, uint64_t seed, void* wv) override {
    float* w = static_cast<float*>(wv);
    const Range& r = eng->desc().part[static_cast<size_t>(sid - 1)];
    cudaStream_t st = eng->stream();
    for (size_t l = r.first; l <= r.last; ++l) {
      float* b = w + (l - r.first) * off.total;
      k::fill(b + off.g1, 1.0, d, st);
      sample(b + off.wqkv, 3 * d * d, d, 3 * d, derive_key(seed, 2 * l, 1));
      sample(b + off.wo, d * d, d, d, derive_key(seed, 2 * l, 2));
      k::fill(b + off.g2, 1.0, d, st);
      sample(b + off.wgu, 2 * d * f, d, 2 * f, derive_key(seed, 2 * l + 1, 1));
      sample(b + off.wd, f * d, f, d, derive_key(seed, 2 * l + 1, 2));
    }
  }
  void init_edges(uint64_t seed, void* e, void* de) override {
    if (e) sample(static_cast<float*>(e), V * d, V, d, derive_key(seed, 0));
    if (de) {
      k::fill(static_cast<float*>(de), 1.0, d, eng->stream());
      sample(static_cast<float*>(de) + d, d * V, d, V, derive_key(seed, 1));
    }
  }

  // ------------------------------------------------------------ workspace
  template <typename T_>
  T_* buf(int slot, size_t elems) {
    return static_cast<T_*>(eng->ws(elems * sizeof(T_), slot));
  }
  struct Cache {
    float *h_in, *rstd1, *lse, *h_mid, *rstd2;
    bf16 *xn1, *qkv, *o, *xn2, *gu, *a;
  };
  static size_t al(size_t b) { return (b + 255) / 256 * 256; }
  // with_x = false: the layer inputs X (xn1, o, xn2, a) live in the deferred
  // weight-gradient buffers instead (WSet below)
  Cache cache(size_t slot, size_t Mt, size_t rows, bool with_x) {
    const size_t xb = with_x ? al(Mt * d * 2) * 3 + al(Mt * f * 2) : 0;
    const size_t bytes = al(Mt * d * 4) * 2 + al(Mt * 4) * 2 + al(rows * H * T * 4) + al(Mt * 3 * d * 2) +
                         al(Mt * 2 * f * 2) + xb;
    char* p = static_cast<char*>(eng->ws(bytes, 100 + static_cast<int>(slot)));  // slot = cache_id - 100
    Cache c{};
    auto take = [&](size_t b) {
      char* r = p;
      p += al(b);
      return r;
    };
    c.h_in = reinterpret_cast<float*>(take(Mt * d * 4));
    c.h_mid = reinterpret_cast<float*>(take(Mt * d * 4));
    c.rstd1 = reinterpret_cast<float*>(take(Mt * 4));
    c.rstd2 = reinterpret_cast<float*>(take(Mt * 4));
    c.lse = reinterpret_cast<float*>(take(rows * H * T * 4));
    c.qkv = reinterpret_cast<bf16*>(take(Mt * 3 * d * 2));
    c.gu = reinterpret_cast<bf16*>(take(Mt * 2 * f * 2));
    if (with_x) {
      c.xn1 = reinterpret_cast<bf16*>(take(Mt * d * 2));
      c.o = reinterpret_cast<bf16*>(take(Mt * d * 2));
      c.xn2 = reinterpret_cast<bf16*>(take(Mt * d * 2));
      c.a = reinterpret_cast<bf16*>(take(Mt * f * 2));
    }
    return c;
  }

  // ------------------------------------------------------------ deferred weight gradients
  // A layer's four weight gradients (gW += X^T dY for Wqkv, Wo, Wgu, Wd) feed
  // nothing inside the iteration but Adam, so they are deferred to the end of
  // the backward phase and computed ONCE over all m microbatches (GEMM depth
  // K = m * Mt tokens instead of m GEMMs of depth Mt): with M = d small, a
  // per-microbatch wgrad has too few output tiles for 148 SMs and pays a
  // split-K reduction; the batched one fills the machine.  This is the
  // "W pass" of zero-bubble pipeline schedules, and in a multi-GPU pipeline it
  // runs in the drain bubble.  The layer inputs X and output gradients dY are
  // written by the forward / backward straight into per-layer buffers
  // [m * Mt x width] (microbatch k at rows k * Mt), so deferral costs no copies.
  // Numerics: one fp32 GEMM over all tokens replaces the reference's
  // per-microbatch Gradients::accumulate (model.cpp:299-305) -- a different
  // fp32 association, still deterministic.  CKF_WGRAD_DEFER=0, or too little
  // free HBM, selects the per-microbatch form.
  struct WSet {
    bf16 *xn1, *o, *xn2, *a;        // X: inputs of Wqkv, Wo, Wgu, Wd
    bf16 *dqkv, *dho, *dgu, *dhd;   // dY: output gradients of Wqkv, Wo, Wgu, Wd
  };
  static constexpr int kWSlot = 300000;
  bool defer_ = false;
  int defer_m_ = 1;
  size_t defer_Mt_ = 0;
  std::vector<std::pair<int, size_t>> pending_;
  size_t wrow_elems() const { return 8 * d + 3 * f; }  // X (3d + f) + dY (5d + 2f) bf16 per token
  WSet wset(int sid, size_t li, int k) {
    const size_t R = static_cast<size_t>(defer_m_) * defer_Mt_, o = static_cast<size_t>(k) * defer_Mt_;
    bf16* p = static_cast<bf16*>(eng->ws(R * wrow_elems() * 2, kWSlot + 1024 * (sid - 1) + static_cast<int>(li)));
    WSet w;
    size_t at = 0;
    auto take = [&](size_t width) {
      bf16* r = p + at * R + o * width;
      at += width;
      return r;
    };
    w.xn1 = take(d);
    w.o = take(d);
    w.xn2 = take(d);
    w.a = take(f);
    w.dqkv = take(3 * d);
    w.dho = take(d);
    w.dgu = take(2 * f);
    w.dhd = take(d);
    return w;
  }
  // per-microbatch form: X in the activation cache, dY in scratch
  WSet wset_local(const Cache& c, bf16* dh_bf, size_t Mt) {
    WSet w{c.xn1, c.o, c.xn2, c.a, nullptr, dh_bf, nullptr, dh_bf};
    w.dgu = buf<bf16>(47, Mt * 2 * f);
    w.dqkv = 3 * d <= 2 * f ? w.dgu : static_cast<bf16*>(eng->ws(Mt * 3 * d * 2, 56));  // dgu is dead by then
    return w;
  }

  void begin_iteration(int m, size_t rows) override {
    pending_.clear();
    const char* env = std::getenv("CKF_WGRAD_DEFER");
    bool want = !(env && env[0] == '0') && m > 1;
    const size_t Mt = rows * T;
    // the deferred buffers of this (m, Mt) already exist: nothing to size (and no
    // cudaMemGetInfo, which can stall the launching thread for tens of ms on some hosts)
    const bool allocated = want && defer_ && defer_m_ == m && defer_Mt_ == Mt;
    if (want && !allocated) {
      size_t layers = 0;
      const Desc& D = eng->desc();
      for (size_t i = 0; i < D.s; ++i)
        if (eng->mine(eng->owner_of_stage(static_cast<int>(i + 1)))) layers += D.part[i].count();
      const size_t need = layers * static_cast<size_t>(m) * Mt * wrow_elems() * 2;
      size_t fr = 0, tot = 0;
      CKF_CUDA(cudaMemGetInfo(&fr, &tot));
      const size_t have = (defer_m_ == m && defer_Mt_ == Mt && defer_) ? need : 0;  // already allocated
      want = need <= have + fr / 2;
    }
    reserve_ = 0;
    if (want) {
      size_t layers = 0;
      const Desc& D = eng->desc();
      for (size_t i = 0; i < D.s; ++i)
        if (eng->mine(eng->owner_of_stage(static_cast<int>(i + 1)))) layers += D.part[i].count();
      const bool have = defer_m_ == m && defer_Mt_ == Mt && defer_;
      reserve_ = have ? 0 : layers * static_cast<size_t>(m) * Mt * wrow_elems() * 2;
    }
    defer_ = want;
    defer_m_ = want ? m : 1;
    defer_Mt_ = Mt;
  }
  size_t reserve_ = 0;
  size_t reserved_bytes() const override { return reserve_; }
  long state_token() const override { return (defer_ ? 1 : 0) | (fuse_swiglu() ? 2 : 0); }
  // per token of a fused group: the activation cache of every resident layer
  // (cache(): h_in, h_mid, rstd1/2, lse, qkv, gu; the X inputs live in the
  // deferred buffers), bf16 logits, and the per-call fp32 / bf16 scratch
  size_t group_bytes_per_token() const override {
    size_t layers = 0;
    const Desc& D = eng->desc();
    for (size_t i = 0; i < D.s; ++i)
      if (eng->mine(eng->owner_of_stage(static_cast<int>(i + 1)))) layers += D.part[i].count();
    const size_t per_layer = 8 * d + 8 + 4 * H + 6 * d + 4 * f + 8 * d + 4 * f;  // + X when not deferred
    // head: Q (2 V) + the fused loss's partial sums and row scalars + xs (head_xent_workspace)
    const size_t head = 2 * V + 4 * std::max<size_t>(tc::xent_partials(static_cast<int>(V)), 256) + 24 + 2 * d;
    return layers * per_layer + head + 8 + 26 * d + 2 * std::max(d, f) + 4 * H + 64;
  }

  void flush_grads() override {
    if (!defer_ || pending_.empty()) return;
    std::sort(pending_.begin(), pending_.end());
    const int R = static_cast<int>(static_cast<size_t>(defer_m_) * defer_Mt_);
    const int di = static_cast<int>(d), fi = static_cast<int>(f);
    for (const auto& [sid, li] : pending_) {
      const WSet w = wset(sid, li, 0);
      float* G = gf(sid, li);
      gemm(di, 3 * di, R, w.xn1, di, true, w.dqkv, 3 * di, true, G + off.wqkv, 3 * di, tc::kAccF32);
      gemm(di, di, R, w.o, di, true, w.dho, di, true, G + off.wo, di, tc::kAccF32);
      gemm(di, 2 * fi, R, w.xn2, di, true, w.dgu, 2 * fi, true, G + off.wgu, 2 * fi, tc::kAccF32);
      gemm(fi, di, R, w.a, fi, true, w.dhd, di, true, G + off.wd, di, tc::kAccF32);
      eng->grad_bucket_ready(G, off.total);  // data parallel: this layer's all-reduce overlaps the next wgrads
    }
    pending_.clear();
  }

  // ------------------------------------------------------------ timed launch helpers
  void gemm(int M, int N, int K, const bf16* A, int lda, bool a_mn, const bf16* B, int ldb, bool b_mn, void* C,
            int ldc, int epi, const float2* rope_tab = nullptr, int rope_cols = 0, void* aux = nullptr,
            int ldaux = 0) {
    tc::GemmDesc g;
    g.aux = aux;
    g.ldaux = ldaux;
    g.rope_tab = rope_tab;
    g.rope_T = static_cast<int>(T);
    g.rope_cols = rope_cols;
    g.rope_hd = static_cast<int>(hd);
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.a_mn = a_mn;
    g.B = B;
    g.ldb = ldb;
    g.b_mn = b_mn;
    g.C = C;
    g.ldc = ldc;
    g.epi = epi;
    gemm_desc(g);
  }
  void gemm_desc(const tc::GemmDesc& g) {
    eng->kt_begin();
    tc::gemm_bf16(g, eng->stream());
    // bytes of C per output element: bf16 store; fp32 store; fp32 read+write; SwiGLU fwd
    // (g, u stored + a: 3 bf16 per gate/up pair = 3 B per output); SwiGLU bwd (g, u read, dg, du written)
    const int epi = g.epi;
    const double M = g.M, N = g.N, K = g.K;
    const double cb = epi == tc::kStoreBF16 || epi == tc::kXentFwd ? 2.0 : epi == tc::kStoreF32 ? 4.0
                    : epi == tc::kAccF32 ? 8.0 : epi == tc::kSwiGLU ? 3.0 : 8.0;
    eng->kt_end(KC_GEMM, 2.0 * M * N * K, 2.0 * (M * K + K * N) + cb * M * N);
  }

  // LM head + mean token cross-entropy, and (train) the head backward into gE_inv and dxn
  // (model.cpp:250-253, 322-342; kernels_serial.cpp:163-185).  Fused (head_xent.cu: no logits
  // tensor, no pass over [tokens x V] outside the GEMMs) unless CKF_HEAD_FUSED=0 selects the
  // bf16-logits path (logits GEMM -> xent_bf16 in place -> GEMMs on the bf16 gradient).
  static bool head_fused() {
    static const bool v = [] {
      const char* e = std::getenv("CKF_HEAD_FUSED");
      return !(e && e[0] == '0');
    }();
    return v;
  }
  void head(const bf16* xnF, const float* hF, const float* rstdF, const float* gF, const bf16* Einv, const int* lab,
            size_t Mt, size_t Mmb, bool train, double* row_loss, double* loss_dev, float* dxn, float* gde) {
    cudaStream_t st = eng->stream();
    const int Mi = static_cast<int>(Mt), di = static_cast<int>(d), Vi = static_cast<int>(V);
    const float gs = static_cast<float>(1.0 / static_cast<double>(Mmb));
    if (head_fused()) {
      llama::HeadXent hx;
      hx.xn = xnF;
      hx.Einv = Einv;
      hx.labels = lab;
      hx.M = Mi;
      hx.d = di;
      hx.V = Vi;
      hx.grad_scale = gs;
      hx.train = train;
      hx.row_loss = row_loss;
      hx.dxn = dxn;
      hx.gEinv = gde + d;
      hx.ws = eng->ws(llama::head_xent_workspace(Mt, d, V), 53);
      hx.h = hF;
      hx.rstd = rstdF;
      hx.gain = gF;
      const double P = tc::xent_partials(Vi);
      llama::head_xent(
          hx, [&](const tc::GemmDesc& g) { gemm_desc(g); },
          [&](const std::function<void()>& f) { timed(KC_LOSS, 0.0, Mt * (P * 4.0 + 4.0 * d + 24.0), f); }, st);
      timed(KC_LOSS, 0.0, Mt * 8.0, [&] { llama::fold_mean(row_loss, Mt, 1.0 / static_cast<double>(Mmb), loss_dev, st); });
      return;
    }
    bf16* logits = buf<bf16>(53, Mt * V);
    gemm(Mi, Vi, di, xnF, di, false, Einv, Vi, true, logits, Vi, tc::kStoreBF16);
    timed(KC_LOSS, 0.0, Mt * V * (train ? 6.0 : 2.0), [&] {
      llama::xent_bf16(logits, lab, Mt, V, gs, train ? 1 : 0, row_loss, st);
      llama::fold_mean(row_loss, Mt, 1.0 / static_cast<double>(Mmb), loss_dev, st);  // sum of microbatch means
    });
    if (!train) return;
    gemm(di, Vi, Mi, xnF, di, true, logits, Vi, true, gde + d, Vi, tc::kAccF32);
    gemm(Mi, di, Vi, logits, Vi, false, Einv, Vi, false, dxn, di, tc::kStoreF32);
  }
  template <typename F>
  void timed(int cls, double flops, double bytes, F&& f) {
    eng->kt_begin();
    f();
    eng->kt_end(cls, flops, bytes);
  }

  // ------------------------------------------------------------ one microbatch
  // Per-slot state (kept from mb_forward to mb_backward): tokens, labels, the
  // gradient of the final residual stream, and one cache slab per applied layer.
  static int slot_id(int mb, int k) { return 1000 + 8 * mb + k; }
  static int cache_id(int mb, size_t applied) { return 100000 + 64 * mb + static_cast<int>(applied); }
  struct Applied {
    int sid;
    size_t li;  // layer index within the stage
  };
  std::vector<Applied> applied_order(const int* order) const {
    std::vector<Applied> v;
    const Desc& D = eng->desc();
    for (size_t oi = 0; oi < D.s; ++oi) {
      const Range& r = D.part[static_cast<size_t>(order[oi] - 1)];
      for (size_t li = 0; li < r.count(); ++li) v.push_back({order[oi], li});
    }
    return v;
  }
  Cache cache_for(int mb, size_t applied, size_t Mt, size_t rows, bool with_x) {
    return cache(static_cast<size_t>(cache_id(mb, applied)) - 100, Mt, rows, with_x);
  }

  void mb_forward(int mb, const int* order, const void* xv, const void*, size_t rows, bool train,
                  double* loss_dev) override {
    const Desc& D = eng->desc();
    cudaStream_t st = eng->stream();
    const size_t Mt = rows * T;
    const size_t Mmb = loss_rows ? loss_rows * T : Mt;  // tokens of ONE microbatch (fused groups carry several)
    if (Mmb > D.max_rows) raise(1, "microbatch tokens exceed the engine's max_rows (tokens per microbatch)");
    const int* x = static_cast<const int*>(xv);

    int* tok = buf<int>(slot_id(mb, 0), Mt);
    int* lab = buf<int>(slot_id(mb, 1), Mt);
    float* dh = buf<float>(slot_id(mb, 2), Mt * d);
    bf16* dh_bf = buf<bf16>(slot_id(mb, 3), Mt * d);
    float* h = buf<float>(42, Mt * d);
    float* dxn = buf<float>(45, Mt * d);
    const int nblk = llama::rmsnorm_bwd_blocks(Mt);
    float* gpart = buf<float>(49, static_cast<size_t>(nblk) * d);
    bf16* xnF = buf<bf16>(50, Mt * d);
    float* rstdF = buf<float>(51, Mt);
    float* hF = buf<float>(52, Mt * d);
    double* row_loss = buf<double>(54, Mt);

    llama::split_tokens(x, rows, T, tok, lab, st);

    // ---------------- forward (model.cpp:226-253)
    int at = 0;  // pipeline position of h (0 = embedding)
    if (eng->mine(eng->owner_of_embed()))
      timed(KC_NORM, 0.0, Mt * d * 8.0, [&] {
        llama::embed_fwd(tok, Mt, static_cast<const float*>(eng->embed().w), d, h, st);
      });
    size_t slot = 0;
    for (size_t oi = 0; oi < D.s; ++oi) {
      const int sid = order[oi];
      const int own = eng->owner_of_stage(sid);
      eng->move(h, Mt * d * 4, at, sid);
      at = sid;
      const Range& r = D.part[static_cast<size_t>(sid - 1)];
      for (size_t li = 0; li < r.count(); ++li, ++slot) {
        if (!eng->mine(own)) continue;
        const bool dfr = train && defer_;
        const Cache c = cache_for(train ? mb : 0, slot, Mt, rows, !dfr);
        layer_fwd(sid, li, c, dfr ? wset(sid, li, wk) : wset_local(c, nullptr, Mt), h, rows, Mt);
      }
    }
    if (layers_only_) return;  // redundant-computation hot copy: the stages' forward only
    eng->move(h, Mt * d * 4, at, static_cast<int>(D.s) + 1);
    if (!eng->mine(eng->owner_of_deembed())) return;
    const float* gF = static_cast<const float*>(eng->deembed().w);
    const bf16* Einv = eng->deembed().wlp + d;
    timed(KC_NORM, 0.0, Mt * d * 10.0, [&] { llama::rmsnorm_fwd(h, gF, Mt, d, xnF, rstdF, hF, st); });
    // head, loss and head backward (model.cpp:322-342): gE_inv += xnF^T dlogits, dxn = dlogits E_inv^T
    float* gde = static_cast<float*>(eng->deembed().g);
    head(xnF, hF, rstdF, gF, Einv, lab, Mt, Mmb, train, row_loss, loss_dev, dxn, gde);
    if (!train) return;
    CKF_CUDA(cudaMemsetAsync(dh, 0, Mt * d * 4, st));
    timed(KC_NORM, 0.0, Mt * d * 18.0, [&] {
      llama::rmsnorm_bwd(dxn, hF, gF, rstdF, Mt, d, dh, dh_bf, gpart, st);
      llama::gain_fold(gpart, nblk, d, gde, st);
    });
  }

  // Redundant computation (trainer.cpp:162-171, cost_model.cpp:242-279): the node after each
  // stage holds a hot copy of it and runs its forward for every microbatch; on one GPU that is
  // one extra forward of every stage's layers (activations discarded), after the microbatch's
  // backward so the training caches are intact.
  bool layers_only_ = false;
  void redundant_forward(const int* order, const void* x, size_t rows) override {
    layers_only_ = true;
    mb_forward(0, order, x, nullptr, rows, false, nullptr);
    layers_only_ = false;
  }

  void mb_backward(int mb, const int* order, const void*, size_t rows) override {
    cudaStream_t st = eng->stream();
    const size_t Mt = rows * T;
    int* tok = buf<int>(slot_id(mb, 0), Mt);
    float* dh = buf<float>(slot_id(mb, 2), Mt * d);
    bf16* dh_bf = buf<bf16>(slot_id(mb, 3), Mt * d);
    float* dxn = buf<float>(45, Mt * d);
    bf16* scratch_bf = buf<bf16>(46, Mt * std::max(d, f));  // da / do staging
    float* Dsum = buf<float>(48, rows * H * T);
    const int nblk = llama::rmsnorm_bwd_blocks(Mt);
    float* gpart = buf<float>(49, static_cast<size_t>(nblk) * d);
    const std::vector<Applied> applied = applied_order(order);
    const int me = eng->rank();
    int at = static_cast<int>(eng->desc().s) + 1;  // dL/dh_final sits at the de-embedding
    bf16* cur = dh_bf;                              // where bf16(dh) currently lives
    for (size_t ai = applied.size(); ai-- > 0;) {
      const Applied& a = applied[ai];
      const int own = eng->owner_of_stage(a.sid);
      if (eng->move(dh, Mt * d * 4, at, a.sid)) {
        llama::f32_to_bf16(dh, dh_bf, Mt * d, st);
        cur = dh_bf;
      }
      at = a.sid;
      if (!eng->mine(own)) continue;
      const Cache c = cache_for(mb, ai, Mt, rows, !defer_);
      const WSet w = defer_ ? wset(a.sid, a.li, wk) : wset_local(c, dh_bf, Mt);
      if (cur != w.dhd) CKF_CUDA(cudaMemcpyAsync(w.dhd, cur, Mt * d * 2, cudaMemcpyDeviceToDevice, st));
      // bf16(dh) after this layer goes straight to where the next applied layer reads it
      bf16* out = dh_bf;
      if (defer_ && ai > 0 && eng->owner_of_stage(applied[ai - 1].sid) == me)
        out = wset(applied[ai - 1].sid, applied[ai - 1].li, wk).dhd;
      layer_bwd(a.sid, a.li, c, w, dh, out, dxn, scratch_bf, Dsum, gpart, nblk, rows, Mt);
      cur = out;
    }
    eng->move(dh, Mt * d * 4, at, 0);
    if (eng->mine(eng->owner_of_embed())) {
      void* sc = eng->ws(llama::embed_bwd_scratch(Mt), 55);
      timed(KC_NORM, 0.0, Mt * d * 12.0, [&] {
        llama::embed_bwd(tok, Mt, dh, d, static_cast<float*>(eng->embed().g), sc, st);
      });
    }
  }

  // ------------------------------------------------------------ plan-driven ops (schedule 2)
  // Microbatch k owns h / dh / bf16(dh) buffers for the whole iteration (slot_id(k, 4/2/3)); its
  // tokens and labels are split once per iteration; the activation caches rotate over `slots`
  // (cache_for(k % slots, ...)), which the plan's in-flight limit makes safe.  Same kernels and
  // arithmetic as mb_forward / mb_backward, one op of the global plan at a time.
  bool supports_plan() const override { return true; }
  int pslots_ = 1, pm_ = 0;
  size_t prows_ = 0;
  std::vector<bf16*> pcur_;  // per microbatch: where bf16(dh) currently lives
  int* ptok_ = nullptr;
  int* plab_ = nullptr;
  void plan_begin(int m, size_t rows, int slots, const void* x) override {
    pslots_ = std::max(1, slots);
    pm_ = m;
    prows_ = rows;
    const size_t Mt = rows * T;
    if (Mt > eng->desc().max_rows) raise(1, "microbatch tokens exceed the engine's max_rows (tokens per microbatch)");
    pcur_.assign(static_cast<size_t>(m), nullptr);
    ptok_ = buf<int>(57, static_cast<size_t>(m) * Mt);
    plab_ = buf<int>(58, static_cast<size_t>(m) * Mt);
    llama::split_tokens(static_cast<const int*>(x), static_cast<size_t>(m) * rows, T, ptok_, plab_, eng->stream());
  }
  // with the peer transport the residual stream and its gradient live in the engine's mailbox
  // (peers copy into it); otherwise in per-microbatch workspace slots
  float* ph(int k) {
    if (void* p = eng->mailbox(k, 0)) return static_cast<float*>(p);
    return buf<float>(slot_id(k, 4), prows_ * T * d);
  }
  float* pdh(int k) {
    if (void* p = eng->mailbox(k, 1)) return static_cast<float*>(p);
    return buf<float>(slot_id(k, 2), prows_ * T * d);
  }
  bf16* pdh_bf(int k) { return buf<bf16>(slot_id(k, 3), prows_ * T * d); }
  void* plan_buffer(int k, int phase, size_t* bytes) override {
    *bytes = prows_ * T * d * sizeof(float);
    return phase == 0 ? static_cast<void*>(ph(k)) : static_cast<void*>(pdh(k));
  }
  void plan_received(int k, int phase) override {
    if (phase != 1) return;
    llama::f32_to_bf16(pdh(k), pdh_bf(k), prows_ * T * d, eng->stream());  // bf16(dh) for the next dgrad
    pcur_[static_cast<size_t>(k)] = pdh_bf(k);
  }
  // position of stage sid's first layer in microbatch k's applied order
  size_t applied_base(const int* order, int sid) const {
    const Desc& D = eng->desc();
    size_t a = 0;
    for (size_t oi = 0; oi < D.s && order[oi] != sid; ++oi) a += D.part[static_cast<size_t>(order[oi] - 1)].count();
    return a;
  }
  void plan_op(int kind, int k, int sid, const int* order, double* loss_dev) override {
    cudaStream_t st = eng->stream();
    const size_t rows = prows_, Mt = rows * T;
    const int* tok = ptok_ + static_cast<size_t>(k) * Mt;
    const int* lab = plab_ + static_cast<size_t>(k) * Mt;
    const int slot = k % pslots_;
    wk = k;
    switch (kind) {
      case 0: {  // embedding (model.cpp:226)
        float* h = ph(k);
        timed(KC_NORM, 0.0, Mt * d * 8.0, [&] {
          llama::embed_fwd(tok, Mt, static_cast<const float*>(eng->embed().w), d, h, st);
        });
        break;
      }
      case 1: {  // the stage's layers, forward (model.cpp:228-249)
        float* h = ph(k);
        const Range& r = eng->desc().part[static_cast<size_t>(sid - 1)];
        const size_t a0 = applied_base(order, sid);
        for (size_t li = 0; li < r.count(); ++li) {
          const Cache c = cache_for(slot, a0 + li, Mt, rows, !defer_);
          layer_fwd(sid, li, c, defer_ ? wset(sid, li, k) : wset_local(c, nullptr, Mt), h, rows, Mt);
        }
        break;
      }
      case 3: {  // head: loss + head backward (model.cpp:250-253, 322-342)
        float* h = ph(k);
        float* dh = pdh(k);
        bf16* dh_bf = pdh_bf(k);
        float* dxn = buf<float>(45, Mt * d);
        const int nblk = llama::rmsnorm_bwd_blocks(Mt);
        float* gpart = buf<float>(49, static_cast<size_t>(nblk) * d);
        bf16* xnF = buf<bf16>(50, Mt * d);
        float* rstdF = buf<float>(51, Mt);
        float* hF = buf<float>(52, Mt * d);
        double* row_loss = buf<double>(54, Mt);
        const float* gF = static_cast<const float*>(eng->deembed().w);
        const bf16* Einv = eng->deembed().wlp + d;
        timed(KC_NORM, 0.0, Mt * d * 10.0, [&] { llama::rmsnorm_fwd(h, gF, Mt, d, xnF, rstdF, hF, st); });
        float* gde = static_cast<float*>(eng->deembed().g);
        head(xnF, hF, rstdF, gF, Einv, lab, Mt, Mt, true, row_loss, loss_dev, dxn, gde);
        CKF_CUDA(cudaMemsetAsync(dh, 0, Mt * d * 4, st));
        timed(KC_NORM, 0.0, Mt * d * 18.0, [&] {
          llama::rmsnorm_bwd(dxn, hF, gF, rstdF, Mt, d, dh, dh_bf, gpart, st);
          llama::gain_fold(gpart, nblk, d, gde, st);
        });
        pcur_[static_cast<size_t>(k)] = dh_bf;
        break;
      }
      case 4: {  // the stage's layers, backward (model.cpp:343-372)
        float* dh = pdh(k);
        bf16* dh_bf = pdh_bf(k);
        float* dxn = buf<float>(45, Mt * d);
        bf16* scratch_bf = buf<bf16>(46, Mt * std::max(d, f));
        float* Dsum = buf<float>(48, rows * H * T);
        const int nblk = llama::rmsnorm_bwd_blocks(Mt);
        float* gpart = buf<float>(49, static_cast<size_t>(nblk) * d);
        const Range& r = eng->desc().part[static_cast<size_t>(sid - 1)];
        const size_t a0 = applied_base(order, sid);
        const std::vector<Applied> applied = applied_order(order);
        bf16*& cur = pcur_[static_cast<size_t>(k)];
        if (!cur) cur = dh_bf;
        for (size_t li = r.count(); li-- > 0;) {
          const size_t ai = a0 + li;
          const Cache c = cache_for(slot, ai, Mt, rows, !defer_);
          const WSet w = defer_ ? wset(sid, li, k) : wset_local(c, dh_bf, Mt);
          if (cur != w.dhd) CKF_CUDA(cudaMemcpyAsync(w.dhd, cur, Mt * d * 2, cudaMemcpyDeviceToDevice, st));
          // bf16(dh) after this layer goes straight to where the next applied layer reads it when
          // that layer runs on this rank (the next op of this microbatch here)
          bf16* out = dh_bf;
          if (defer_ && ai > 0 && eng->mine(eng->owner_of_stage(applied[ai - 1].sid)))
            out = wset(applied[ai - 1].sid, applied[ai - 1].li, k).dhd;
          layer_bwd(sid, li, c, w, dh, out, dxn, scratch_bf, Dsum, gpart, nblk, rows, Mt);
          cur = out;
        }
        break;
      }
      case 5: {  // embedding gradient (model.cpp:373-377)
        void* sc = eng->ws(llama::embed_bwd_scratch(Mt), 55);
        float* dh = pdh(k);
        timed(KC_NORM, 0.0, Mt * d * 12.0, [&] {
          llama::embed_bwd(tok, Mt, dh, d, static_cast<float*>(eng->embed().g), sc, st);
        });
        break;
      }
      default:
        raise(1, "plan op kind not executable by the block");
    }
  }

  // SwiGLU fused into the gate/up GEMM (forward) and the down-projection dgrad
  // (backward) epilogues; CKF_FUSE_SWIGLU=0 selects the separate kernels (same bits)
  static bool fuse_swiglu() {
    const char* v = std::getenv("CKF_FUSE_SWIGLU");
    return !(v && v[0] == '0');
  }
  // the attention backward's D = rowsum(dO . O) in the O-projection dgrad's epilogue (CKF_FUSE_DSUM=0:
  // the separate dsum kernel)
  static bool fuse_dsum() {
    static const bool on = [] {
      const char* v = std::getenv("CKF_FUSE_DSUM");
      return !(v && v[0] == '0');
    }();
    return on;
  }
  const bf16* wbf(int sid, size_t li) { return eng->stage(sid).wlp + li * off.total; }
  const float* wf(int sid, size_t li) { return static_cast<const float*>(eng->stage(sid).w) + li * off.total; }
  float* gf(int sid, size_t li) { return static_cast<float*>(eng->stage(sid).g) + li * off.total; }

  double attn_flops_fwd(size_t rows) const {
    return 2.0 * rows * H * static_cast<double>(T) * T * hd;  // QK^T + PV, causal half
  }

  void layer_fwd(int sid, size_t li, const Cache& c, const WSet& w, float* h, size_t rows, size_t Mt) {
    cudaStream_t st = eng->stream();
    const bf16* W = wbf(sid, li);
    const float* Wf = wf(sid, li);
    const int Mi = static_cast<int>(Mt), di = static_cast<int>(d), fi = static_cast<int>(f);
    timed(KC_NORM, 0.0, Mt * d * 10.0, [&] { llama::rmsnorm_fwd(h, Wf + off.g1, Mt, d, w.xn1, c.rstd1, c.h_in, st); });
    if (hd == 64 || (hd == 128 && (2 * d) % 256 == 0)) {  // RoPE fused into the QKV GEMM epilogue (q, k blocks)
      gemm(Mi, 3 * di, di, w.xn1, di, false, W + off.wqkv, 3 * di, true, c.qkv, 3 * di, tc::kStoreBF16,
           llama::rope_table_pair_major(T, hd, st), static_cast<int>(2 * d));
    } else {
      gemm(Mi, 3 * di, di, w.xn1, di, false, W + off.wqkv, 3 * di, true, c.qkv, 3 * di, tc::kStoreBF16);
      timed(KC_NORM, 0.0, Mt * d * 8.0, [&] { llama::rope(c.qkv, Mt, T, d, H, 0, st); });
    }
    timed(KC_ATTN, attn_flops_fwd(rows), Mt * d * 8.0, [&] {
      if (llama::attn_fwd_tc_supported(T, hd))
        llama::attn_fwd_tc(c.qkv, rows, T, H, hd, w.o, c.lse, st);  // tcgen05 + TMEM
      else
        llama::attn_fwd(c.qkv, rows, T, H, hd, w.o, c.lse, st);
    });
    gemm(Mi, di, di, w.o, di, false, W + off.wo, di, true, h, di, tc::kAccF32);
    timed(KC_NORM, 0.0, Mt * d * 10.0, [&] { llama::rmsnorm_fwd(h, Wf + off.g2, Mt, d, w.xn2, c.rstd2, c.h_mid, st); });
    if (fuse_swiglu()) {  // a = silu(g) * u in the gate/up GEMM's epilogue
      gemm(Mi, 2 * fi, di, w.xn2, di, false, W + off.wgu, 2 * fi, true, c.gu, 2 * fi, tc::kSwiGLU, nullptr, 0, w.a, fi);
    } else {
      gemm(Mi, 2 * fi, di, w.xn2, di, false, W + off.wgu, 2 * fi, true, c.gu, 2 * fi, tc::kStoreBF16);
      timed(KC_NORM, 0.0, Mt * f * 6.0, [&] { llama::swiglu_fwd(c.gu, Mt, f, w.a, st); });
    }
    gemm(Mi, di, fi, w.a, fi, false, W + off.wd, di, true, h, di, tc::kAccF32);
  }

  // w.dhd holds bf16(dh) on entry; bf16(dh) after the layer goes to dh_bf_out
  void layer_bwd(int sid, size_t li, const Cache& c, const WSet& w, float* dh, bf16* dh_bf_out, float* dxn, bf16* sbf,
                 float* Dsum, float* gpart, int nblk, size_t rows, size_t Mt) {
    cudaStream_t st = eng->stream();
    const bf16* W = wbf(sid, li);
    const float* Wf = wf(sid, li);
    float* G = gf(sid, li);
    const int Mi = static_cast<int>(Mt), di = static_cast<int>(d), fi = static_cast<int>(f);
    const bool now = !defer_;  // weight gradients now, or batched in flush_grads()
    if (defer_ && std::find(pending_.begin(), pending_.end(), std::make_pair(sid, li)) == pending_.end())
      pending_.emplace_back(sid, li);
    // MLP half: h_out = h_mid + swiglu(xn2 Wgu) Wd
    bf16* da = sbf;
    if (now) gemm(fi, di, Mi, w.a, fi, true, w.dhd, di, true, G + off.wd, di, tc::kAccF32);   // gWd += a^T dh
    if (fuse_swiglu()) {  // da = dh Wd^T stays on chip; the epilogue emits dgu
      gemm(Mi, fi, di, w.dhd, di, false, W + off.wd, di, false, w.dgu, 2 * fi, tc::kSwiGLUBwd, nullptr, 0, c.gu, 2 * fi);
    } else {
      gemm(Mi, fi, di, w.dhd, di, false, W + off.wd, di, false, da, fi, tc::kStoreBF16);  // da = dh Wd^T
      timed(KC_NORM, 0.0, Mt * f * 10.0, [&] { llama::swiglu_bwd(c.gu, da, Mt, f, w.dgu, st); });
    }
    if (now) gemm(di, 2 * fi, Mi, w.xn2, di, true, w.dgu, 2 * fi, true, G + off.wgu, 2 * fi, tc::kAccF32);
    gemm(Mi, di, 2 * fi, w.dgu, 2 * fi, false, W + off.wgu, 2 * fi, false, dxn, di, tc::kStoreF32);  // dxn2
    timed(KC_NORM, 0.0, Mt * d * 18.0, [&] {
      llama::rmsnorm_bwd(dxn, c.h_mid, Wf + off.g2, c.rstd2, Mt, d, dh, w.dho, gpart, st);
      llama::gain_fold(gpart, nblk, d, G + off.g2, st);
    });
    // attention half: h_mid = h_in + attn(rope(xn1 Wqkv)) Wo
    bf16* d_o = sbf;
    if (now) gemm(di, di, Mi, w.o, di, true, w.dho, di, true, G + off.wo, di, tc::kAccF32);   // gWo += o^T dh
    const bool attn_tc = llama::attn_fwd_tc_supported(T, hd);
    {  // do = dh Wo^T; with the tcgen05 attention its epilogue also forms D = rowsum(do . o) per head
      tc::GemmDesc g;
      g.M = Mi;
      g.N = di;
      g.K = di;
      g.A = w.dho;
      g.lda = di;
      g.B = W + off.wo;
      g.ldb = di;
      g.C = d_o;
      g.ldc = di;
      g.epi = tc::kStoreBF16;
      if (attn_tc && fuse_dsum()) {
        g.dsum_o = w.o;
        g.dsum_out = Dsum;
        g.dsum_T = static_cast<int>(T);
        g.dsum_hd = static_cast<int>(hd);
      }
      gemm_desc(g);
    }
    timed(KC_ATTN, 2.5 * attn_flops_fwd(rows), Mt * d * 16.0, [&] {
      if (attn_tc)  // tcgen05 + TMEM, the RoPE backward in its dK / dQ epilogues
        llama::attn_bwd_tc(c.qkv, w.o, c.lse, d_o, rows, T, H, hd, w.dqkv, Dsum, st, true, fuse_dsum());
      else
        llama::attn_bwd(c.qkv, w.o, c.lse, d_o, rows, T, H, hd, w.dqkv, Dsum, st);
    });
    if (!attn_tc) timed(KC_NORM, 0.0, Mt * d * 8.0, [&] { llama::rope(w.dqkv, Mt, T, d, H, 1, st); });
    if (now) gemm(di, 3 * di, Mi, w.xn1, di, true, w.dqkv, 3 * di, true, G + off.wqkv, 3 * di, tc::kAccF32);
    gemm(Mi, di, 3 * di, w.dqkv, 3 * di, false, W + off.wqkv, 3 * di, false, dxn, di, tc::kStoreF32);  // dxn1
    timed(KC_NORM, 0.0, Mt * d * 18.0, [&] {
      llama::rmsnorm_bwd(dxn, c.h_in, Wf + off.g1, c.rstd1, Mt, d, dh, dh_bf_out, gpart, st);
      llama::gain_fold(gpart, nblk, d, G + off.g1, st);
    });
  }

  void predict(const int*, const void*, size_t, void*) override {
    raise(1, "predict is defined for the residual-MLP block");
  }
};

std::unique_ptr<BlockImpl> make_llama_block(Engine* e) { return std::make_unique<LlamaBlock>(e); }

}  // namespace ckf
