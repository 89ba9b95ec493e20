// fp32 parity mode of the LLaMA-style stage block (north_star: "bf16 with fp32
// accumulation plus an fp32 parity mode").  Same block, layouts, init streams and
// iteration structure as llama_block.cu, but every activation, GEMM operand and
// attention probability is fp32: GEMMs on the CUDA-core kernel (gemm_simt.cu),
// attention with the causal probabilities materialised per (sequence, head).  It
// exists to pin the block arithmetic to the fp64 oracle (oracle/llama_oracle.py)
// at ~1e-5 instead of the bf16 path's percent-level tolerances; it is not a
// throughput path (O(T^2) probability buffers, no tensor cores).
//
// Structure follows the reference where one exists (proj/src/model.cpp:211-378):
// stages in the microbatch's execution order with a per-applied-layer cache, the
// reverse walk, gradients accumulated straight into the stage accumulators.
#include <cmath>
#include <vector>

#include "engine.h"
#include "llama_kernels.h"

namespace ckf {
namespace {

using llama::kNormEps;
using llama::kRopeTheta;

// block-wide max / sum over any blockDim (multiple of 32) in a fixed order; red: >= 32 floats
__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < nw; ++i) r = fmaxf(r, red[i]);
  return r;
}
__device__ __forceinline__ float block_sum_f(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < nw; ++i) r += red[i];
  return r;
}

// ---------------------------------------------------------------- elementwise kernels (fp32)
// y = x * rstd * g (fp32), rstd, copy of x: one warp per row
__global__ void rms_fwd_f32(const float* __restrict__ x, const float* __restrict__ g, size_t rows, int d,
                            float* __restrict__ y, float* __restrict__ rstd, float* __restrict__ xcopy) {
  const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) ss += xr[c] * xr[c];
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / static_cast<float>(d) + kNormEps);
  if (lane == 0) rstd[r] = rs;
  for (int c = lane; c < d; c += 32) {
    y[r * d + c] = xr[c] * rs * g[c];
    if (xcopy) xcopy[r * d + c] = xr[c];
  }
}

// rotary embedding on q and k column blocks of qkv [ntok x 3d] (fp32, in place); pairs (j, j + hd/2)
__global__ void rope_f32(float* __restrict__ qkv, const float2* __restrict__ tab, size_t ntok, int T, int d, int hd,
                         int inverse) {
  const int half = hd / 2, per_tok = 2 * d / 2;  // (j) pairs over the q and k blocks
  const size_t n = ntok * static_cast<size_t>(per_tok);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t t = i / per_tok;
    const int rem = static_cast<int>(i % per_tok);
    const int hh = rem / half, j = rem % half;  // head (q heads then k heads), pair index
    float* base = qkv + t * 3 * d + static_cast<size_t>(hh) * hd;
    const float2 cs = tab[static_cast<size_t>(t % T) * half + j];
    const float s = inverse ? -cs.y : cs.y;
    const float a = base[j], b = base[j + half];
    base[j] = a * cs.x - b * s;
    base[j + half] = b * cs.x + a * s;
  }
}

__global__ void swiglu_fwd_f32(const float* __restrict__ gu, size_t ntok, int f, float* __restrict__ a) {
  const size_t n = ntok * f;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t t = i / f, c = i % f;
    const float g = gu[t * 2 * f + c], u = gu[t * 2 * f + f + c];
    a[i] = g / (1.f + expf(-g)) * u;
  }
}

__global__ void swiglu_bwd_f32(const float* __restrict__ gu, const float* __restrict__ da, size_t ntok, int f,
                               float* __restrict__ dgu) {
  const size_t n = ntok * f;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t t = i / f, c = i % f;
    const float g = gu[t * 2 * f + c], u = gu[t * 2 * f + f + c];
    const float sg = 1.f / (1.f + expf(-g));
    dgu[t * 2 * f + c] = da[i] * u * sg * (1.f + g * (1.f - sg));
    dgu[t * 2 * f + f + c] = da[i] * g * sg;
  }
}

// ---------------------------------------------------------------- attention (fp32, causal)
// P[bh][q][k] = softmax_k(scale * q.k) for k <= q (0 above the diagonal); o[q] = sum_k P v[k].
// One CTA per (query, sequence x head); scores in shared memory (T floats).
__global__ void attn_fwd_f32(const float* __restrict__ qkv, int T, int H, int hd, float scale, float* __restrict__ P,
                             float* __restrict__ o) {
  extern __shared__ float sc[];
  __shared__ float red[32];
  const int q = blockIdx.x, bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * hd, ld = 3 * d;
  const float* qr = qkv + (static_cast<size_t>(b) * T + q) * ld + h * hd;
  float mx = -INFINITY;
  for (int k = threadIdx.x; k <= q; k += blockDim.x) {
    const float* kr = qkv + (static_cast<size_t>(b) * T + k) * ld + d + h * hd;
    float s = 0.f;
    for (int j = 0; j < hd; ++j) s += qr[j] * kr[j];
    s *= scale;
    sc[k] = s;
    mx = fmaxf(mx, s);
  }
  mx = block_max(mx, red);
  float sum = 0.f;
  for (int k = threadIdx.x; k <= q; k += blockDim.x) {
    const float e = expf(sc[k] - mx);
    sc[k] = e;
    sum += e;
  }
  sum = block_sum_f(sum, red);
  const float inv = 1.f / sum;
  float* pr = P + (static_cast<size_t>(bh) * T + q) * T;
  for (int k = threadIdx.x; k < T; k += blockDim.x) {
    const float p = k <= q ? sc[k] * inv : 0.f;
    if (k <= q) sc[k] = p;
    pr[k] = p;
  }
  __syncthreads();
  float* orow = o + (static_cast<size_t>(b) * T + q) * d + h * hd;
  for (int j = threadIdx.x; j < hd; j += blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k <= q; ++k) acc += sc[k] * qkv[(static_cast<size_t>(b) * T + k) * ld + 2 * d + h * hd + j];
    orow[j] = acc;
  }
}

// dS[bh][q][k] = P (dP - sum_k P dP) * scale with dP[q][k] = do[q] . v[k]  (in place over a copy of P)
__global__ void attn_ds_f32(const float* __restrict__ qkv, const float* __restrict__ dout, const float* __restrict__ P,
                            int T, int H, int hd, float scale, float* __restrict__ dS) {
  extern __shared__ float sc[];
  __shared__ float red[32];
  const int q = blockIdx.x, bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * hd, ld = 3 * d;
  const float* dor = dout + (static_cast<size_t>(b) * T + q) * d + h * hd;
  const float* pr = P + (static_cast<size_t>(bh) * T + q) * T;
  float dsum = 0.f;
  for (int k = threadIdx.x; k <= q; k += blockDim.x) {
    const float* vr = qkv + (static_cast<size_t>(b) * T + k) * ld + 2 * d + h * hd;
    float dp = 0.f;
    for (int j = 0; j < hd; ++j) dp += dor[j] * vr[j];
    sc[k] = dp;
    dsum += pr[k] * dp;
  }
  dsum = block_sum_f(dsum, red);
  float* dr = dS + (static_cast<size_t>(bh) * T + q) * T;
  for (int k = threadIdx.x; k < T; k += blockDim.x) dr[k] = k <= q ? pr[k] * (sc[k] - dsum) * scale : 0.f;
}

// dq[q] = sum_k dS[q][k] k[k]  (rows of the dq block of dqkv)
__global__ void attn_dq_f32(const float* __restrict__ qkv, const float* __restrict__ dS, int T, int H, int hd,
                            float* __restrict__ dqkv) {
  const int q = blockIdx.x, bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * hd, ld = 3 * d;
  const float* dr = dS + (static_cast<size_t>(bh) * T + q) * T;
  for (int j = threadIdx.x; j < hd; j += blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k <= q; ++k) acc += dr[k] * qkv[(static_cast<size_t>(b) * T + k) * ld + d + h * hd + j];
    dqkv[(static_cast<size_t>(b) * T + q) * ld + h * hd + j] = acc;
  }
}

// dk[k] = sum_q dS[q][k] q[q];  dv[k] = sum_q P[q][k] do[q]   (q >= k)
__global__ void attn_dkdv_f32(const float* __restrict__ qkv, const float* __restrict__ dout,
                              const float* __restrict__ P, const float* __restrict__ dS, int T, int H, int hd,
                              float* __restrict__ dqkv) {
  const int k = blockIdx.x, bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * hd, ld = 3 * d;
  for (int j = threadIdx.x; j < hd; j += blockDim.x) {
    float ak = 0.f, av = 0.f;
    for (int q = k; q < T; ++q) {
      const size_t pq = (static_cast<size_t>(bh) * T + q) * T + k;
      ak += dS[pq] * qkv[(static_cast<size_t>(b) * T + q) * ld + h * hd + j];
      av += P[pq] * dout[(static_cast<size_t>(b) * T + q) * d + h * hd + j];
    }
    dqkv[(static_cast<size_t>(b) * T + k) * ld + d + h * hd + j] = ak;
    dqkv[(static_cast<size_t>(b) * T + k) * ld + 2 * d + h * hd + j] = av;
  }
}

unsigned grid1(size_t n) { return static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 32)); }

struct Off {
  size_t g1, wqkv, wo, g2, wgu, wd, total;
};

}  // namespace

struct LlamaF32Block final : BlockImpl {
  explicit LlamaF32Block(Engine* e) : BlockImpl(e) {
    const Desc& D = eng->desc();
    d = D.d;
    f = D.hid;
    V = D.out;
    H = D.heads;
    T = D.T;
    hd = d / H;
    off.g1 = 0;
    off.wqkv = d;
    off.wo = off.wqkv + 3 * d * d;
    off.g2 = off.wo + d * d;
    off.wgu = off.g2 + d;
    off.wd = off.wgu + 2 * d * f;
    off.total = off.wd + f * d;
    if (D.in != D.out) raise(1, "LLaMA block: input_dim and output_dim are both the vocabulary size");
    if (d % H || hd % 2) raise(1, "LLaMA block: model_dim must split into heads of even width");
    if (T > 4096) raise(1, "LLaMA fp32 parity mode: seq_len <= 4096 (materialised probabilities)");
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
  // identical init streams to llama_block.cu (so the parity and bf16 modes share weights)
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

  template <typename T_>
  T_* buf(int slot, size_t elems) {
    return static_cast<T_*>(eng->ws(elems * sizeof(T_), slot));
  }
  struct Cache {
    float *h_in, *h_mid, *rstd1, *rstd2, *xn1, *qkv, *P, *att, *xn2, *gu, *a;
  };
  Cache cache(size_t applied, size_t Mt, size_t rows) {
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t nP = rows * H * T * T;
    const size_t fl = al(Mt * d * 4) * 5 + al(Mt * 4) * 2 + al(Mt * 3 * d * 4) + al(nP * 4) + al(Mt * 2 * f * 4) +
                      al(Mt * f * 4);
    char* p = static_cast<char*>(eng->ws(fl, 200000 + static_cast<int>(applied)));
    auto take = [&](size_t bytes) {
      char* r = p;
      p += al(bytes);
      return reinterpret_cast<float*>(r);
    };
    Cache c;
    c.h_in = take(Mt * d * 4);
    c.h_mid = take(Mt * d * 4);
    c.xn1 = take(Mt * d * 4);
    c.att = take(Mt * d * 4);
    c.xn2 = take(Mt * d * 4);
    c.rstd1 = take(Mt * 4);
    c.rstd2 = take(Mt * 4);
    c.qkv = take(Mt * 3 * d * 4);
    c.P = take(nP * 4);
    c.gu = take(Mt * 2 * f * 4);
    c.a = take(Mt * f * 4);
    return c;
  }
  struct Applied {
    int sid;
    size_t li;
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
  float* wf(int sid, size_t li) { return static_cast<float*>(eng->stage(sid).w) + li * off.total; }
  float* gf(int sid, size_t li) { return static_cast<float*>(eng->stage(sid).g) + li * off.total; }
  // C[M,N] (+)= op(A) op(B) on CUDA cores, row-major (gemm_simt.cu)
  void mm(bool ta, bool tb, size_t M, size_t N, size_t K, const float* A, size_t lda, const float* B, size_t ldb,
          float* C, size_t ldc, bool acc) {
    eng->kt_begin();
    k::gemm_simt(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, acc, eng->stream());
    eng->kt_end(KC_GEMM, 2.0 * M * N * K, 4.0 * (M * K + K * N + M * N));
  }
  void rms(const float* x, const float* g, size_t rows, float* y, float* rstd, float* xcopy) {
    rms_fwd_f32<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, eng->stream()>>>(x, g, rows, static_cast<int>(d), y,
                                                                                   rstd, xcopy);
    CKF_LAUNCH_CHECK();
  }
  void rms_bwd(const float* dxn, const float* x, const float* g, const float* rstd, size_t Mt, float* dh, float* G) {
    const int nblk = llama::rmsnorm_bwd_blocks(Mt);
    float* gpart = buf<float>(249, static_cast<size_t>(nblk) * d);
    llama::rmsnorm_bwd(dxn, x, g, rstd, Mt, d, dh, nullptr, gpart, eng->stream());
    llama::gain_fold(gpart, nblk, d, G, eng->stream());
  }

  void mb_forward(int, const int* order, const void* xv, const void*, size_t rows, bool train,
                  double* loss_dev) override {
    const Desc& D = eng->desc();
    cudaStream_t st = eng->stream();
    const size_t Mt = rows * T;
    if (Mt > D.max_rows) raise(1, "microbatch tokens exceed the engine's max_rows (tokens per microbatch)");
    for (size_t i = 0; i < D.s; ++i)
      if (!eng->mine(eng->owner_of_stage(static_cast<int>(i + 1))))
        raise(1, "the LLaMA fp32 parity mode runs with every stage on one GPU");
    const int* x = static_cast<const int*>(xv);
    int* tok = buf<int>(240, Mt);
    int* lab = buf<int>(241, Mt);
    float* h = buf<float>(242, Mt * d);
    llama::split_tokens(x, rows, T, tok, lab, st);
    llama::embed_fwd(tok, Mt, static_cast<const float*>(eng->embed().w), d, h, st);
    const float2* tab = llama::rope_table(T, hd, st);
    const float scale = 1.f / std::sqrt(static_cast<float>(hd));
    const std::vector<Applied> ap = applied_order(order);
    const dim3 ag(static_cast<unsigned>(T), static_cast<unsigned>(rows * H));
    for (size_t ai = 0; ai < ap.size(); ++ai) {
      const Cache c = cache(ai, Mt, rows);
      const float* W = wf(ap[ai].sid, ap[ai].li);
      rms(h, W + off.g1, Mt, c.xn1, c.rstd1, c.h_in);
      mm(false, false, Mt, 3 * d, d, c.xn1, d, W + off.wqkv, 3 * d, c.qkv, 3 * d, false);
      rope_f32<<<grid1(Mt * d), 256, 0, st>>>(c.qkv, tab, Mt, static_cast<int>(T), static_cast<int>(d),
                                                static_cast<int>(hd), 0);
      CKF_LAUNCH_CHECK();
      attn_fwd_f32<<<ag, 128, T * sizeof(float), st>>>(c.qkv, static_cast<int>(T), static_cast<int>(H),
                                                        static_cast<int>(hd), scale, c.P, c.att);
      CKF_LAUNCH_CHECK();
      mm(false, false, Mt, d, d, c.att, d, W + off.wo, d, h, d, true);  // h += att Wo
      rms(h, W + off.g2, Mt, c.xn2, c.rstd2, c.h_mid);
      mm(false, false, Mt, 2 * f, d, c.xn2, d, W + off.wgu, 2 * f, c.gu, 2 * f, false);
      swiglu_fwd_f32<<<grid1(Mt * f), 256, 0, st>>>(c.gu, Mt, static_cast<int>(f), c.a);
      CKF_LAUNCH_CHECK();
      mm(false, false, Mt, d, f, c.a, f, W + off.wd, d, h, d, true);  // h += a Wd
    }
    // head (model.cpp:251-253, 322-342): logits = RMSNorm(h; gF) E_inv; mean token CE
    const float* gF = static_cast<const float*>(eng->deembed().w);
    const float* Einv = gF + d;
    float* xnF = buf<float>(243, Mt * d);
    float* rstdF = buf<float>(244, Mt);
    float* hF = buf<float>(245, Mt * d);
    float* logits = buf<float>(246, Mt * V);
    float* dlogits = train ? buf<float>(254, Mt * V) : nullptr;
    rms(h, gF, Mt, xnF, rstdF, hF);
    mm(false, false, Mt, V, d, xnF, d, Einv, V, logits, V, false);
    // mean token cross-entropy and (softmax - onehot) / tokens (kernels_serial.cpp:163-185)
    k::xent_loss_grad(logits, lab, Mt, V, dlogits, loss_dev, eng->scratch(), st);
    if (!train) return;
    logits = dlogits;
    float* gde = static_cast<float*>(eng->deembed().g);
    float* dh = buf<float>(247, Mt * d);
    float* dxn = buf<float>(248, Mt * d);
    mm(true, false, d, V, Mt, xnF, d, logits, V, gde + d, V, true);   // gE_inv += xnF^T dlogits
    mm(false, true, Mt, d, V, logits, V, Einv, V, dxn, d, false);     // dxnF = dlogits E_inv^T
    CKF_CUDA(cudaMemsetAsync(dh, 0, Mt * d * 4, st));
    rms_bwd(dxn, hF, gF, rstdF, Mt, dh, gde);
  }

  void mb_backward(int, const int* order, const void*, size_t rows) override {
    cudaStream_t st = eng->stream();
    const size_t Mt = rows * T;
    int* tok = buf<int>(240, Mt);
    float* dh = buf<float>(247, Mt * d);
    float* dxn = buf<float>(248, Mt * d);
    float* t1 = buf<float>(250, Mt * std::max(2 * f, 3 * d));
    float* t2 = buf<float>(251, Mt * std::max(f, d));
    float* dS = buf<float>(252, rows * H * T * T);
    const float2* tab = llama::rope_table(T, hd, st);
    const float scale = 1.f / std::sqrt(static_cast<float>(hd));
    const std::vector<Applied> ap = applied_order(order);
    const dim3 ag(static_cast<unsigned>(T), static_cast<unsigned>(rows * H));
    for (size_t ai = ap.size(); ai-- > 0;) {
      const Cache c = cache(ai, Mt, rows);
      const float* W = wf(ap[ai].sid, ap[ai].li);
      float* G = gf(ap[ai].sid, ap[ai].li);
      // MLP half: h_out = h_mid + swiglu(xn2 Wgu) Wd
      mm(true, false, f, d, Mt, c.a, f, dh, d, G + off.wd, d, true);         // gWd += a^T dh
      mm(false, true, Mt, f, d, dh, d, W + off.wd, d, t2, f, false);         // da = dh Wd^T
      swiglu_bwd_f32<<<grid1(Mt * f), 256, 0, st>>>(c.gu, t2, Mt, static_cast<int>(f), t1);  // dgu
      CKF_LAUNCH_CHECK();
      mm(true, false, d, 2 * f, Mt, c.xn2, d, t1, 2 * f, G + off.wgu, 2 * f, true);
      mm(false, true, Mt, d, 2 * f, t1, 2 * f, W + off.wgu, 2 * f, dxn, d, false);  // dxn2
      rms_bwd(dxn, c.h_mid, W + off.g2, c.rstd2, Mt, dh, G + off.g2);
      // attention half: h_mid = h_in + attn(rope(xn1 Wqkv)) Wo
      mm(true, false, d, d, Mt, c.att, d, dh, d, G + off.wo, d, true);       // gWo += att^T dh
      mm(false, true, Mt, d, d, dh, d, W + off.wo, d, t2, d, false);         // d_att = dh Wo^T
      attn_ds_f32<<<ag, 128, T * sizeof(float), st>>>(c.qkv, t2, c.P, static_cast<int>(T), static_cast<int>(H),
                                                       static_cast<int>(hd), scale, dS);
      CKF_LAUNCH_CHECK();
      attn_dq_f32<<<ag, 64, 0, st>>>(c.qkv, dS, static_cast<int>(T), static_cast<int>(H), static_cast<int>(hd), t1);
      CKF_LAUNCH_CHECK();
      attn_dkdv_f32<<<ag, 64, 0, st>>>(c.qkv, t2, c.P, dS, static_cast<int>(T), static_cast<int>(H),
                                       static_cast<int>(hd), t1);
      CKF_LAUNCH_CHECK();
      rope_f32<<<grid1(Mt * d), 256, 0, st>>>(t1, tab, Mt, static_cast<int>(T), static_cast<int>(d),
                                                static_cast<int>(hd), 1);
      CKF_LAUNCH_CHECK();
      mm(true, false, d, 3 * d, Mt, c.xn1, d, t1, 3 * d, G + off.wqkv, 3 * d, true);
      mm(false, true, Mt, d, 3 * d, t1, 3 * d, W + off.wqkv, 3 * d, dxn, d, false);  // dxn1
      rms_bwd(dxn, c.h_in, W + off.g1, c.rstd1, Mt, dh, G + off.g1);
    }
    void* sc = eng->ws(llama::embed_bwd_scratch(Mt), 253);
    llama::embed_bwd(tok, Mt, dh, d, static_cast<float*>(eng->embed().g), sc, st);
  }

  void predict(const int*, const void*, size_t, void*) override {
    raise(1, "predict is defined for the residual-MLP block");
  }
};

std::unique_ptr<BlockImpl> make_llama_f32_block(Engine* e) { return std::make_unique<LlamaF32Block>(e); }

}  // namespace ckf
