// Causal flash attention forward / backward for the LLaMA stage block.
//
// Tiles of 64 queries x 64 keys, 4 warps per CTA (16 rows each), operands
// staged in XOR-swizzled shared memory by cp.async (double-buffered K/V or
// Q/dO), fragments by ldmatrix, bf16 MMAs with fp32 accumulation, online
// softmax in registers (exp2 domain).  The backward is split into a dK/dV
// kernel (one CTA per key block, loops over query blocks) and a dQ kernel (one
// CTA per query block, loops over key blocks): every output element is
// written by exactly one thread -> no atomics, bit-deterministic.
// TODO(perf): move S/P/O to TMEM with tcgen05 (FA4-style) for the bf16 path.
#include "common.cuh"
#include "llama_kernels.h"

namespace ckf::llama {
namespace {

constexpr int BQ = 64, BKV = 64, kThreads = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// [64 rows][HD] bf16 tile, 16-byte chunks XOR-swizzled by (row & 7)
template <int HD>
__device__ __forceinline__ uint32_t tile_off(int row, int col) {
  return static_cast<uint32_t>(row * HD * 2 + ((((col >> 3) ^ (row & 7))) << 4));
}

template <int HD>
__device__ __forceinline__ void load_tile(bf16* s, const bf16* g, size_t ld, int rows_valid) {
  constexpr int chunks = 64 * HD / 8;
  for (int c = threadIdx.x; c < chunks; c += kThreads) {
    const int row = c / (HD / 8), col = (c % (HD / 8)) * 8;
    char* dst = reinterpret_cast<char*>(s) + tile_off<HD>(row, col);
    if (row < rows_valid)
      cp_async16(dst, g + static_cast<size_t>(row) * ld + col);
    else
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
  }
}

// A fragments of a 16 x HD row block (rows r0..r0+15) of a tile
template <int HD>
__device__ __forceinline__ void load_a_frags(uint32_t (&f)[HD / 16][4], const bf16* s, int r0, int lane) {
  const uint32_t base = smem_addr(s);
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int row = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int col = kk * 16 + (lane >> 4) * 8;
    ldsm_x4(f[kk], base + tile_off<HD>(row, col));
  }
}

// acc[16 x 64] += A[16 x HD] * X^T where X is a [64 rows][HD] tile (B non-transposed)
template <int HD>
__device__ __forceinline__ void mma_abt(float (&acc)[8][4], const uint32_t (&a)[HD / 16][4], const bf16* s, int lane) {
  const uint32_t base = smem_addr(s);
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      const int row = np * 16 + (lane & 7) + (lane >> 4) * 8;
      const int col = kk * 16 + ((lane >> 3) & 1) * 8;
      ldsm_x4(b, base + tile_off<HD>(row, col));
      mma16816(acc[2 * np], a[kk], b[0], b[1]);
      mma16816(acc[2 * np + 1], a[kk], b[2], b[3]);
    }
  }
}

// acc[16 x HD] += P[16 x 64] * X where X is a [64 rows][HD] tile (B transposed load)
template <int HD>
__device__ __forceinline__ void mma_px(float (&acc)[HD / 8][4], const uint32_t (&p)[4][4], const bf16* s, int lane) {
  const uint32_t base = smem_addr(s);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
    for (int dp = 0; dp < HD / 16; ++dp) {
      uint32_t b[4];
      const int row = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int col = dp * 16 + (lane >> 4) * 8;
      ldsm_x4_t(b, base + tile_off<HD>(row, col));
      mma16816(acc[2 * dp], p[kk], b[0], b[1]);
      mma16816(acc[2 * dp + 1], p[kk], b[2], b[3]);
    }
  }
}

__device__ __forceinline__ void pack_p(uint32_t (&p)[4][4], const float (&s)[8][4]) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    p[kk][0] = pack2(s[2 * kk][0], s[2 * kk][1]);
    p[kk][1] = pack2(s[2 * kk][2], s[2 * kk][3]);
    p[kk][2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
    p[kk][3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
  }
}

// ---------------------------------------------------------------- forward
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_fwd_kernel(const bf16* __restrict__ qkv, int T, int H,
                                                            bf16* __restrict__ o, float* __restrict__ lse,
                                                            float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sQ = reinterpret_cast<bf16*>(smem);
  bf16* sK = sQ + 64 * HD;       // [2][64*HD]
  bf16* sV = sK + 2 * 64 * HD;   // [2][64*HD]
  const int nqb = T / BQ;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const size_t ld = static_cast<size_t>(3) * H * HD;
  const bf16* Q = qkv + static_cast<size_t>(b) * T * ld + static_cast<size_t>(h) * HD;
  const bf16* K = Q + static_cast<size_t>(H) * HD;
  const bf16* V = Q + static_cast<size_t>(2) * H * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  load_tile<HD>(sQ, Q + static_cast<size_t>(qb) * BQ * ld, ld, BQ);
  load_tile<HD>(sK, K, ld, BKV);
  load_tile<HD>(sV, V, ld, BKV);
  cp_commit();

  uint32_t qf[HD / 16][4];
  float acc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const int qrow0 = qb * BQ + warp * 16 + g;

  for (int j = 0; j <= qb; ++j) {
    if (j + 1 <= qb) {
      load_tile<HD>(sK + ((j + 1) & 1) * 64 * HD, K + static_cast<size_t>(j + 1) * BKV * ld, ld, BKV);
      load_tile<HD>(sV + ((j + 1) & 1) * 64 * HD, V + static_cast<size_t>(j + 1) * BKV * ld, ld, BKV);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) load_a_frags<HD>(qf, sQ, warp * 16, lane);
    const bf16* k = sK + (j & 1) * 64 * HD;
    const bf16* v = sV + (j & 1) * 64 * HD;
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
    mma_abt<HD>(s, qf, k, lane);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = s[nt][e] * scale_log2;
        if (j == qb) {
          const int key = j * BKV + nt * 8 + 2 * t + (e & 1);
          const int q = qrow0 + (e >> 1) * 8;
          if (key > q) x = -INFINITY;
        }
        s[nt][e] = x;
        mx[e >> 1] = fmaxf(mx[e >> 1], x);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m[r], mx[r]);
      const float alpha = exp2f(m[r] - mn);
      m[r] = mn;
      l[r] *= alpha;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        acc[i][2 * r] *= alpha;
        acc[i][2 * r + 1] *= alpha;
      }
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(s[nt][e] - m[e >> 1]);
        s[nt][e] = p;
        l[e >> 1] += p;
      }
    }
    uint32_t pf[4][4];
    pack_p(pf, s);
    mma_px<HD>(acc, pf, v, lane);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
  const size_t ldo = static_cast<size_t>(H) * HD;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = qrow0 + r * 8;
    const float inv = 1.f / l[r];
    bf16* orow = o + (static_cast<size_t>(b) * T + q) * ldo + static_cast<size_t>(h) * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i)
      *reinterpret_cast<uint32_t*>(orow + i * 8 + 2 * t) = pack2(acc[i][2 * r] * inv, acc[i][2 * r + 1] * inv);
    if (t == 0) lse[static_cast<size_t>(bh) * T + q] = (m[r] + log2f(l[r])) * kLn2;
  }
}

// ---------------------------------------------------------------- backward
// D[bh*T + q] = sum_c dO[q, c] * O[q, c]
template <int HD>
__global__ void attn_dsum_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, int B, int T, int H,
                                 float* __restrict__ D) {
  const size_t w = blockIdx.x * static_cast<size_t>(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (w >= static_cast<size_t>(B) * T * H) return;
  const size_t tok = w / H;
  const int h = static_cast<int>(w % H);
  const size_t off = tok * H * HD + static_cast<size_t>(h) * HD;
  float acc = 0.f;
  for (int c = 2 * lane; c < HD; c += 64) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + off + c));
    const float2 d = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dout + off + c));
    acc += a.x * d.x + a.y * d.y;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  const int b = static_cast<int>(tok / T), q = static_cast<int>(tok % T);
  if (lane == 0) D[(static_cast<size_t>(b) * H + h) * T + q] = acc;
}

// dK, dV for one key block; loops over query blocks qb >= kb
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_dkdv_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                             const float* __restrict__ lse,
                                                             const float* __restrict__ D, int T, int H,
                                                             bf16* __restrict__ dqkv, float scale,
                                                             float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sK = reinterpret_cast<bf16*>(smem);
  bf16* sV = sK + 64 * HD;
  bf16* sQ = sV + 64 * HD;        // [2][64*HD]
  bf16* sdO = sQ + 2 * 64 * HD;   // [2][64*HD]
  float* sL = reinterpret_cast<float*>(sdO + 2 * 64 * HD);  // [2][64] lse * log2e
  float* sD = sL + 2 * 64;                                   // [2][64]
  const int nqb = T / BQ;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const size_t ld = static_cast<size_t>(3) * H * HD, ldo = static_cast<size_t>(H) * HD;
  const bf16* Q = qkv + static_cast<size_t>(b) * T * ld + static_cast<size_t>(h) * HD;
  const bf16* K = Q + static_cast<size_t>(H) * HD;
  const bf16* V = Q + static_cast<size_t>(2) * H * HD;
  const bf16* dO = dout + static_cast<size_t>(b) * T * ldo + static_cast<size_t>(h) * HD;
  const float* Lg = lse + static_cast<size_t>(bh) * T;
  const float* Dg = D + static_cast<size_t>(bh) * T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  auto load_q = [&](int qb, int buf) {
    load_tile<HD>(sQ + buf * 64 * HD, Q + static_cast<size_t>(qb) * BQ * ld, ld, BQ);
    load_tile<HD>(sdO + buf * 64 * HD, dO + static_cast<size_t>(qb) * BQ * ldo, ldo, BQ);
    if (threadIdx.x < 64) {
      sL[buf * 64 + threadIdx.x] = Lg[qb * BQ + threadIdx.x] * kLog2e;
      sD[buf * 64 + threadIdx.x] = Dg[qb * BQ + threadIdx.x];
    }
  };
  load_tile<HD>(sK, K + static_cast<size_t>(kb) * BKV * ld, ld, BKV);
  load_tile<HD>(sV, V + static_cast<size_t>(kb) * BKV * ld, ld, BKV);
  load_q(kb, 0);
  cp_commit();

  uint32_t kf[HD / 16][4], vf[HD / 16][4];
  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int key0 = kb * BKV + warp * 16 + g;

  for (int qb = kb; qb < nqb; ++qb) {
    const int buf = (qb - kb) & 1;
    if (qb + 1 < nqb) {
      load_q(qb + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (qb == kb) {
      load_a_frags<HD>(kf, sK, warp * 16, lane);
      load_a_frags<HD>(vf, sV, warp * 16, lane);
    }
    const bf16* q = sQ + buf * 64 * HD;
    const bf16* d_o = sdO + buf * 64 * HD;
    const float* L2 = sL + buf * 64;
    const float* Dq = sD + buf * 64;
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
    mma_abt<HD>(s, kf, q, lane);    // S^T = K Q^T  (rows = keys)
    mma_abt<HD>(dp, vf, d_o, lane); // dP^T = V dO^T
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = nt * 8 + 2 * t + (e & 1);
        const int key = key0 + (e >> 1) * 8;
        float p = exp2f(s[nt][e] * scale_log2 - L2[qi]);
        if (qb == kb && qb * BQ + qi < key) p = 0.f;
        s[nt][e] = p;
        dp[nt][e] = p * (dp[nt][e] - Dq[qi]);
      }
    }
    uint32_t pf[4][4], dsf[4][4];
    pack_p(pf, s);
    pack_p(dsf, dp);
    mma_px<HD>(dv, pf, d_o, lane);   // dV += P^T dO
    mma_px<HD>(dk, dsf, q, lane);    // dK += dS^T Q
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = key0 + r * 8;
    bf16* krow = dqkv + (static_cast<size_t>(b) * T + key) * ld + static_cast<size_t>(H) * HD + static_cast<size_t>(h) * HD;
    bf16* vrow = krow + static_cast<size_t>(H) * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      *reinterpret_cast<uint32_t*>(krow + i * 8 + 2 * t) = pack2(dk[i][2 * r] * scale, dk[i][2 * r + 1] * scale);
      *reinterpret_cast<uint32_t*>(vrow + i * 8 + 2 * t) = pack2(dv[i][2 * r], dv[i][2 * r + 1]);
    }
  }
}

// dQ for one query block; loops over key blocks kb <= qb
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_dq_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                           const float* __restrict__ lse, const float* __restrict__ D,
                                                           int T, int H, bf16* __restrict__ dqkv, float scale,
                                                           float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sQ = reinterpret_cast<bf16*>(smem);
  bf16* sdO = sQ + 64 * HD;
  bf16* sK = sdO + 64 * HD;      // [2][64*HD]
  bf16* sV = sK + 2 * 64 * HD;   // [2][64*HD]
  const int nqb = T / BQ;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const size_t ld = static_cast<size_t>(3) * H * HD, ldo = static_cast<size_t>(H) * HD;
  const bf16* Q = qkv + static_cast<size_t>(b) * T * ld + static_cast<size_t>(h) * HD;
  const bf16* K = Q + static_cast<size_t>(H) * HD;
  const bf16* V = Q + static_cast<size_t>(2) * H * HD;
  const bf16* dO = dout + static_cast<size_t>(b) * T * ldo + static_cast<size_t>(h) * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int qrow0 = qb * BQ + warp * 16 + g;

  load_tile<HD>(sQ, Q + static_cast<size_t>(qb) * BQ * ld, ld, BQ);
  load_tile<HD>(sdO, dO + static_cast<size_t>(qb) * BQ * ldo, ldo, BQ);
  load_tile<HD>(sK, K, ld, BKV);
  load_tile<HD>(sV, V, ld, BKV);
  cp_commit();
  float L2[2], Dr[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    L2[r] = lse[static_cast<size_t>(bh) * T + qrow0 + r * 8] * kLog2e;
    Dr[r] = D[static_cast<size_t>(bh) * T + qrow0 + r * 8];
  }
  uint32_t qf[HD / 16][4], df[HD / 16][4];
  float dq[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int j = 0; j <= qb; ++j) {
    if (j + 1 <= qb) {
      load_tile<HD>(sK + ((j + 1) & 1) * 64 * HD, K + static_cast<size_t>(j + 1) * BKV * ld, ld, BKV);
      load_tile<HD>(sV + ((j + 1) & 1) * 64 * HD, V + static_cast<size_t>(j + 1) * BKV * ld, ld, BKV);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
      load_a_frags<HD>(qf, sQ, warp * 16, lane);
      load_a_frags<HD>(df, sdO, warp * 16, lane);
    }
    const bf16* k = sK + (j & 1) * 64 * HD;
    const bf16* v = sV + (j & 1) * 64 * HD;
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
    mma_abt<HD>(s, qf, k, lane);   // S = Q K^T
    mma_abt<HD>(dp, df, v, lane);  // dP = dO V^T
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = j * BKV + nt * 8 + 2 * t + (e & 1);
        const int q = qrow0 + (e >> 1) * 8;
        float p = exp2f(s[nt][e] * scale_log2 - L2[e >> 1]);
        if (j == qb && key > q) p = 0.f;
        dp[nt][e] = p * (dp[nt][e] - Dr[e >> 1]);
      }
    }
    uint32_t dsf[4][4];
    pack_p(dsf, dp);
    mma_px<HD>(dq, dsf, k, lane);  // dQ += dS K
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    bf16* qrow = dqkv + (static_cast<size_t>(b) * T + qrow0 + r * 8) * ld + static_cast<size_t>(h) * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i)
      *reinterpret_cast<uint32_t*>(qrow + i * 8 + 2 * t) = pack2(dq[i][2 * r] * scale, dq[i][2 * r + 1] * scale);
  }
}

template <int HD>
void fwd_t(const bf16* qkv, size_t B, size_t T, size_t H, bf16* o, float* lse, cudaStream_t s) {
  const size_t smem = 5 * 64 * HD * sizeof(bf16);
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = true;
  }
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(HD));
  dim3 grid(static_cast<unsigned>(T / BQ), static_cast<unsigned>(B * H));
  attn_fwd_kernel<HD><<<grid, kThreads, smem, s>>>(qkv, static_cast<int>(T), static_cast<int>(H), o, lse, scale_log2);
  CKF_LAUNCH_CHECK();
}

template <int HD>
void bwd_t(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
           bf16* dqkv, float* Dsum, cudaStream_t s) {
  const size_t warps = B * T * H;
  attn_dsum_kernel<HD><<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(o, dout, static_cast<int>(B),
                                                                             static_cast<int>(T), static_cast<int>(H), Dsum);
  CKF_LAUNCH_CHECK();
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  const float scale_log2 = kLog2e * scale;
  const size_t smem_kv = 6 * 64 * HD * sizeof(bf16) + 4 * 64 * sizeof(float);
  const size_t smem_q = 6 * 64 * HD * sizeof(bf16);
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(attn_dkdv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_kv)));
    CKF_CUDA(cudaFuncSetAttribute(attn_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_q)));
    attr = true;
  }
  dim3 grid(static_cast<unsigned>(T / BQ), static_cast<unsigned>(B * H));
  attn_dkdv_kernel<HD><<<grid, kThreads, smem_kv, s>>>(qkv, dout, lse, Dsum, static_cast<int>(T), static_cast<int>(H),
                                                       dqkv, scale, scale_log2);
  CKF_LAUNCH_CHECK();
  attn_dq_kernel<HD><<<grid, kThreads, smem_q, s>>>(qkv, dout, lse, Dsum, static_cast<int>(T), static_cast<int>(H), dqkv,
                                                    scale, scale_log2);
  CKF_LAUNCH_CHECK();
}

}  // namespace

void attn_fwd(const bf16* qkv, size_t B, size_t T, size_t H, size_t hd, bf16* o, float* lse, cudaStream_t s) {
  if (T % BQ) raise(1, "attention: seq_len must be a multiple of 64");
  if (hd == 64)
    fwd_t<64>(qkv, B, T, H, o, lse, s);
  else if (hd == 128)
    fwd_t<128>(qkv, B, T, H, o, lse, s);
  else
    raise(1, "attention: head_dim must be 64 or 128");
}

void attn_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
              size_t hd, bf16* dqkv, float* Dsum, cudaStream_t s) {
  if (T % BQ) raise(1, "attention: seq_len must be a multiple of 64");
  if (hd == 64)
    bwd_t<64>(qkv, o, lse, dout, B, T, H, dqkv, Dsum, s);
  else if (hd == 128)
    bwd_t<128>(qkv, o, lse, dout, B, T, H, dqkv, Dsum, s);
  else
    raise(1, "attention: head_dim must be 64 or 128");
}

}  // namespace ckf::llama
