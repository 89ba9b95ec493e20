// Bandwidth-bound kernels of the LLaMA-style stage block: embedding gather /
// deterministic scatter, RMSNorm fwd/bwd (+ gain gradients), RoPE, SwiGLU,
// cross-entropy over bf16 logits.  One warp per row for the row-wise ops,
// 128-bit vector loads, warp-shuffle reductions; every reduction has a fixed
// order so a training run is bit-reproducible (the GPU analogue of the
// reference's fixed-order reductions, kernels.hpp:10-13).
#include <cub/device/device_radix_sort.cuh>

#include <vector>

#include "common.cuh"
#include "llama_kernels.h"
#include "sm100.cuh"

namespace ckf::llama {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const int* __restrict__ tok, size_t ntok, const float4* __restrict__ E, size_t d4,
                                 float4* __restrict__ h) {
  const size_t t = blockIdx.x * static_cast<size_t>(kWarpsPerBlock) + threadIdx.x / 32;
  if (t >= ntok) return;
  const float4* src = E + static_cast<size_t>(tok[t]) * d4;
  float4* dst = h + t * d4;
  for (size_t c = threadIdx.x & 31; c < d4; c += 32) dst[c] = src[c];
}

__global__ void iota_kernel(int* __restrict__ v, size_t n) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = static_cast<int>(i);
}

// one warp per sorted position; the first position of each token segment sums
// the segment's rows in (stable-sorted = token) order and adds once to gE
__global__ void embed_bwd_kernel(const int* __restrict__ keys, const int* __restrict__ pos, size_t ntok,
                                 const float4* __restrict__ dh, size_t d4, float4* __restrict__ gE) {
  const size_t i = blockIdx.x * static_cast<size_t>(kWarpsPerBlock) + threadIdx.x / 32;
  if (i >= ntok) return;
  const int key = keys[i];
  if (i > 0 && keys[i - 1] == key) return;
  size_t end = i + 1;
  while (end < ntok && keys[end] == key) ++end;
  for (size_t c = threadIdx.x & 31; c < d4; c += 32) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (size_t j = i; j < end; ++j) {
      const float4 v = dh[static_cast<size_t>(pos[j]) * d4 + c];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    float4 g = gE[static_cast<size_t>(key) * d4 + c];
    g.x += acc.x;
    g.y += acc.y;
    g.z += acc.z;
    g.w += acc.w;
    gE[static_cast<size_t>(key) * d4 + c] = g;
  }
}

// ---------------------------------------------------------------- RMSNorm
// one warp per row; the row lives in registers (lane owns columns lane + 32 i)
template <int V4>  // float4 per lane (d = 128 * V4)
__global__ void __launch_bounds__(256) rmsnorm_fwd_kernel(const float4* __restrict__ x, const float4* __restrict__ g,
                                                          size_t rows, __nv_bfloat162* __restrict__ y,
                                                          float* __restrict__ rstd, float4* __restrict__ xcopy) {
  constexpr int d4 = 32 * V4;
  const size_t r = blockIdx.x * static_cast<size_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float4 v[V4];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    v[i] = x[r * d4 + lane + 32 * i];
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = warp_sum_f(ss);
  const float rs = rsqrtf(ss / static_cast<float>(4 * d4) + kNormEps);
  if (lane == 0) rstd[r] = rs;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const size_t c = r * d4 + lane + 32 * i;
    const float4 gg = g[lane + 32 * i];
    const __nv_bfloat162 y0 = __floats2bfloat162_rn(v[i].x * rs * gg.x, v[i].y * rs * gg.y);
    const __nv_bfloat162 y1 = __floats2bfloat162_rn(v[i].z * rs * gg.z, v[i].w * rs * gg.w);
    reinterpret_cast<uint2*>(y)[c] = make_uint2(*reinterpret_cast<const uint32_t*>(&y0),
                                                *reinterpret_cast<const uint32_t*>(&y1));  // one 8-byte store
    if (xcopy) xcopy[c] = v[i];
  }
}

constexpr int kBwdRowsPerBlock = 16;  // 512 CTAs for 8192 rows: enough warps in flight per SM

// dh += rstd*u - x*rstd^3*(u.x)/d with u = g*dy; gain partial += dy*x*rstd.
// One warp per row (lane owns columns lane + 32 i); dy, x and dh of the row are loaded
// together.  The gains and each warp's gain partials live in shared memory, not registers,
// which keeps d = 512 at two 256-thread blocks per SM without spills (more rows in flight); the 8 warps'
// partials are folded in fixed order.
template <int V4>  // float4 per lane (d = 128 * V4)
__global__ void __launch_bounds__(256, (V4 <= 4 ? 2 : 1))
    rmsnorm_bwd_kernel(const float4* __restrict__ dy, const float4* __restrict__ x, const float4* __restrict__ g,
                       const float* __restrict__ rstd, size_t rows, float4* __restrict__ dh,
                       __nv_bfloat162* __restrict__ dh_bf, float* __restrict__ gpart) {
  extern __shared__ float4 sg[];  // [kWarpsPerBlock][d4] gain partials, then [d4] gains
  constexpr int d4 = 32 * V4;
  float4* sgg = sg + kWarpsPerBlock * d4;
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  float4* gpw = sg + static_cast<size_t>(w) * d4;
  for (int c = threadIdx.x; c < d4; c += blockDim.x) sgg[c] = g[c];
#pragma unroll
  for (int i = 0; i < V4; ++i) gpw[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  // persistent: warp w of block b takes rows b * W + w, then every gridDim.x * W rows (a fixed
  // assignment, so each block's gain partial sums a fixed row set in a fixed order)
  for (size_t r = static_cast<size_t>(blockIdx.x) * kWarpsPerBlock + w; r < rows;
       r += static_cast<size_t>(gridDim.x) * kWarpsPerBlock) {
    const float rs = rstd[r];
    float4 a[V4], b[V4], o4[V4];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) {  // dy, x and the dh being accumulated into: all in flight at once
      a[i] = dy[r * d4 + lane + 32 * i];
      b[i] = x[r * d4 + lane + 32 * i];
      if (V4 <= 8) o4[i] = dh[r * d4 + lane + 32 * i];
    }
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const float4 gg = sgg[lane + 32 * i];
      dot += gg.x * a[i].x * b[i].x + gg.y * a[i].y * b[i].y + gg.z * a[i].z * b[i].z + gg.w * a[i].w * b[i].w;
    }
    dot = warp_sum_f(dot);
    const float coef = rs * rs * rs * dot / static_cast<float>(4 * d4);
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const size_t c = r * d4 + lane + 32 * i;
      const float4 gg = sgg[lane + 32 * i];
      float4 o = V4 <= 8 ? o4[i] : dh[c];
      o.x += rs * gg.x * a[i].x - b[i].x * coef;
      o.y += rs * gg.y * a[i].y - b[i].y * coef;
      o.z += rs * gg.z * a[i].z - b[i].z * coef;
      o.w += rs * gg.w * a[i].w - b[i].w * coef;
      dh[c] = o;
      if (dh_bf) {
        const __nv_bfloat162 b0 = __floats2bfloat162_rn(o.x, o.y), b1 = __floats2bfloat162_rn(o.z, o.w);
        reinterpret_cast<uint2*>(dh_bf)[c] = make_uint2(*reinterpret_cast<const uint32_t*>(&b0),
                                                        *reinterpret_cast<const uint32_t*>(&b1));
      }
      float4 gp = gpw[lane + 32 * i];
      gp.x += a[i].x * b[i].x * rs;
      gp.y += a[i].y * b[i].y * rs;
      gp.z += a[i].z * b[i].z * rs;
      gp.w += a[i].w * b[i].w * rs;
      gpw[lane + 32 * i] = gp;
    }
  }
  __syncthreads();
  const float* sgf = reinterpret_cast<const float*>(sg);
  for (int c = threadIdx.x; c < 4 * d4; c += blockDim.x) {
    float acc = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarpsPerBlock; ++ww) acc += sgf[ww * 4 * d4 + c];
    gpart[static_cast<size_t>(blockIdx.x) * 4 * d4 + c] = acc;
  }
}

// gg[c] += sum_b gpart[b, c]: a CTA owns 2 columns; its 128 slices sum the fixed
// residue classes b = slice (mod 128) -- 128 independent loads in flight per column
// instead of a serial walk, d / 2 CTAs (8.8 vs 17 us at d = 512) -- then one thread per column folds the
// slices in order (fixed order: the result does not depend on the GPU)
constexpr int kFoldCols = 2, kFoldSlices = 128;
__global__ void gain_fold_kernel(const float* __restrict__ gpart, int nblk, int d, float* __restrict__ gg) {
  __shared__ float part[kFoldSlices][kFoldCols + 1];
  const int cl = threadIdx.x % kFoldCols, sl = threadIdx.x / kFoldCols;
  const int c = blockIdx.x * kFoldCols + cl;
  float acc = 0.f;
  if (c < d)
    for (int b = sl; b < nblk; b += kFoldSlices) acc += gpart[static_cast<size_t>(b) * d + c];
  part[sl][cl] = acc;
  __syncthreads();
  if (threadIdx.x < kFoldCols && c < d) {
    float s = 0.f;
#pragma unroll 8
    for (int k = 0; k < kFoldSlices; ++k) s += part[k][cl];
    gg[c] += s;
  }
}

// ---------------------------------------------------------------- RoPE
// cos/sin table [T][hd/2] (float2), built once per (T, hd) on the device
__global__ void rope_table_kernel(float2* __restrict__ tab, int T, int hd, int pair_major) {
  const int half = hd / 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T * half) return;
  // [T][hd/2] (position-major) or [hd/2][T] (pair-major: consecutive positions adjacent, so
  // a warp of consecutive rows reads one table entry each with coalesced loads)
  const int pos = pair_major ? i % T : i / half, j = pair_major ? i / T : i % half;
  const double inv = exp2(-static_cast<double>(2 * j) / hd * log2(static_cast<double>(kRopeTheta)));
  double sn, cs;
  sincos(static_cast<double>(pos) * inv, &sn, &cs);
  tab[i] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
}

// one thread = 4 consecutive rotation pairs (j..j+3, j+half..j+half+3) of one head of q or k
__global__ void rope_kernel(__nv_bfloat16* __restrict__ qkv, const float2* __restrict__ tab, int ntok, int T, int d,
                            int hd, int inverse) {
  const int half = hd / 2, per_head = half / 4, per_tok = 2 * d / 8;  // items per token (q and k)
  const unsigned n = static_cast<unsigned>(ntok) * static_cast<unsigned>(per_tok);  // < 2^32 (host check)
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int t = static_cast<int>(i / static_cast<unsigned>(per_tok));  // 32-bit division
    const int rem = static_cast<int>(i - static_cast<unsigned>(t) * static_cast<unsigned>(per_tok));
    const int hh = rem / per_head;  // 0..2H-1 (q heads then k heads)
    const int j = (rem % per_head) * 4;
    __nv_bfloat16* base = qkv + static_cast<size_t>(t) * 3 * d + static_cast<size_t>(hh) * hd;
    uint2 u1 = *reinterpret_cast<const uint2*>(base + j);
    uint2 u2 = *reinterpret_cast<const uint2*>(base + j + half);
    __nv_bfloat162* p1 = reinterpret_cast<__nv_bfloat162*>(&u1);
    __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&u2);
    const float2* cs = tab + static_cast<size_t>(t % T) * half + j;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float2 a = __bfloat1622float2(p1[q]), b = __bfloat1622float2(p2[q]);
      const float2 c0 = cs[2 * q], c1 = cs[2 * q + 1];
      const float s0 = inverse ? -c0.y : c0.y, s1 = inverse ? -c1.y : c1.y;
      p1[q] = __floats2bfloat162_rn(a.x * c0.x - b.x * s0, a.y * c1.x - b.y * s1);
      p2[q] = __floats2bfloat162_rn(b.x * c0.x + a.x * s0, b.y * c1.x + a.y * s1);
    }
    *reinterpret_cast<uint2*>(base + j) = u1;
    *reinterpret_cast<uint2*>(base + j + half) = u2;
  }
}

// ---------------------------------------------------------------- SwiGLU
// 8 columns per thread, 16-byte loads/stores; gu = [gate | up] rows of 2f
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = __bfloat1622float2(p[q]);
    f[2 * q] = v.x;
    f[2 * q + 1] = v.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) p[q] = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
  return u;
}

__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu, int ntok, int f,
                                  __nv_bfloat16* __restrict__ a) {
  const unsigned f8 = static_cast<unsigned>(f) / 8;
  const unsigned n = static_cast<unsigned>(ntok) * f8;  // < 2^32 for any microbatch this engine runs
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned t = i / f8, c = (i - t * f8) * 8;
    const __nv_bfloat16* row = gu + static_cast<size_t>(t) * 2 * f;
    float g[8], u[8], o[8];
    unpack8(*reinterpret_cast<const uint4*>(row + c), g);
    unpack8(*reinterpret_cast<const uint4*>(row + f + c), u);
#pragma unroll
    for (int k = 0; k < 8; k += 2) f2split(swiglu_fwd2(f2(g[k], g[k + 1]), f2(u[k], u[k + 1])), o[k], o[k + 1]);
    *reinterpret_cast<uint4*>(a + static_cast<size_t>(t) * f + c) = pack8(o);
  }
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu, const __nv_bfloat16* __restrict__ da,
                                  int ntok, int f, __nv_bfloat16* __restrict__ dgu) {
  const unsigned f8 = static_cast<unsigned>(f) / 8;
  const unsigned n = static_cast<unsigned>(ntok) * f8;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned t = i / f8, c = (i - t * f8) * 8;
    const __nv_bfloat16* row = gu + static_cast<size_t>(t) * 2 * f;
    float g[8], u[8], dd[8], dg[8], du[8];
    unpack8(*reinterpret_cast<const uint4*>(row + c), g);
    unpack8(*reinterpret_cast<const uint4*>(row + f + c), u);
    unpack8(*reinterpret_cast<const uint4*>(da + static_cast<size_t>(t) * f + c), dd);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      f32x2 dg2, du2;
      swiglu_bwd2(f2(g[k], g[k + 1]), f2(u[k], u[k + 1]), f2(dd[k], dd[k + 1]), dg2, du2);
      f2split(dg2, dg[k], dg[k + 1]);
      f2split(du2, du[k], du[k + 1]);
    }
    __nv_bfloat16* out = dgu + static_cast<size_t>(t) * 2 * f;
    *reinterpret_cast<uint4*>(out + c) = pack8(dg);
    *reinterpret_cast<uint4*>(out + f + c) = pack8(du);
  }
}

// ---------------------------------------------------------------- cross-entropy
constexpr int kXentThreads = 512;

__global__ void __launch_bounds__(kXentThreads) xent_kernel(__nv_bfloat16* __restrict__ logits,
                                                            const int* __restrict__ labels, size_t V, float gscale,
                                                            int grad, double* __restrict__ row_loss) {
  __shared__ float sm[kXentThreads / 32], ss[kXentThreads / 32];
  const size_t r = blockIdx.x;
  __nv_bfloat16* row = logits + r * V;
  float m = -INFINITY, s = 0.f;
  const bool vec = (V % 8 == 0);
  if (vec) {
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    for (size_t c = threadIdx.x; c < V / 8; c += kXentThreads) {
      uint4 u = rv[c];
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(p[q]);
        const float mx = fmaxf(m, fmaxf(f.x, f.y));
        s = s * __expf(m - mx) + __expf(f.x - mx) + __expf(f.y - mx);
        m = mx;
      }
    }
  } else {
    for (size_t c = threadIdx.x; c < V; c += kXentThreads) {
      const float f = __bfloat162float(row[c]);
      const float mx = fmaxf(m, f);
      s = s * __expf(m - mx) + __expf(f - mx);
      m = mx;
    }
  }
  // warp then block combine of (max, sum)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mx = fmaxf(m, m2);
    s = (mx == -INFINITY) ? 0.f : s * __expf(m - mx) + s2 * __expf(m2 - mx);
    m = mx;
  }
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  if (l == 0) {
    sm[w] = m;
    ss[w] = s;
  }
  __syncthreads();
  float M = -INFINITY, S = 0.f;
  for (int i = 0; i < kXentThreads / 32; ++i) {
    if (sm[i] == -INFINITY) continue;
    const float mx = fmaxf(M, sm[i]);
    S = S * __expf(M - mx) + ss[i] * __expf(sm[i] - mx);
    M = mx;
  }
  const float lse = M + __logf(S);
  const int y = labels[r];
  if (threadIdx.x == 0) row_loss[r] = static_cast<double>(lse) - static_cast<double>(__bfloat162float(row[y]));
  __syncthreads();  // everyone has read row[y] before it is overwritten
  if (!grad) return;
  if (vec) {
    uint4* rv = reinterpret_cast<uint4*>(row);
    for (size_t c = threadIdx.x; c < V / 8; c += kXentThreads) {
      uint4 u = rv[c];
      __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(p[q]);
        const size_t j = c * 8 + 2 * q;
        const float g0 = (__expf(f.x - lse) - (static_cast<int>(j) == y ? 1.f : 0.f)) * gscale;
        const float g1 = (__expf(f.y - lse) - (static_cast<int>(j + 1) == y ? 1.f : 0.f)) * gscale;
        p[q] = __floats2bfloat162_rn(g0, g1);
      }
      rv[c] = u;
    }
  } else {
    for (size_t c = threadIdx.x; c < V; c += kXentThreads) {
      const float f = __bfloat162float(row[c]);
      row[c] = __float2bfloat16((__expf(f - lse) - (static_cast<int>(c) == y ? 1.f : 0.f)) * gscale);
    }
  }
}

// Register-resident variant (V % 8 == 0, V / 8 <= NC * kXentThreads): each thread keeps its NC
// 16-byte chunks of the row in registers, so the logits are read from HBM once and the
// gradient overwrites them in place; exact two-pass max / sum (one exp2 per logit per pass).
template <int NC>
__global__ void __launch_bounds__(kXentThreads) xent_reg_kernel(__nv_bfloat16* __restrict__ logits,
                                                                const int* __restrict__ labels, int V, float gscale,
                                                                int grad, double* __restrict__ row_loss) {
  __shared__ float red[kXentThreads / 32];
  __shared__ float bcast[2];
  constexpr float kL2e = 1.4426950408889634f;
  const size_t r = blockIdx.x;
  uint4* rv = reinterpret_cast<uint4*>(logits + r * static_cast<size_t>(V));
  const int V8 = V / 8;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint4 u[NC];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = threadIdx.x + k * kXentThreads;
    u[k] = c < V8 ? rv[c] : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);  // bf16 -inf
    const uint32_t* q = reinterpret_cast<const uint32_t*>(&u[k]);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      m = fmaxf(m, fmaxf(__uint_as_float(q[e] << 16), __uint_as_float(q[e] & 0xffff0000u)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (l == 0) red[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = red[0];
    for (int i = 1; i < kXentThreads / 32; ++i) M = fmaxf(M, red[i]);
    bcast[0] = M;
  }
  __syncthreads();
  const float M = bcast[0], Ml = M * kL2e;
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(&u[k]);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      s += exp2f(fmaf(__uint_as_float(q[e] << 16), kL2e, -Ml)) +
           exp2f(fmaf(__uint_as_float(q[e] & 0xffff0000u), kL2e, -Ml));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int y = labels[r];
  float xy = 0.f;
  if (threadIdx.x == 0) xy = __bfloat162float(logits[r * static_cast<size_t>(V) + y]);
  __syncthreads();  // red[] reuse; row[y] read before any gradient store
  if (l == 0) red[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float S = 0.f;
    for (int i = 0; i < kXentThreads / 32; ++i) S += red[i];
    const float lse = M + __logf(S);
    bcast[1] = lse;
    row_loss[r] = static_cast<double>(lse) - static_cast<double>(xy);
  }
  if (!grad) return;
  __syncthreads();
  const float Ll = bcast[1] * kL2e;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = threadIdx.x + k * kXentThreads;
    if (c >= V8) continue;
    const uint32_t* q = reinterpret_cast<const uint32_t*>(&u[k]);
    uint4 o;
    uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = 8 * c + 2 * e;
      const float g0 = (exp2f(fmaf(__uint_as_float(q[e] << 16), kL2e, -Ll)) - (j == y ? 1.f : 0.f)) * gscale;
      const float g1 = (exp2f(fmaf(__uint_as_float(q[e] & 0xffff0000u), kL2e, -Ll)) - (j + 1 == y ? 1.f : 0.f)) * gscale;
      const __nv_bfloat162 b = __floats2bfloat162_rn(g0, g1);
      po[e] = *reinterpret_cast<const uint32_t*>(&b);
    }
    rv[c] = o;
  }
}

// Persistent, row-pipelined variant (V % 8 == 0, 2 rows fit in shared memory): row i + 2 is
// bulk-copied (cp.async.bulk) into shared memory while row i is reduced, so the logits are
// read from HBM once, the gradient is written once, and the load latency is hidden.
// exp2 as one MUFU op (ex2.approx.ftz: ~2 ulp, results below 2^-126 flush to 0) -- exp2f()'s
// range fix-ups cost three more instructions per element, and this kernel is issue-bound
// (measured: 2.81 -> 2.52 ms at 65,536 x 50,304; a polynomial exp2 on the FMA pipe for 3/8
// of the elements was slower, 3.01 ms, so MUFU is not the bound).
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr int kXentPipeThreads = 512;
__global__ void __launch_bounds__(kXentPipeThreads, 1)
    xent_pipe_kernel(__nv_bfloat16* __restrict__ logits, const int* __restrict__ labels, int rows, int V, float gscale,
                     int grad, double* __restrict__ row_loss) {
  extern __shared__ uint8_t xsm_raw[];
  uint8_t* xsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(xsm_raw) + 127) & ~uintptr_t(127));
  const uint32_t rowb = static_cast<uint32_t>(V) * 2, rowb_al = (rowb + 127) & ~127u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(xsm + 2 * rowb_al);
  float* red = reinterpret_cast<float*>(bar + 2);
  constexpr float kL2e = 1.4426950408889634f;
  const int V8 = V / 8, w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar[0], 1);
    sm100::mbar_init(&bar[1], 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int i) {  // thread 0: row blockIdx.x + i * gridDim.x into buffer i & 1
    const int r = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    if (r >= rows) return;
    sm100::mbar_arrive_expect_tx(&bar[i & 1], rowb);
    sm100::bulk_load(xsm + (i & 1) * rowb_al, logits + static_cast<size_t>(r) * V, rowb, &bar[i & 1]);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  for (int i = 0;; ++i) {
    const int r = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    if (r >= rows) break;
    const uint32_t base = sm100::smem_u32(xsm + (i & 1) * rowb_al);
    sm100::mbar_wait(&bar[i & 1], (i >> 1) & 1);
    float m = -INFINITY;
    for (int c = threadIdx.x; c < V8; c += kXentPipeThreads) {
      const uint4 u = sm100::ld_shared_v4(base + 16 * c);
      const uint32_t q[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) m = fmaxf(m, fmaxf(__uint_as_float(q[e] << 16), __uint_as_float(q[e] & 0xffff0000u)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (l == 0) red[w] = m;
    __syncthreads();
    float M = red[0];
#pragma unroll
    for (int k = 1; k < kXentPipeThreads / 32; ++k) M = fmaxf(M, red[k]);
    const float Ml = M * kL2e;
    float sum = 0.f;
    for (int c = threadIdx.x; c < V8; c += kXentPipeThreads) {
      const uint4 u = sm100::ld_shared_v4(base + 16 * c);
      const uint32_t q[4] = {u.x, u.y, u.z, u.w};
      float s8[8];
#define CKF_X(E) s8[E] = ex2_mufu(fmaf(__uint_as_float((E & 1) ? (q[E / 2] & 0xffff0000u) : (q[E / 2] << 16)), kL2e, -Ml));
      CKF_X(0) CKF_X(1) CKF_X(2) CKF_X(3) CKF_X(4) CKF_X(5) CKF_X(6) CKF_X(7)
#undef CKF_X
      sum += ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncthreads();  // red[] (max) consumed
    if (l == 0) red[w] = sum;
    __syncthreads();
    float S = 0.f;
#pragma unroll
    for (int k = 0; k < kXentPipeThreads / 32; ++k) S += red[k];
    const float lse = M + __logf(S);
    const int y = labels[r];
    if (threadIdx.x == 0) {
      uint16_t hy;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(hy) : "r"(base + 2u * static_cast<uint32_t>(y)));
      row_loss[r] = static_cast<double>(lse) - static_cast<double>(__uint_as_float(static_cast<uint32_t>(hy) << 16));
    }
    if (grad) {
      const float Ll = lse * kL2e;
      uint4* dst = reinterpret_cast<uint4*>(logits + static_cast<size_t>(r) * V);
      for (int c = threadIdx.x; c < V8; c += kXentPipeThreads) {
        const uint4 u = sm100::ld_shared_v4(base + 16 * c);
        const uint32_t q[4] = {u.x, u.y, u.z, u.w};
        uint32_t o[4];
        float p8[8];
#define CKF_X(E) p8[E] = ex2_mufu(fmaf(__uint_as_float((E & 1) ? (q[E / 2] & 0xffff0000u) : (q[E / 2] << 16)), kL2e, -Ll));
        CKF_X(0) CKF_X(1) CKF_X(2) CKF_X(3) CKF_X(4) CKF_X(5) CKF_X(6) CKF_X(7)
#undef CKF_X
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = 8 * c + 2 * e;
          const float g0 = (p8[2 * e] - (j == y ? 1.f : 0.f)) * gscale;
          const float g1 = (p8[2 * e + 1] - (j + 1 == y ? 1.f : 0.f)) * gscale;
          const __nv_bfloat162 b = __floats2bfloat162_rn(g0, g1);
          o[e] = *reinterpret_cast<const uint32_t*>(&b);
        }
        dst[c] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
    __syncthreads();  // buffer i & 1 and red[] free
    if (threadIdx.x == 0) issue(i + 2);
  }
}

__global__ void fold_mean_kernel(const double* __restrict__ v, size_t n, double scale, double* __restrict__ out) {
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < n; i += 1024) acc += v[i];
  acc = block_sum<double, 1024>(acc);
  if (threadIdx.x == 0) *out = acc * scale;
}

__global__ void split_tokens_kernel(const int* __restrict__ x, size_t rows, size_t T, int* __restrict__ tok,
                                    int* __restrict__ lab) {
  const size_t n = rows * T;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / T, j = i % T;
    tok[i] = x[r * (T + 1) + j];
    lab[i] = x[r * (T + 1) + j + 1];
  }
}

__global__ void f2bf_kernel(const float4* __restrict__ x, __nv_bfloat162* __restrict__ y, size_t n4) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    y[2 * i] = __floats2bfloat162_rn(v.x, v.y);
    y[2 * i + 1] = __floats2bfloat162_rn(v.z, v.w);
  }
}

unsigned blocks_for_rows(size_t rows) { return static_cast<unsigned>((rows + kWarpsPerBlock - 1) / kWarpsPerBlock); }

void need_d(size_t d) {
  if (d % 128 != 0 || d > 4096) raise(1, "LLaMA model_dim must be a multiple of 128 and <= 4096");
}

}  // namespace

void embed_fwd(const int* tok, size_t ntok, const float* E, size_t d, float* h, cudaStream_t s) {
  need_d(d);
  embed_fwd_kernel<<<blocks_for_rows(ntok), 32 * kWarpsPerBlock, 0, s>>>(
      tok, ntok, reinterpret_cast<const float4*>(E), d / 4, reinterpret_cast<float4*>(h));
  CKF_LAUNCH_CHECK();
}

size_t embed_bwd_scratch(size_t ntok) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<int>(ntok));
  return temp + 3 * ntok * sizeof(int) + 1024;
}

void embed_bwd(const int* tok, size_t ntok, const float* dh, size_t d, float* gE, void* scratch, cudaStream_t s) {
  need_d(d);
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<int>(ntok));
  char* p = static_cast<char*>(scratch);
  int* keys = reinterpret_cast<int*>(p);
  int* vin = keys + ntok;
  int* vout = vin + ntok;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(vout + ntok) + 255) & ~uintptr_t(255));
  iota_kernel<<<static_cast<unsigned>((ntok + 255) / 256), 256, 0, s>>>(vin, ntok);
  CKF_LAUNCH_CHECK();
  CKF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, temp, tok, keys, vin, vout, static_cast<int>(ntok), 0, 32, s));
  embed_bwd_kernel<<<blocks_for_rows(ntok), 32 * kWarpsPerBlock, 0, s>>>(
      keys, vout, ntok, reinterpret_cast<const float4*>(dh), d / 4, reinterpret_cast<float4*>(gE));
  CKF_LAUNCH_CHECK();
}

template <int V4>
void rmsnorm_fwd_t(const float* x, const float* g, size_t rows, bf16* y, float* rstd, float* xcopy, cudaStream_t s) {
  rmsnorm_fwd_kernel<V4><<<blocks_for_rows(rows), 32 * kWarpsPerBlock, 0, s>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(g), rows,
      reinterpret_cast<__nv_bfloat162*>(y), rstd, reinterpret_cast<float4*>(xcopy));
  CKF_LAUNCH_CHECK();
}

void rmsnorm_fwd(const float* x, const float* g, size_t rows, size_t d, bf16* y, float* rstd, float* xcopy,
                 cudaStream_t s) {
  need_d(d);
  switch (d / 128) {
    case 1: return rmsnorm_fwd_t<1>(x, g, rows, y, rstd, xcopy, s);
    case 2: return rmsnorm_fwd_t<2>(x, g, rows, y, rstd, xcopy, s);
    case 3: return rmsnorm_fwd_t<3>(x, g, rows, y, rstd, xcopy, s);
    case 4: return rmsnorm_fwd_t<4>(x, g, rows, y, rstd, xcopy, s);
    case 6: return rmsnorm_fwd_t<6>(x, g, rows, y, rstd, xcopy, s);
    case 8: return rmsnorm_fwd_t<8>(x, g, rows, y, rstd, xcopy, s);
    case 12: return rmsnorm_fwd_t<12>(x, g, rows, y, rstd, xcopy, s);
    case 16: return rmsnorm_fwd_t<16>(x, g, rows, y, rstd, xcopy, s);
    case 24: return rmsnorm_fwd_t<24>(x, g, rows, y, rstd, xcopy, s);
    case 32: return rmsnorm_fwd_t<32>(x, g, rows, y, rstd, xcopy, s);
    default: raise(1, "LLaMA model_dim / 128 must be one of 1,2,3,4,6,8,12,16,24,32");
  }
}

// Persistent grid: two 256-thread blocks per SM (one at d > 512, where the kernel's launch bounds
// allow one), so the gain partials the fold reads are 2 x #SMs rows of d, not one per 16 rows
// (8 MB -> 1.2 MB per launch at 32,768 x 1,024; the fold 8.6 -> ~3 us)
int rmsnorm_bwd_blocks(size_t rows) {
  static const int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  const size_t want = (rows + kBwdRowsPerBlock - 1) / kBwdRowsPerBlock;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(want, static_cast<size_t>(2 * sms))));
}

template <int V4>
void rmsnorm_bwd_t(const float* dy, const float* x, const float* g, const float* rstd, size_t rows, float* dh,
                   bf16* dh_bf, float* gpart, cudaStream_t s) {
  const size_t smem = (kWarpsPerBlock + 1) * V4 * 32 * sizeof(float4);  // partials + gains
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(rmsnorm_bwd_kernel<V4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    attr = true;
  }
  rmsnorm_bwd_kernel<V4><<<rmsnorm_bwd_blocks(rows), 32 * kWarpsPerBlock, smem, s>>>(
      reinterpret_cast<const float4*>(dy), reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(g),
      rstd, rows, reinterpret_cast<float4*>(dh), reinterpret_cast<__nv_bfloat162*>(dh_bf), gpart);
  CKF_LAUNCH_CHECK();
}

void rmsnorm_bwd(const float* dy, const float* x, const float* g, const float* rstd, size_t rows, size_t d, float* dh,
                 bf16* dh_bf, float* gpart, cudaStream_t s) {
  need_d(d);
  switch (d / 128) {
    case 1: return rmsnorm_bwd_t<1>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 2: return rmsnorm_bwd_t<2>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 3: return rmsnorm_bwd_t<3>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 4: return rmsnorm_bwd_t<4>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 6: return rmsnorm_bwd_t<6>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 12: return rmsnorm_bwd_t<12>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 24: return rmsnorm_bwd_t<24>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 8: return rmsnorm_bwd_t<8>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 16: return rmsnorm_bwd_t<16>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    case 32: return rmsnorm_bwd_t<32>(dy, x, g, rstd, rows, dh, dh_bf, gpart, s);
    default: raise(1, "LLaMA model_dim / 128 must be one of 1,2,3,4,6,8,12,16,24,32");
  }
}

void gain_fold(const float* gpart, int nblk, size_t d, float* gg, cudaStream_t s) {
  gain_fold_kernel<<<static_cast<unsigned>((d + kFoldCols - 1) / kFoldCols), kFoldCols * kFoldSlices, 0, s>>>(
      gpart, nblk, static_cast<int>(d), gg);
  CKF_LAUNCH_CHECK();
}

static const float2* rope_table_impl(size_t T, size_t hd, int pair_major, cudaStream_t s) {
  // per-(T, hd, layout) cos/sin table, built once per device
  struct Tab {
    size_t T, hd;
    int pm, dev;
    float2* p;
  };
  static std::vector<Tab> tabs;
  int dev = 0;
  CKF_CUDA(cudaGetDevice(&dev));
  for (auto& t : tabs)
    if (t.T == T && t.hd == hd && t.pm == pair_major && t.dev == dev) return t.p;
  float2* tab = nullptr;
  CKF_CUDA(cudaMalloc(&tab, T * hd / 2 * sizeof(float2)));
  ++alloc_epoch();
  rope_table_kernel<<<static_cast<unsigned>((T * hd / 2 + 255) / 256), 256, 0, s>>>(tab, static_cast<int>(T),
                                                                                   static_cast<int>(hd), pair_major);
  CKF_LAUNCH_CHECK();
  tabs.push_back({T, hd, pair_major, dev, tab});
  return tab;
}

const float2* rope_table(size_t T, size_t hd, cudaStream_t s) { return rope_table_impl(T, hd, 0, s); }
const float2* rope_table_pair_major(size_t T, size_t hd, cudaStream_t s) { return rope_table_impl(T, hd, 1, s); }

void rope(bf16* qkv, size_t ntok, size_t T, size_t d, size_t heads, int inverse, cudaStream_t s) {
  const size_t hd = d / heads;
  if (hd % 8) raise(1, "head_dim must be a multiple of 8 for RoPE");
  const float2* tab = rope_table(T, hd, s);
  const size_t items = ntok * (2 * d / 8);
  if (items >= (1ull << 32)) raise(1, "rope: too many tokens in one call");
  rope_kernel<<<grid_for(items, 256), 256, 0, s>>>(qkv, tab, static_cast<int>(ntok), static_cast<int>(T),
                                                   static_cast<int>(d), static_cast<int>(hd), inverse);
  CKF_LAUNCH_CHECK();
}

void swiglu_fwd(const bf16* gu, size_t ntok, size_t f, bf16* a, cudaStream_t s) {
  if (f % 8) raise(1, "ffn width must be a multiple of 8");
  if (ntok * f / 8 >= (1ull << 32)) raise(1, "swiglu: microbatch too large");
  swiglu_fwd_kernel<<<grid_for(ntok * f / 8, 256), 256, 0, s>>>(gu, static_cast<int>(ntok), static_cast<int>(f), a);
  CKF_LAUNCH_CHECK();
}

void swiglu_bwd(const bf16* gu, const bf16* da, size_t ntok, size_t f, bf16* dgu, cudaStream_t s) {
  if (f % 8) raise(1, "ffn width must be a multiple of 8");
  swiglu_bwd_kernel<<<grid_for(ntok * f / 8, 256), 256, 0, s>>>(gu, da, static_cast<int>(ntok), static_cast<int>(f),
                                                                 dgu);
  CKF_LAUNCH_CHECK();
}

void xent_bf16(bf16* logits, const int* labels, size_t rows, size_t V, float grad_scale, int grad, double* row_loss,
               cudaStream_t s) {
  if (rows == 0) return;
  const size_t v8 = V / 8, per = (v8 + kXentThreads - 1) / kXentThreads;
  const int vi = static_cast<int>(V);
  const size_t pipe_smem = 2 * ((V * 2 + 127) / 128 * 128) + 16 + 64 + 128;
  if (V % 8 == 0 && pipe_smem <= 227 * 1024 && rows < (1u << 31)) {
    static int sms = 0;
    static size_t attr = 0;
    if (!sms) {
      int dev = 0;
      CKF_CUDA(cudaGetDevice(&dev));
      CKF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (pipe_smem > attr) {
      CKF_CUDA(cudaFuncSetAttribute(xent_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(pipe_smem)));
      attr = pipe_smem;
    }
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(rows, static_cast<size_t>(sms)));
    xent_pipe_kernel<<<grid, kXentPipeThreads, pipe_smem, s>>>(logits, labels, static_cast<int>(rows), vi, grad_scale,
                                                             grad, row_loss);
    CKF_LAUNCH_CHECK();
    return;
  }
  if (V % 8 == 0 && per <= 16) {
#define CKF_XENT_CASE(N)                                                                                          \
  if (per <= N) {                                                                                                  \
    xent_reg_kernel<N><<<static_cast<unsigned>(rows), kXentThreads, 0, s>>>(logits, labels, vi, grad_scale, grad, \
                                                                         row_loss);                               \
    CKF_LAUNCH_CHECK();                                                                                            \
    return;                                                                                                        \
  }
    CKF_XENT_CASE(1) CKF_XENT_CASE(2) CKF_XENT_CASE(4) CKF_XENT_CASE(8) CKF_XENT_CASE(13) CKF_XENT_CASE(16)
#undef CKF_XENT_CASE
  }
  xent_kernel<<<static_cast<unsigned>(rows), kXentThreads, 0, s>>>(logits, labels, V, grad_scale, grad, row_loss);
  CKF_LAUNCH_CHECK();
}

void fold_mean(const double* row_loss, size_t rows, double scale, double* out, cudaStream_t s) {
  fold_mean_kernel<<<1, 1024, 0, s>>>(row_loss, rows, scale, out);
  CKF_LAUNCH_CHECK();
}

void split_tokens(const int* x, size_t rows, size_t T, int* tok, int* lab, cudaStream_t s) {
  split_tokens_kernel<<<grid_for(rows * T, 256), 256, 0, s>>>(x, rows, T, tok, lab);
  CKF_LAUNCH_CHECK();
}

void f32_to_bf16(const float* x, bf16* y, size_t n, cudaStream_t s) {
  if (n % 4) raise(1, "f32_to_bf16 needs n % 4 == 0");
  f2bf_kernel<<<grid_for(n / 4, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x),
                                                    reinterpret_cast<__nv_bfloat162*>(y), n / 4);
  CKF_LAUNCH_CHECK();
}

}  // namespace ckf::llama
