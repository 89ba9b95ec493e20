// Causal attention forward on the 5th-generation tensor cores (hd = 64).
//
// One CTA per (128-query tile, sequence x head).  Q, K, V tiles arrive by TMA
// straight from the packed qkv activation (one 2-D tensor map, box 64 x 128,
// 128-byte swizzle: K-major for Q and K, MN-major for V as the PV B operand).
// S = Q K^T is accumulated in TMEM (double-buffered, 2 x 128 columns),
// softmax runs one query row per thread of the 4 softmax warps (tcgen05.ld),
// P is written back to swizzled shared memory as the A operand of O += P V,
// whose fp32 accumulator also lives in TMEM (64 columns).
//
// Two passes over the key tiles: pass 1 computes the row max / sum (log-sum-
// exp), pass 2 recomputes S and accumulates O with P = exp(S - lse) already
// normalised -- no accumulator rescaling, so the tensor core never waits for
// a TMEM read-modify-write.  Costs one extra Q K^T per tile (+50 % MMA work).
//
// Warp roles (256 threads): 0 TMA producer, 1 MMA issuer (one lane),
// 2 TMEM allocator, 4..7 softmax / epilogue (query row = 32 (w-4) + lane).
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "llama_kernels.h"
#include "sm100.cuh"

namespace ckf::llama {
namespace {

using namespace ckf::sm100;

constexpr int TQ = 128, TK = 128, HD = 64;
constexpr int kThreads = 256;
constexpr int kThreadsBwd = 384;  // backward: 8 softmax warps (2 per TMEM lane quarter, column halves)
constexpr uint32_t kTile = TQ * HD * 2;      // 16 KiB: one 128 x 64 bf16 tile
constexpr uint32_t kPBuf = TQ * TK * 2;      // 32 KiB: P as [2 K-chunks][128 rows][128 B]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Forward (single pass, FA4-style lazy rescaling).  128 queries x 64-key tiles:
// S double-buffered in TMEM (2 x 64 columns) + O (64 columns) = 256 columns and
// 104 KiB of shared memory per CTA -> two CTAs per SM.  Each softmax thread owns
// one query row: running max m (log2 domain) and sum l; P = exp2(S*scale - m)
// is written to swizzled smem for O += P V.  m is only raised when a tile's max
// exceeds it by more than kRescale (P stays <= 2^kRescale, exact in bf16 range);
// then the thread rescales its O row in TMEM (tcgen05.ld/st) after the previous
// P V has completed.  K and V are each loaded once.
constexpr int FK = 64;                        // keys per forward tile
constexpr uint32_t kKTile = FK * HD * 2;      // 8 KiB (64 keys x 64 hd)
constexpr uint32_t kPTile = TQ * FK * 2;      // 16 KiB: P [128 rows][128 B]
constexpr int kKStages = 4, kVStages = 3;
constexpr float kRescale = 8.f;

struct Smem {
  uint8_t q[kTile];
  uint8_t k[kKStages][kKTile];
  uint8_t v[kVStages][kKTile];
  uint8_t p[2][kPTile];
  uint64_t q_full;
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], s_free[2], p_full[2], p_free[2];
  uint64_t o_full;
  uint32_t tmem;
};

__device__ __forceinline__ void tmem_st32_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_kv,
                       int T, int H, __nv_bfloat16* __restrict__ o, float* __restrict__ lse, float scale_log2,
                       long long* __restrict__ dbg) {
  extern __shared__ uint8_t smem_raw[];
  const long long t_start = clock64();
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);  // heavy (late) query tiles first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int nkb = 2 * qb + 2;  // causal: 64-key tiles 0 .. 2qb+1
  const int row0 = b * T;
  const int qcol = h * HD, kcol = (H + h) * HD, vcol = (2 * H + h) * HD;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_kv);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], 4);
      mbar_init(&sm.p_full[i], 4);
      mbar_init(&sm.p_free[i], 1);
    }
    mbar_init(&sm.o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<256>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S[0] cols 0-63, S[1] 64-127, O 128-191

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: Q once, then K_j and V_j (each exactly once)
      mbar_arrive_expect_tx(&sm.q_full, kTile);
      tma_load_2d(sm.q, &tm_qkv, &sm.q_full, qcol, row0 + qb * TQ);
      for (int j = 0; j < nkb; ++j) {
        const int ks = j % kKStages, vs = j % kVStages;
        mbar_wait(&sm.k_empty[ks], ((j / kKStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.k_full[ks], kKTile);
        tma_load_2d(sm.k[ks], &tm_kv, &sm.k_full[ks], kcol, row0 + j * FK);
        mbar_wait(&sm.v_empty[vs], ((j / kVStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.v_full[vs], kKTile);
        tma_load_2d(sm.v[vs], &tm_kv, &sm.v_full[vs], vcol, row0 + j * FK);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: S_{j+1} is issued before P_j is awaited
      constexpr uint32_t kIdS = idesc_bf16_f32(TQ, FK, false, false);  // S = Q K^T  (128 x 64)
      constexpr uint32_t kIdO = idesc_bf16_f32(TQ, HD, false, true);   // O += P V   (V MN-major)
      mbar_wait(&sm.q_full, 0);
      const uint32_t qa = smem_u32(sm.q);
      auto issue_s = [&](int j) {
        const int ks = j % kKStages, sb = j & 1;
        mbar_wait(&sm.k_full[ks], (j / kKStages) & 1);
        mbar_wait(&sm.s_free[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sm.k[ks]);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + sb * FK, umma_desc_sw128(qa + k * 32, 16, 1024), umma_desc_sw128(ka + k * 32, 16, 1024),
                    kIdS, k > 0 ? 1u : 0u);
        umma_commit(&sm.s_full[sb]);
        umma_commit(&sm.k_empty[ks]);
      };
      issue_s(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) issue_s(j + 1);
        const int pb = j & 1, vs = j % kVStages;
        mbar_wait(&sm.v_full[vs], (j / kVStages) & 1);
        mbar_wait(&sm.p_full[pb], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(sm.p[pb]), va = smem_u32(sm.v[vs]);
#pragma unroll
        for (int k = 0; k < FK / 16; ++k)
          umma_bf16(tmem + 128, umma_desc_sw128(pa + k * 32, 16, 1024), umma_desc_sw128(va + k * 2048, 8192, 1024),
                    kIdO, (j > 0 || k > 0) ? 1u : 0u);
        umma_commit(&sm.p_free[pb]);
        umma_commit(&sm.v_empty[vs]);
      }
      umma_commit(&sm.o_full);
    }
  } else if (warp >= 4) {
    // ---------------- softmax: one query row per thread, online with lazy rescaling
    const int r = (warp - 4) * 32 + lane;
    const int q = qb * TQ + r;
    const uint32_t trow = tmem + (static_cast<uint32_t>((warp - 4) * 32) << 16);
    float m = -INFINITY, l = 0.f;  // m: running max of S * scale_log2
    long long w_s = 0, w_p = 0, t_first = 0;
    for (int j = 0; j < nkb; ++j) {
      const int sb = j & 1, pb = j & 1;
      const long long t0 = clock64();
      mbar_wait(&sm.s_full[sb], (j >> 1) & 1);
      const long long t1 = clock64();
      if (j == 0) t_first = t1 - t_start;
      w_s += t1 - t0;
      tc_fence_after();
      uint32_t u[64];
      tmem_ld32(trow + sb * FK, *reinterpret_cast<uint32_t(*)[32]>(&u[0]));
      tmem_ld32(trow + sb * FK + 32, *reinterpret_cast<uint32_t(*)[32]>(&u[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.s_free[sb]);
      const int kbase = j * FK;
      const int nvalid = min(FK, q - kbase + 1);  // keys <= q are visible (causal)
      // row max of the visible scores: 8 independent chains (no 64-deep FMNMX dependency)
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
      if (nvalid >= FK) {
#pragma unroll
        for (int t = 0; t < FK; ++t) mx8[t & 7] = fmaxf(mx8[t & 7], __uint_as_float(u[t]));
      } else {
#pragma unroll
        for (int t = 0; t < FK; ++t)
          if (t < nvalid) mx8[t & 7] = fmaxf(mx8[t & 7], __uint_as_float(u[t]));
      }
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * scale_log2;
      // lazy rescale: only when this tile's max exceeds the running max by > kRescale
      const bool need = mx > m + kRescale;
      const float mn = need ? mx : m;
      const float alpha = need ? ex2(m - mn) : 1.f;  // m = -inf on the first tile -> 0
      if (__any_sync(0xffffffffu, need) && j > 0) {
        // the previous P V must have landed before this warp rewrites its O rows
        mbar_wait(&sm.p_free[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t ov[32];
          tmem_ld32(trow + 128 + hf * 32, ov);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) ov[t] = __float_as_uint(__uint_as_float(ov[t]) * alpha);
          tmem_st32(trow + 128 + hf * 32, ov);
        }
        tmem_st32_wait();
      }
      l *= alpha;
      m = mn;
      const long long t2 = clock64();
      mbar_wait(&sm.p_free[pb], ((j >> 1) & 1) ^ 1);  // P V_{j-2} has read this P buffer
      w_p += clock64() - t2;
      const uint32_t prow = smem_u32(sm.p[pb]) + r * 128;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // 32 keys at a time: P -> bf16 -> swizzled smem
        uint32_t w[16];
        float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          const int tt = hf * 32 + t;
          float p0 = ex2(fmaf(__uint_as_float(u[tt]), scale_log2, -m));
          float p1 = ex2(fmaf(__uint_as_float(u[tt + 1]), scale_log2, -m));
          if (nvalid < FK) {
            p0 = tt < nvalid ? p0 : 0.f;
            p1 = tt + 1 < nvalid ? p1 : 0.f;
          }
          l4[(t >> 1) & 3] += p0 + p1;
          w[t / 2] = pack_bf16(p0, p1);
        }
        l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
#pragma unroll
        for (int pc = 0; pc < 4; ++pc)
          st_shared_v4(prow + (((hf * 4 + pc) ^ (r & 7)) << 4), w[4 * pc], w[4 * pc + 1], w[4 * pc + 2],
                       w[4 * pc + 3]);
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[pb]);
    }
    // ---------------- epilogue: O / l -> bf16, lse
    mbar_wait(&sm.o_full, 0);
    tc_fence_after();
    const float inv = 1.f / l;
    const size_t ldo = static_cast<size_t>(H) * HD;
    __nv_bfloat16* orow = o + (static_cast<size_t>(row0) + q) * ldo + static_cast<size_t>(h) * HD;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      uint32_t u[32];
      tmem_ld32(trow + 128 + hf * 32, u);
      tmem_ld_wait();
#pragma unroll
      for (int piece = 0; piece < 4; ++piece) {
        uint4 v;
        v.x = pack_bf16(__uint_as_float(u[8 * piece + 0]) * inv, __uint_as_float(u[8 * piece + 1]) * inv);
        v.y = pack_bf16(__uint_as_float(u[8 * piece + 2]) * inv, __uint_as_float(u[8 * piece + 3]) * inv);
        v.z = pack_bf16(__uint_as_float(u[8 * piece + 4]) * inv, __uint_as_float(u[8 * piece + 5]) * inv);
        v.w = pack_bf16(__uint_as_float(u[8 * piece + 6]) * inv, __uint_as_float(u[8 * piece + 7]) * inv);
        reinterpret_cast<uint4*>(orow + hf * 32)[piece] = v;
      }
    }
    lse[static_cast<size_t>(bh) * T + q] = (m + log2f(l)) * kLn2;
    if (dbg && threadIdx.x == 128) {
      long long* d = dbg + 8 * (blockIdx.y * gridDim.x + blockIdx.x);
      d[0] = nkb;
      d[1] = t_first;
      d[2] = w_s;
      d[3] = w_p;
      d[4] = clock64() - t_start;
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      d[5] = smid;
      d[6] = t_start;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<256>(tmem);
}

// ---------------------------------------------------------------- backward
// D[bh*T + q] = sum_c dO[q, c] O[q, c]   (one warp per (token, head))
__global__ void dsum_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout, int B, int T,
                            int H, float* __restrict__ D) {
  // 8 lanes per (token, head), 16-byte loads: a warp covers 4 (token, head) rows
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  const long long row = i >> 3;
  const int part = static_cast<int>(i & 7);
  const bool live = row < static_cast<long long>(B) * T * H;
  float acc = 0.f;
  if (live) {
    const size_t off = static_cast<size_t>(row) * HD + 8 * part;  // o / dout are [tok][H][HD]: row index = tok * H + h
    const uint4 a = *reinterpret_cast<const uint4*>(o + off);
    const uint4 d = *reinterpret_cast<const uint4*>(dout + off);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pd = reinterpret_cast<const __nv_bfloat162*>(&d);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 x = __bfloat1622float2(pa[q]), y = __bfloat1622float2(pd[q]);
      acc += x.x * y.x + x.y * y.y;
    }
  }
#pragma unroll
  for (int s = 4; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (live && part == 0) {
    const long long tok = row / H;
    const int h = static_cast<int>(row % H);
    const int b = static_cast<int>(tok / T), q = static_cast<int>(tok % T);
    D[(static_cast<size_t>(b) * H + h) * T + q] = acc;
  }
}

// Inverse rotary rotation of one 64-wide head row (pairs (j, j + 32)), in place on fp32
// values: the transpose of the forward rotation (llama_kernels.cu rope_kernel, inverse = 1).
__device__ __forceinline__ void rope_inverse64(uint32_t (&v)[64], const float2* __restrict__ cs) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float2 t = __ldg(cs + j);
    const float a = __uint_as_float(v[j]), b = __uint_as_float(v[j + 32]);
    v[j] = __float_as_uint(a * t.x + b * t.y);
    v[j + 32] = __float_as_uint(b * t.x - a * t.y);
  }
}

// Both backward kernels are persistent (one CTA per SM) over work units sorted
// longest-first.  K/V (dK dV kernel) or Q/dO (dQ kernel) of a unit are
// double-buffered in shared memory and the TMEM accumulators are double-
// buffered (two sets), so a unit's set-up (operand loads, first S) and its
// epilogue (TMEM -> global) overlap the neighbouring unit's tiles instead of
// being paid once per CTA launch.  Tile / unit counters run across units, so
// every mbarrier keeps a single phase sequence.
struct SmemKV {  // dK / dV kernel
  uint8_t k[2][kTile], v[2][kTile];
  uint8_t q[2][kTile], d_o[2][kTile];
  uint8_t p[kPBuf], ds[kPBuf];
  float lse[2][TQ], dsum[2][TQ];  // per-query lse / D of the tile, bulk-copied with its Q / dO
  uint64_t kv_full[2], kv_empty[2], qd_full[2], qd_empty[2], s_full, s_free, pd_full, pd_free, acc_full[2],
      acc_free[2];
  uint32_t tmem;
};

// Unit u = (key tile kb, sequence x head bh), kb-major: kb = 0 (nqb query tiles) first.
//   S^T = K Q^T, dP^T = V dO^T (TMEM)  ->  P^T = exp(S^T - lse), dS^T = P^T (dP^T - D)  (softmax warps,
//   row = key)  ->  dV += P^T dO, dK += dS^T Q (TMEM accumulators, B operands MN-major from the tiles)
__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                        const float* __restrict__ lse, const float* __restrict__ D, int T, int H, int BH,
                        __nv_bfloat16* __restrict__ dqkv, float scale, float scale_log2, const float2* __restrict__ rope,
                        long long* __restrict__ dbg) {
  extern __shared__ uint8_t smem_raw[];
  const long long t_start = clock64();
  long long tw[6] = {0, 0, 0, 0, 0, 0};  // CKF_ATTN_DEBUG phase cycles (softmax warp 4 lane 0 / MMA lane)
  SmemKV& sm = *reinterpret_cast<SmemKV*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int nunits = nqb * BH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
      mbar_init(&sm.qd_full[i], 1);
      mbar_init(&sm.qd_empty[i], 1);
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 8);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_free, 8);
    mbar_init(&sm.pd_full, 8);
    mbar_init(&sm.pd_free, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S^T cols 0-127, dP^T 128-255, set 0: dV 256-319 dK 320-383, set 1: +128

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int kb = u / BH, bh = u - kb * BH, b = bh / H, h = bh - b * H;
        const int row0 = b * T;
        const int kbuf = lu & 1;
        mbar_wait(&sm.kv_empty[kbuf], ((lu >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.kv_full[kbuf], 2 * kTile);
        tma_load_2d(sm.k[kbuf], &tm_qkv, &sm.kv_full[kbuf], (H + h) * HD, row0 + kb * TK);
        tma_load_2d(sm.v[kbuf], &tm_qkv, &sm.kv_full[kbuf], (2 * H + h) * HD, row0 + kb * TK);
        for (int i = 0; i < nqb - kb; ++i, ++g) {
          const int st = g & 1;
          mbar_wait(&sm.qd_empty[st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.qd_full[st], 2 * kTile + 2 * TQ * 4);
          const int qrow = row0 + (kb + i) * TQ;
          tma_load_2d(sm.q[st], &tm_qkv, &sm.qd_full[st], h * HD, qrow);
          tma_load_2d(sm.d_o[st], &tm_do, &sm.qd_full[st], h * HD, qrow);
          const size_t qo = static_cast<size_t>(bh) * T + (kb + i) * TQ;
          bulk_load(sm.lse[st], lse + qo, TQ * 4, &sm.qd_full[st]);
          bulk_load(sm.dsum[st], D + qo, TQ * 4, &sm.qd_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_bf16_f32(TK, TQ, false, false);  // [keys x q], K = hd
      constexpr uint32_t kIdA = idesc_bf16_f32(TK, HD, false, true);   // [keys x hd], K = q, B MN-major
      const uint32_t pa = smem_u32(sm.p), da = smem_u32(sm.ds);
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int ntiles = nqb - u / BH;
        const int kbuf = lu & 1;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(kbuf * 128);
        mbar_wait(&sm.kv_full[kbuf], (lu >> 1) & 1);
        const uint32_t ka = smem_u32(sm.k[kbuf]), va = smem_u32(sm.v[kbuf]);
        auto issue_s = [&](int gi) {  // S^T = K Q^T, dP^T = V dO^T of global tile gi
          const int st = gi & 1;
          mbar_wait(&sm.qd_full[st], (gi >> 1) & 1);
          mbar_wait(&sm.s_free, (gi & 1) ^ 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            umma_bf16(tmem, umma_desc_sw128(ka + k * 32, 16, 1024), umma_desc_sw128(qa + k * 32, 16, 1024), kIdS,
                      k > 0 ? 1u : 0u);
            umma_bf16(tmem + 128, umma_desc_sw128(va + k * 32, 16, 1024), umma_desc_sw128(oa + k * 32, 16, 1024),
                      kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit(&sm.s_full);
        };
        long long c0_ = clock64();
        issue_s(g);  // overlaps the previous unit's epilogue
        long long c1_ = clock64();
        tw[0] += c1_ - c0_;
        mbar_wait(&sm.acc_free[kbuf], ((lu >> 1) & 1) ^ 1);  // this accumulator set was drained two units ago
        tw[1] += clock64() - c1_;
        for (int i = 0; i < ntiles; ++i) {
          const int gi = g + i, st = gi & 1;
          c0_ = clock64();
          if (i + 1 < ntiles) issue_s(gi + 1);
          c1_ = clock64();
          tw[0] += c1_ - c0_;
          mbar_wait(&sm.pd_full, gi & 1);
          tw[2] += clock64() - c1_;
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
#pragma unroll
          for (int k = 0; k < TQ / 16; ++k) {
            const uint32_t aoff = (k >> 2) * (128 * 128) + (k & 3) * 32;
            umma_bf16(acc, umma_desc_sw128(pa + aoff, 16, 1024), umma_desc_sw128(oa + k * 2048, 8192, 1024), kIdA,
                      (i > 0 || k > 0) ? 1u : 0u);
            umma_bf16(acc + 64, umma_desc_sw128(da + aoff, 16, 1024), umma_desc_sw128(qa + k * 2048, 8192, 1024),
                      kIdA, (i > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&sm.pd_free);
          umma_commit(&sm.qd_empty[st]);
        }
        umma_commit(&sm.acc_full[kbuf]);
        umma_commit(&sm.kv_empty[kbuf]);
        g += ntiles;
      }
      if (dbg) {
        long long* d = dbg + 16 * blockIdx.x + 8;
        d[0] = tw[0];  // issue_s incl. its qd_full / s_free waits
        d[1] = tw[1];  // acc_free waits
        d[2] = tw[2];  // pd_full waits
        d[3] = clock64() - t_start;
      }
    }
  } else if (warp >= 4) {
    const int sw = warp - 4, quarter = sw & 3, half = sw >> 2;
    const int r = quarter * 32 + lane;  // key row within the tile
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t pbase = smem_u32(sm.p), dbase = smem_u32(sm.ds);
    const size_t ld = static_cast<size_t>(3) * H * HD;
    // Unit epilogue (column half 0 -> dV, half 1 -> dK x scale), run one tile late: after the
    // first tile of the next unit, when the accumulator set has long been complete.
    auto epilogue = [&](int eu, int elu) {
      const int ekb = eu / BH, ebh = eu - ekb * BH, eb = ebh / H, eh = ebh - eb * H;
      const int aset = elu & 1;
      const long long e0 = clock64();
      mbar_wait(&sm.acc_full[aset], (elu >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* dst = dqkv + (static_cast<size_t>(eb) * T + ekb * TK + r) * ld +
                           static_cast<size_t>(half ? (H + eh) * HD : (2 * H + eh) * HD);
      const float mul = half ? scale : 1.f;
      uint32_t w32[64];
      tmem_ld32(trow + 256 + aset * 128 + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&w32[0]));
      tmem_ld32(trow + 256 + aset * 128 + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&w32[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
      if (half && rope) rope_inverse64(w32, rope + static_cast<size_t>(ekb * TK + r) * 32);  // dK
#pragma unroll
      for (int piece = 0; piece < 8; ++piece) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(w32[8 * piece + 0]) * mul, __uint_as_float(w32[8 * piece + 1]) * mul);
        w.y = pack_bf16(__uint_as_float(w32[8 * piece + 2]) * mul, __uint_as_float(w32[8 * piece + 3]) * mul);
        w.z = pack_bf16(__uint_as_float(w32[8 * piece + 4]) * mul, __uint_as_float(w32[8 * piece + 5]) * mul);
        w.w = pack_bf16(__uint_as_float(w32[8 * piece + 6]) * mul, __uint_as_float(w32[8 * piece + 7]) * mul);
        reinterpret_cast<uint4*>(dst)[piece] = w;
      }
      tw[3] += clock64() - e0;
    };
    int pend_u = -1, pend_lu = 0;
    int g = 0, lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      const int kb = u / BH;
      const int ntiles = nqb - kb;
      for (int i = 0; i < ntiles; ++i) {
        const int gi = g + i, st = gi & 1;
        const long long a0 = clock64();
        mbar_wait(&sm.s_full, gi & 1);
        mbar_wait(&sm.qd_full[st], (gi >> 1) & 1);  // (already complete) makes the bulk-copied lse / D visible
        tc_fence_after();
        const long long a1 = clock64();
        // this thread's 64 columns of S^T and dP^T in one go; the TMEM is released right away
        // so the next tile's S^T / dP^T MMAs start while P / dS are computed from registers
        uint32_t us[64], ud[64];
        tmem_ld32(trow + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&us[0]));
        tmem_ld32(trow + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&us[32]));
        tmem_ld32(trow + 128 + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&ud[0]));
        tmem_ld32(trow + 128 + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&ud[32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free);
        mbar_wait(&sm.pd_free, (gi & 1) ^ 1);  // the previous tile's dV/dK MMAs have read P / dS
        const long long a2 = clock64();
        tw[0] += a1 - a0;
        tw[1] += a2 - a1;
        const uint32_t rowoff = static_cast<uint32_t>(half * (128 * 128) + r * 128);
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {  // 8 columns (queries) at a time: P^T, dS^T -> bf16 -> swizzled smem
          const int c = half * 64 + 8 * g8;
          // broadcast 128-bit shared loads (explicit ld.shared: the struct reference is generic)
          const uint32_t la_ = smem_u32(&sm.lse[st][c]), da_ = smem_u32(&sm.dsum[st][c]);
          const uint4 la = ld_shared_v4(la_), lb = ld_shared_v4(la_ + 16);
          const uint4 da4 = ld_shared_v4(da_), db4 = ld_shared_v4(da_ + 16);
          const float lq[8] = {__uint_as_float(la.x), __uint_as_float(la.y), __uint_as_float(la.z),
                               __uint_as_float(la.w), __uint_as_float(lb.x), __uint_as_float(lb.y),
                               __uint_as_float(lb.z), __uint_as_float(lb.w)};
          const float dq8[8] = {__uint_as_float(da4.x), __uint_as_float(da4.y), __uint_as_float(da4.z),
                                __uint_as_float(da4.w), __uint_as_float(db4.x), __uint_as_float(db4.y),
                                __uint_as_float(db4.z), __uint_as_float(db4.w)};
          float pv[8], dv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float p = ex2(fmaf(__uint_as_float(us[8 * g8 + e]), scale_log2, -lq[e] * kLog2e));
            pv[e] = p;
            dv[e] = p * (__uint_as_float(ud[8 * g8 + e]) - dq8[e]);
          }
          if (i == 0) {  // diagonal tile: a query before the key sees nothing
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (c + e < r) pv[e] = dv[e] = 0.f;
          }
          const uint32_t off = rowoff + ((g8 ^ (r & 7)) << 4);
          st_shared_v4(pbase + off, pack_bf16(pv[0], pv[1]), pack_bf16(pv[2], pv[3]), pack_bf16(pv[4], pv[5]),
                       pack_bf16(pv[6], pv[7]));
          st_shared_v4(dbase + off, pack_bf16(dv[0], dv[1]), pack_bf16(dv[2], dv[3]), pack_bf16(dv[4], dv[5]),
                       pack_bf16(dv[6], dv[7]));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pd_full);
        tw[2] += clock64() - a2;
        tw[4] += 1;
        if (i == 0 && pend_u >= 0) {
          epilogue(pend_u, pend_lu);
          pend_u = -1;
        }
      }
      g += ntiles;
      pend_u = u;
      pend_lu = lu;
    }
    if (pend_u >= 0) epilogue(pend_u, pend_lu);
    if (dbg && threadIdx.x == 128) {
      long long* d = dbg + 16 * blockIdx.x;
      d[0] = tw[4];  // tiles
      d[1] = tw[0];  // s_full waits
      d[2] = tw[1];  // pd_free waits
      d[3] = tw[2];  // softmax compute + P/dS stores
      d[4] = tw[3];  // unit epilogues (incl. acc_full waits)
      d[5] = clock64() - t_start;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<512>(tmem);
}

struct SmemQ {  // dQ kernel
  uint8_t q[2][kTile], d_o[2][kTile];
  uint8_t k[2][kTile], v[2][kTile];
  uint8_t ds[kPBuf];
  float lse[2][TQ], dsum[2][TQ];  // per-query lse / D of the unit, bulk-copied with its Q / dO
  uint64_t qd_full[2], qd_empty[2], kv_full[2], kv_empty[2], s_full, s_free, ds_full, ds_free, acc_full[2],
      acc_free[2];
  uint32_t tmem;
};

// Unit u = (query tile qb, sequence x head bh), longest (qb = nqb - 1) first.
//   S = Q K^T, dP = dO V^T (TMEM) -> dS = P (dP - D) (softmax warps, row = query) -> dQ += dS K
__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_dq_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const float* __restrict__ lse, const float* __restrict__ D, int T, int H, int BH,
                      __nv_bfloat16* __restrict__ dqkv, float scale, float scale_log2, const float2* __restrict__ rope) {
  extern __shared__ uint8_t smem_raw[];
  SmemQ& sm = *reinterpret_cast<SmemQ*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int nunits = nqb * BH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.qd_full[i], 1);
      mbar_init(&sm.qd_empty[i], 1);
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 8);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_free, 8);
    mbar_init(&sm.ds_full, 8);
    mbar_init(&sm.ds_free, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S cols 0-127, dP 128-255, dQ set 0: 256-319, set 1: 320-383

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int qi = u / BH, bh = u - qi * BH, b = bh / H, h = bh - b * H;
        const int qb = nqb - 1 - qi, row0 = b * T;
        const int qbuf = lu & 1;
        mbar_wait(&sm.qd_empty[qbuf], ((lu >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.qd_full[qbuf], 2 * kTile + 2 * TQ * 4);
        tma_load_2d(sm.q[qbuf], &tm_qkv, &sm.qd_full[qbuf], h * HD, row0 + qb * TQ);
        tma_load_2d(sm.d_o[qbuf], &tm_do, &sm.qd_full[qbuf], h * HD, row0 + qb * TQ);
        const size_t qo = static_cast<size_t>(bh) * T + qb * TQ;
        bulk_load(sm.lse[qbuf], lse + qo, TQ * 4, &sm.qd_full[qbuf]);
        bulk_load(sm.dsum[qbuf], D + qo, TQ * 4, &sm.qd_full[qbuf]);
        for (int j = 0; j <= qb; ++j, ++g) {
          const int st = g & 1;
          mbar_wait(&sm.kv_empty[st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.kv_full[st], 2 * kTile);
          tma_load_2d(sm.k[st], &tm_qkv, &sm.kv_full[st], (H + h) * HD, row0 + j * TK);
          tma_load_2d(sm.v[st], &tm_qkv, &sm.kv_full[st], (2 * H + h) * HD, row0 + j * TK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_bf16_f32(TQ, TK, false, false);  // [q x keys], K = hd
      constexpr uint32_t kIdQ = idesc_bf16_f32(TQ, HD, false, true);   // [q x hd], K = keys, B MN-major
      const uint32_t da = smem_u32(sm.ds);
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int nkb = nqb - u / BH;  // qb + 1
        const int qbuf = lu & 1;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(qbuf * 64);
        mbar_wait(&sm.qd_full[qbuf], (lu >> 1) & 1);
        const uint32_t qa = smem_u32(sm.q[qbuf]), oa = smem_u32(sm.d_o[qbuf]);
        auto issue_s = [&](int gj) {  // S = Q K^T, dP = dO V^T of global tile gj
          const int st = gj & 1;
          mbar_wait(&sm.kv_full[st], (gj >> 1) & 1);
          mbar_wait(&sm.s_free, (gj & 1) ^ 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sm.k[st]), va = smem_u32(sm.v[st]);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            umma_bf16(tmem, umma_desc_sw128(qa + k * 32, 16, 1024), umma_desc_sw128(ka + k * 32, 16, 1024), kIdS,
                      k > 0 ? 1u : 0u);
            umma_bf16(tmem + 128, umma_desc_sw128(oa + k * 32, 16, 1024), umma_desc_sw128(va + k * 32, 16, 1024),
                      kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit(&sm.s_full);
        };
        issue_s(g);
        mbar_wait(&sm.acc_free[qbuf], ((lu >> 1) & 1) ^ 1);
        for (int j = 0; j < nkb; ++j) {
          const int gj = g + j, st = gj & 1;
          if (j + 1 < nkb) issue_s(gj + 1);  // overlaps the softmax warps' dS of tile j
          mbar_wait(&sm.ds_full, gj & 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sm.k[st]);
#pragma unroll
          for (int k = 0; k < TK / 16; ++k)
            umma_bf16(acc, umma_desc_sw128(da + (k >> 2) * (128 * 128) + (k & 3) * 32, 16, 1024),
                      umma_desc_sw128(ka + k * 2048, 8192, 1024), kIdQ, (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&sm.ds_free);
          umma_commit(&sm.kv_empty[st]);
        }
        umma_commit(&sm.acc_full[qbuf]);
        umma_commit(&sm.qd_empty[qbuf]);
        g += nkb;
      }
    }
  } else if (warp >= 4) {
    const int sw = warp - 4, quarter = sw & 3, half = sw >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t dbase = smem_u32(sm.ds);
    const size_t ld = static_cast<size_t>(3) * H * HD;
    // unit epilogue (dQ x scale), run one tile late like the dK / dV kernel's
    auto epilogue = [&](int eu, int elu) {
      const int eqi = eu / BH, ebh = eu - eqi * BH, eb = ebh / H, eh = ebh - eb * H;
      const int eq = (nqb - 1 - eqi) * TQ + r;
      const int aset = elu & 1;
      mbar_wait(&sm.acc_full[aset], (elu >> 1) & 1);
      tc_fence_after();
      // the column-half-0 warps write the whole 64-wide row (the rotary pairs (j, j + 32) span both
      // halves), 16 pairs at a time
      __nv_bfloat16* qrow = dqkv + (static_cast<size_t>(eb) * T + eq) * ld + static_cast<size_t>(eh * HD);
      if (!rope) {  // no rotation: each column half writes its own 32 columns
        uint32_t w32[32];
        tmem_ld32(trow + 256 + aset * 64 + half * 32, w32);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
#pragma unroll
        for (int piece = 0; piece < 4; ++piece) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(w32[8 * piece + 0]) * scale, __uint_as_float(w32[8 * piece + 1]) * scale);
          w.y = pack_bf16(__uint_as_float(w32[8 * piece + 2]) * scale, __uint_as_float(w32[8 * piece + 3]) * scale);
          w.z = pack_bf16(__uint_as_float(w32[8 * piece + 4]) * scale, __uint_as_float(w32[8 * piece + 5]) * scale);
          w.w = pack_bf16(__uint_as_float(w32[8 * piece + 6]) * scale, __uint_as_float(w32[8 * piece + 7]) * scale);
          reinterpret_cast<uint4*>(qrow + half * 32)[piece] = w;
        }
        return;
      }
      if (half == 0) {
#pragma unroll 1
        for (int j0 = 0; j0 < 32; j0 += 16) {
          uint32_t lo[16], hi[16];
          tmem_ld16(trow + 256 + aset * 64 + j0, lo);
          tmem_ld16(trow + 256 + aset * 64 + 32 + j0, hi);
          tmem_ld_wait();
          float a[16], b[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            a[j] = __uint_as_float(lo[j]) * scale;
            b[j] = __uint_as_float(hi[j]) * scale;
          }
          {
            const float2* cs = rope + static_cast<size_t>(eq) * 32 + j0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float2 t = __ldg(cs + j);
              const float x = a[j], y = b[j];
              a[j] = x * t.x + y * t.y;
              b[j] = y * t.x - x * t.y;
            }
          }
#pragma unroll
          for (int piece = 0; piece < 2; ++piece) {
            uint4 wa, wb;
            wa.x = pack_bf16(a[8 * piece + 0], a[8 * piece + 1]);
            wa.y = pack_bf16(a[8 * piece + 2], a[8 * piece + 3]);
            wa.z = pack_bf16(a[8 * piece + 4], a[8 * piece + 5]);
            wa.w = pack_bf16(a[8 * piece + 6], a[8 * piece + 7]);
            wb.x = pack_bf16(b[8 * piece + 0], b[8 * piece + 1]);
            wb.y = pack_bf16(b[8 * piece + 2], b[8 * piece + 3]);
            wb.z = pack_bf16(b[8 * piece + 4], b[8 * piece + 5]);
            wb.w = pack_bf16(b[8 * piece + 6], b[8 * piece + 7]);
            reinterpret_cast<uint4*>(qrow + j0)[piece] = wa;
            reinterpret_cast<uint4*>(qrow + 32 + j0)[piece] = wb;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
    };
    int pend_u = -1, pend_lu = 0;
    int g = 0, lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      const int qi = u / BH;
      const int qb = nqb - 1 - qi, nkb = qb + 1;
      mbar_wait(&sm.qd_full[lu & 1], (lu >> 1) & 1);  // (complete before S) lse / D of the unit's queries
      float l2, dq;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(l2) : "r"(smem_u32(&sm.lse[lu & 1][r])));
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(dq) : "r"(smem_u32(&sm.dsum[lu & 1][r])));
      l2 *= kLog2e;
      for (int j = 0; j < nkb; ++j) {
        const int gj = g + j;
        mbar_wait(&sm.s_full, gj & 1);
        tc_fence_after();
        uint32_t us[64], ud[64];
        tmem_ld32(trow + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&us[0]));
        tmem_ld32(trow + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&us[32]));
        tmem_ld32(trow + 128 + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&ud[0]));
        tmem_ld32(trow + 128 + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&ud[32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free);  // the next S / dP may start
        mbar_wait(&sm.ds_free, (gj & 1) ^ 1);
        const uint32_t rowoff = static_cast<uint32_t>(half * (128 * 128) + r * 128);
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {
          const int c = half * 64 + 8 * g8;
          float dv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float p = ex2(fmaf(__uint_as_float(us[8 * g8 + e]), scale_log2, -l2));
            dv[e] = p * (__uint_as_float(ud[8 * g8 + e]) - dq);
          }
          if (j == qb) {  // diagonal tile: keys after the query are invisible
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (c + e > r) dv[e] = 0.f;
          }
          st_shared_v4(dbase + rowoff + ((g8 ^ (r & 7)) << 4), pack_bf16(dv[0], dv[1]), pack_bf16(dv[2], dv[3]),
                       pack_bf16(dv[4], dv[5]), pack_bf16(dv[6], dv[7]));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ds_full);
        if (j == 0 && pend_u >= 0) {
          epilogue(pend_u, pend_lu);
          pend_u = -1;
        }
      }
      g += nkb;
      pend_u = u;
      pend_lu = lu;
    }
    if (pend_u >= 0) epilogue(pend_u, pend_lu);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<512>(tmem);
}

// ---------------------------------------------------------------- backward, ping-pong variant
// Same math as the kernels above, with 64-wide inner tiles and TWO tiles in flight per CTA:
// two S/dP TMEM buffers (128 columns each) and two groups of 4 softmax warps (group b owns
// every tile of parity b, one TMEM lane quarter per warp).  While group b turns S(i) into
// P / dS, the tensor core runs group 1-b's S(i+1) and the dV / dK (dQ) MMAs of tile i-1, so
// the MMA <-> softmax hand-offs overlap instead of serialising.  TMEM: 2 x (S 64 | dP 64)
// + 2 accumulator sets (dV|dK = 128, or dQ = 64) <= 512 columns.  Units, ordering, double-
// buffered unit operands and the deferred unit epilogue are as in the kernels above.
constexpr int PT = 64;                          // inner tile: queries (dK/dV kernel) or keys (dQ kernel)
constexpr uint32_t kPTile64 = PT * HD * 2;      // 8 KiB: 64 rows x 64 hd
constexpr uint32_t kPB = TQ * PT * 2;           // 16 KiB: P^T / dS^T [128 rows][64 cols] bf16, one SW128 chunk
constexpr int kPPStages = 4;

struct SmemKVpp {
  uint8_t k[2][kTile], v[2][kTile];                    // unit operands (128 keys)
  uint8_t q[kPPStages][kPTile64], d_o[kPPStages][kPTile64];
  uint8_t p[2][kPB], ds[2][kPB];                        // per softmax group
  float lse[kPPStages][PT], dsum[kPPStages][PT];
  uint64_t kv_full[2], kv_empty[2], qd_full[kPPStages], qd_empty[kPPStages], s_full[2], s_free[2], pd_full[2],
      pd_free[2], acc_full[2], acc_free[2];
  uint32_t tmem;
};

__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_dkdv_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv128, const __grid_constant__ CUtensorMap tm_qkv64,
                        const __grid_constant__ CUtensorMap tm_do64, const float* __restrict__ lse,
                        const float* __restrict__ D, int T, int H, int BH, __nv_bfloat16* __restrict__ dqkv,
                        float scale, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  SmemKVpp& sm = *reinterpret_cast<SmemKVpp*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int nunits = nqb * BH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv128);
    tma_prefetch(&tm_qkv64);
    tma_prefetch(&tm_do64);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], 4);
      mbar_init(&sm.pd_full[i], 4);
      mbar_init(&sm.pd_free[i], 1);
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 8);
    }
    for (int i = 0; i < kPPStages; ++i) {
      mbar_init(&sm.qd_full[i], 1);
      mbar_init(&sm.qd_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S^T[b] cols 128b..+63, dP^T[b] 128b+64..; acc set a: dV 256+128a, dK +64

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int kb = u / BH, bh = u - kb * BH, b = bh / H, h = bh - b * H;
        const int row0 = b * T;
        const int kbuf = lu & 1;
        mbar_wait(&sm.kv_empty[kbuf], ((lu >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.kv_full[kbuf], 2 * kTile);
        tma_load_2d(sm.k[kbuf], &tm_qkv128, &sm.kv_full[kbuf], (H + h) * HD, row0 + kb * TK);
        tma_load_2d(sm.v[kbuf], &tm_qkv128, &sm.kv_full[kbuf], (2 * H + h) * HD, row0 + kb * TK);
        const int ntiles = 2 * (nqb - kb);
        for (int i = 0; i < ntiles; ++i, ++g) {
          const int st = g % kPPStages;
          mbar_wait(&sm.qd_empty[st], ((g / kPPStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.qd_full[st], 2 * kPTile64 + 2 * PT * 4);
          const int q0 = kb * TK + i * PT;
          tma_load_2d(sm.q[st], &tm_qkv64, &sm.qd_full[st], h * HD, row0 + q0);
          tma_load_2d(sm.d_o[st], &tm_do64, &sm.qd_full[st], h * HD, row0 + q0);
          const size_t qo = static_cast<size_t>(bh) * T + q0;
          bulk_load(sm.lse[st], lse + qo, PT * 4, &sm.qd_full[st]);
          bulk_load(sm.dsum[st], D + qo, PT * 4, &sm.qd_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_bf16_f32(TK, PT, false, false);  // [keys x 64 q], K = hd
      constexpr uint32_t kIdA = idesc_bf16_f32(TK, HD, false, true);   // [keys x hd], K = 64 q, B MN-major
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int ntiles = 2 * (nqb - u / BH);
        const int kbuf = lu & 1;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(kbuf * 128);
        mbar_wait(&sm.kv_full[kbuf], (lu >> 1) & 1);
        const uint32_t ka = smem_u32(sm.k[kbuf]), va = smem_u32(sm.v[kbuf]);
        auto issue_s = [&](int gi) {  // S^T = K Q^T, dP^T = V dO^T of global tile gi into buffer gi & 1
          const int st = gi % kPPStages, bb = gi & 1;
          mbar_wait(&sm.qd_full[st], (gi / kPPStages) & 1);
          mbar_wait(&sm.s_free[bb], ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
          const uint32_t sd = tmem + static_cast<uint32_t>(bb * 128);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            umma_bf16(sd, umma_desc_sw128(ka + k * 32, 16, 1024), umma_desc_sw128(qa + k * 32, 16, 1024), kIdS,
                      k > 0 ? 1u : 0u);
            umma_bf16(sd + 64, umma_desc_sw128(va + k * 32, 16, 1024), umma_desc_sw128(oa + k * 32, 16, 1024),
                      kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit(&sm.s_full[bb]);
        };
        issue_s(g);
        issue_s(g + 1);
        mbar_wait(&sm.acc_free[kbuf], ((lu >> 1) & 1) ^ 1);
        for (int i = 0; i < ntiles; ++i) {
          const int gi = g + i, st = gi % kPPStages, bb = gi & 1;
          mbar_wait(&sm.pd_full[bb], (gi >> 1) & 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
          const uint32_t pa = smem_u32(sm.p[bb]), da = smem_u32(sm.ds[bb]);
#pragma unroll
          for (int k = 0; k < PT / 16; ++k) {
            umma_bf16(acc, umma_desc_sw128(pa + k * 32, 16, 1024), umma_desc_sw128(oa + k * 2048, 8192, 1024), kIdA,
                      (i > 0 || k > 0) ? 1u : 0u);
            umma_bf16(acc + 64, umma_desc_sw128(da + k * 32, 16, 1024), umma_desc_sw128(qa + k * 2048, 8192, 1024),
                      kIdA, (i > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&sm.pd_free[bb]);
          umma_commit(&sm.qd_empty[st]);
          if (i + 2 < ntiles) issue_s(gi + 2);
        }
        umma_commit(&sm.acc_full[kbuf]);
        umma_commit(&sm.kv_empty[kbuf]);
        g += ntiles;
      }
    }
  } else if (warp >= 4) {
    const int sw = warp - 4, quarter = sw & 3, grp = sw >> 2;
    const int r = quarter * 32 + lane;  // key row within the unit
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t pbase = smem_u32(sm.p[grp]), dbase = smem_u32(sm.ds[grp]);
    const size_t ld = static_cast<size_t>(3) * H * HD;
    // unit epilogue (group 0 -> dV, group 1 -> dK x scale), run after this group's first tile of
    // the next unit so the accumulator set has long been complete
    auto epilogue = [&](int eu, int elu) {
      const int ekb = eu / BH, ebh = eu - ekb * BH, eb = ebh / H, eh = ebh - eb * H;
      const int aset = elu & 1;
      mbar_wait(&sm.acc_full[aset], (elu >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* dst = dqkv + (static_cast<size_t>(eb) * T + ekb * TK + r) * ld +
                           static_cast<size_t>(grp ? (H + eh) * HD : (2 * H + eh) * HD);
      const float mul = grp ? scale : 1.f;
      uint32_t w32[64];
      tmem_ld32(trow + 256 + aset * 128 + grp * 64, *reinterpret_cast<uint32_t(*)[32]>(&w32[0]));
      tmem_ld32(trow + 256 + aset * 128 + grp * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&w32[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
#pragma unroll
      for (int piece = 0; piece < 8; ++piece) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(w32[8 * piece + 0]) * mul, __uint_as_float(w32[8 * piece + 1]) * mul);
        w.y = pack_bf16(__uint_as_float(w32[8 * piece + 2]) * mul, __uint_as_float(w32[8 * piece + 3]) * mul);
        w.z = pack_bf16(__uint_as_float(w32[8 * piece + 4]) * mul, __uint_as_float(w32[8 * piece + 5]) * mul);
        w.w = pack_bf16(__uint_as_float(w32[8 * piece + 6]) * mul, __uint_as_float(w32[8 * piece + 7]) * mul);
        reinterpret_cast<uint4*>(dst)[piece] = w;
      }
    };
    int pend_u = -1, pend_lu = 0;
    int g = 0, lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      const int ntiles = 2 * (nqb - u / BH);
      for (int i = grp; i < ntiles; i += 2) {
        const int gi = g + i, st = gi % kPPStages;
        mbar_wait(&sm.s_full[grp], (gi >> 1) & 1);
        mbar_wait(&sm.qd_full[st], (gi / kPPStages) & 1);  // (complete) lse / D of this tile visible
        tc_fence_after();
        uint32_t us[64], ud[64];
        tmem_ld32(trow + grp * 128, *reinterpret_cast<uint32_t(*)[32]>(&us[0]));
        tmem_ld32(trow + grp * 128 + 32, *reinterpret_cast<uint32_t(*)[32]>(&us[32]));
        tmem_ld32(trow + grp * 128 + 64, *reinterpret_cast<uint32_t(*)[32]>(&ud[0]));
        tmem_ld32(trow + grp * 128 + 96, *reinterpret_cast<uint32_t(*)[32]>(&ud[32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[grp]);
        mbar_wait(&sm.pd_free[grp], ((gi >> 1) & 1) ^ 1);  // this group's previous dV/dK MMAs read P / dS
        const uint32_t rowoff = static_cast<uint32_t>(r * 128);
        const uint32_t la_ = smem_u32(&sm.lse[st][0]), da_ = smem_u32(&sm.dsum[st][0]);
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {  // 8 queries at a time: P^T, dS^T -> bf16 -> swizzled smem
          const uint4 la = ld_shared_v4(la_ + 32 * g8), lb = ld_shared_v4(la_ + 32 * g8 + 16);
          const uint4 da4 = ld_shared_v4(da_ + 32 * g8), db4 = ld_shared_v4(da_ + 32 * g8 + 16);
          const float lq[8] = {__uint_as_float(la.x), __uint_as_float(la.y), __uint_as_float(la.z),
                               __uint_as_float(la.w), __uint_as_float(lb.x), __uint_as_float(lb.y),
                               __uint_as_float(lb.z), __uint_as_float(lb.w)};
          const float dq8[8] = {__uint_as_float(da4.x), __uint_as_float(da4.y), __uint_as_float(da4.z),
                                __uint_as_float(da4.w), __uint_as_float(db4.x), __uint_as_float(db4.y),
                                __uint_as_float(db4.z), __uint_as_float(db4.w)};
          float pv[8], dv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float pe = ex2(fmaf(__uint_as_float(us[8 * g8 + e]), scale_log2, -lq[e] * kLog2e));
            pv[e] = pe;
            dv[e] = pe * (__uint_as_float(ud[8 * g8 + e]) - dq8[e]);
          }
          if (i < 2) {  // diagonal: query kb*128 + 64 i + c sees key kb*128 + r iff 64 i + c >= r
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (PT * i + 8 * g8 + e < r) pv[e] = dv[e] = 0.f;
          }
          const uint32_t off = rowoff + ((g8 ^ (r & 7)) << 4);
          st_shared_v4(pbase + off, pack_bf16(pv[0], pv[1]), pack_bf16(pv[2], pv[3]), pack_bf16(pv[4], pv[5]),
                       pack_bf16(pv[6], pv[7]));
          st_shared_v4(dbase + off, pack_bf16(dv[0], dv[1]), pack_bf16(dv[2], dv[3]), pack_bf16(dv[4], dv[5]),
                       pack_bf16(dv[6], dv[7]));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pd_full[grp]);
        if (i == grp && pend_u >= 0) {
          epilogue(pend_u, pend_lu);
          pend_u = -1;
        }
      }
      g += ntiles;
      pend_u = u;
      pend_lu = lu;
    }
    if (pend_u >= 0) epilogue(pend_u, pend_lu);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<512>(tmem);
}

struct SmemQpp {  // dQ kernel, ping-pong
  uint8_t q[2][kTile], d_o[2][kTile];                                // unit operands (128 queries)
  uint8_t k[kPPStages][kPTile64], v[kPPStages][kPTile64];            // 64-key tiles
  uint8_t ds[2][kPB];                                                 // per softmax group
  float lse[2][TQ], dsum[2][TQ];
  uint64_t qd_full[2], qd_empty[2], kv_full[kPPStages], kv_empty[kPPStages], s_full[2], s_free[2], ds_full[2],
      ds_free[2], acc_full[2], acc_free[2];
  uint32_t tmem;
};

// Unit u = (query tile qb, sequence x head bh), longest first; inner tiles of 64 keys.
__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_dq_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv128, const __grid_constant__ CUtensorMap tm_qkv64,
                      const __grid_constant__ CUtensorMap tm_do128, const float* __restrict__ lse,
                      const float* __restrict__ D, int T, int H, int BH, __nv_bfloat16* __restrict__ dqkv, float scale,
                      float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  SmemQpp& sm = *reinterpret_cast<SmemQpp*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int nunits = nqb * BH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv128);
    tma_prefetch(&tm_qkv64);
    tma_prefetch(&tm_do128);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.qd_full[i], 1);
      mbar_init(&sm.qd_empty[i], 1);
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], 4);
      mbar_init(&sm.ds_full[i], 4);
      mbar_init(&sm.ds_free[i], 1);
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 8);
    }
    for (int i = 0; i < kPPStages; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S[b] cols 128b..+63, dP[b] 128b+64..; dQ set a: 256 + 64a

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int qi = u / BH, bh = u - qi * BH, b = bh / H, h = bh - b * H;
        const int qb = nqb - 1 - qi, row0 = b * T;
        const int qbuf = lu & 1;
        mbar_wait(&sm.qd_empty[qbuf], ((lu >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.qd_full[qbuf], 2 * kTile + 2 * TQ * 4);
        tma_load_2d(sm.q[qbuf], &tm_qkv128, &sm.qd_full[qbuf], h * HD, row0 + qb * TQ);
        tma_load_2d(sm.d_o[qbuf], &tm_do128, &sm.qd_full[qbuf], h * HD, row0 + qb * TQ);
        const size_t qo = static_cast<size_t>(bh) * T + qb * TQ;
        bulk_load(sm.lse[qbuf], lse + qo, TQ * 4, &sm.qd_full[qbuf]);
        bulk_load(sm.dsum[qbuf], D + qo, TQ * 4, &sm.qd_full[qbuf]);
        const int ntiles = 2 * (qb + 1);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int st = g % kPPStages;
          mbar_wait(&sm.kv_empty[st], ((g / kPPStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.kv_full[st], 2 * kPTile64);
          tma_load_2d(sm.k[st], &tm_qkv64, &sm.kv_full[st], (H + h) * HD, row0 + j * PT);
          tma_load_2d(sm.v[st], &tm_qkv64, &sm.kv_full[st], (2 * H + h) * HD, row0 + j * PT);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_bf16_f32(TQ, PT, false, false);  // [q x 64 keys], K = hd
      constexpr uint32_t kIdQ = idesc_bf16_f32(TQ, HD, false, true);   // [q x hd], K = 64 keys, B MN-major
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int ntiles = 2 * (nqb - u / BH);
        const int qbuf = lu & 1;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(qbuf * 64);
        mbar_wait(&sm.qd_full[qbuf], (lu >> 1) & 1);
        const uint32_t qa = smem_u32(sm.q[qbuf]), oa = smem_u32(sm.d_o[qbuf]);
        auto issue_s = [&](int gj) {  // S = Q K^T, dP = dO V^T of global tile gj into buffer gj & 1
          const int st = gj % kPPStages, bb = gj & 1;
          mbar_wait(&sm.kv_full[st], (gj / kPPStages) & 1);
          mbar_wait(&sm.s_free[bb], ((gj >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sm.k[st]), va = smem_u32(sm.v[st]);
          const uint32_t sd = tmem + static_cast<uint32_t>(bb * 128);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            umma_bf16(sd, umma_desc_sw128(qa + k * 32, 16, 1024), umma_desc_sw128(ka + k * 32, 16, 1024), kIdS,
                      k > 0 ? 1u : 0u);
            umma_bf16(sd + 64, umma_desc_sw128(oa + k * 32, 16, 1024), umma_desc_sw128(va + k * 32, 16, 1024),
                      kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit(&sm.s_full[bb]);
        };
        issue_s(g);
        issue_s(g + 1);
        mbar_wait(&sm.acc_free[qbuf], ((lu >> 1) & 1) ^ 1);
        for (int j = 0; j < ntiles; ++j) {
          const int gj = g + j, st = gj % kPPStages, bb = gj & 1;
          mbar_wait(&sm.ds_full[bb], (gj >> 1) & 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sm.k[st]), da = smem_u32(sm.ds[bb]);
#pragma unroll
          for (int k = 0; k < PT / 16; ++k)
            umma_bf16(acc, umma_desc_sw128(da + k * 32, 16, 1024), umma_desc_sw128(ka + k * 2048, 8192, 1024), kIdQ,
                      (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&sm.ds_free[bb]);
          umma_commit(&sm.kv_empty[st]);
          if (j + 2 < ntiles) issue_s(gj + 2);
        }
        umma_commit(&sm.acc_full[qbuf]);
        umma_commit(&sm.qd_empty[qbuf]);
        g += ntiles;
      }
    }
  } else if (warp >= 4) {
    const int sw = warp - 4, quarter = sw & 3, grp = sw >> 2;
    const int r = quarter * 32 + lane;  // query row within the unit
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t dbase = smem_u32(sm.ds[grp]);
    const size_t ld = static_cast<size_t>(3) * H * HD;
    // unit epilogue (dQ x scale; group b writes columns 32b..32b+31), one tile late
    auto epilogue = [&](int eu, int elu) {
      const int eqi = eu / BH, ebh = eu - eqi * BH, eb = ebh / H, eh = ebh - eb * H;
      const int eq = (nqb - 1 - eqi) * TQ + r;
      const int aset = elu & 1;
      mbar_wait(&sm.acc_full[aset], (elu >> 1) & 1);
      tc_fence_after();
      uint32_t w32[32];
      tmem_ld32(trow + 256 + aset * 64 + grp * 32, w32);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
      __nv_bfloat16* qrow = dqkv + (static_cast<size_t>(eb) * T + eq) * ld + static_cast<size_t>(eh * HD) + grp * 32;
#pragma unroll
      for (int piece = 0; piece < 4; ++piece) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(w32[8 * piece + 0]) * scale, __uint_as_float(w32[8 * piece + 1]) * scale);
        w.y = pack_bf16(__uint_as_float(w32[8 * piece + 2]) * scale, __uint_as_float(w32[8 * piece + 3]) * scale);
        w.z = pack_bf16(__uint_as_float(w32[8 * piece + 4]) * scale, __uint_as_float(w32[8 * piece + 5]) * scale);
        w.w = pack_bf16(__uint_as_float(w32[8 * piece + 6]) * scale, __uint_as_float(w32[8 * piece + 7]) * scale);
        reinterpret_cast<uint4*>(qrow)[piece] = w;
      }
    };
    int pend_u = -1, pend_lu = 0;
    int g = 0, lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      const int qb = nqb - 1 - u / BH, ntiles = 2 * (qb + 1);
      mbar_wait(&sm.qd_full[lu & 1], (lu >> 1) & 1);  // lse / D of the unit's queries
      float l2, dq;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(l2) : "r"(smem_u32(&sm.lse[lu & 1][r])));
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(dq) : "r"(smem_u32(&sm.dsum[lu & 1][r])));
      l2 *= kLog2e;
      for (int j = grp; j < ntiles; j += 2) {
        const int gj = g + j;
        mbar_wait(&sm.s_full[grp], (gj >> 1) & 1);
        tc_fence_after();
        uint32_t us[64], ud[64];
        tmem_ld32(trow + grp * 128, *reinterpret_cast<uint32_t(*)[32]>(&us[0]));
        tmem_ld32(trow + grp * 128 + 32, *reinterpret_cast<uint32_t(*)[32]>(&us[32]));
        tmem_ld32(trow + grp * 128 + 64, *reinterpret_cast<uint32_t(*)[32]>(&ud[0]));
        tmem_ld32(trow + grp * 128 + 96, *reinterpret_cast<uint32_t(*)[32]>(&ud[32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[grp]);
        mbar_wait(&sm.ds_free[grp], ((gj >> 1) & 1) ^ 1);
        const uint32_t rowoff = static_cast<uint32_t>(r * 128);
        const bool diag = j >= 2 * qb;  // keys 64 j + c vs query qb*128 + r: visible iff 64 j + c <= 128 qb + r
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {
          float dv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float pe = ex2(fmaf(__uint_as_float(us[8 * g8 + e]), scale_log2, -l2));
            dv[e] = pe * (__uint_as_float(ud[8 * g8 + e]) - dq);
          }
          if (diag) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (PT * j + 8 * g8 + e > TQ * qb + r) dv[e] = 0.f;
          }
          st_shared_v4(dbase + rowoff + ((g8 ^ (r & 7)) << 4), pack_bf16(dv[0], dv[1]), pack_bf16(dv[2], dv[3]),
                       pack_bf16(dv[4], dv[5]), pack_bf16(dv[6], dv[7]));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ds_full[grp]);
        if (j == grp && pend_u >= 0) {
          epilogue(pend_u, pend_lu);
          pend_u = -1;
        }
      }
      g += ntiles;
      pend_u = u;
      pend_lu = lu;
    }
    if (pend_u >= 0) epilogue(pend_u, pend_lu);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<512>(tmem);
}

}  // namespace

bool attn_fwd_tc_supported(size_t T, size_t hd) { return hd == HD && T % TQ == 0; }

// CKF_ATTN_DEBUG=1: per-CTA phase timings of the forward kernel (tools/attn_debug.py)
long long* attn_fwd_debug_buffer() {
  static long long* p = [] {
    long long* b = nullptr;
    if (std::getenv("CKF_ATTN_DEBUG")) CKF_CUDA(cudaMalloc(&b, 8 * sizeof(long long) * 65536));
    return b;
  }();
  return p;
}

void attn_fwd_tc(const bf16* qkv, size_t B, size_t T, size_t H, size_t hd, bf16* o, float* lse, cudaStream_t s) {
  if (!attn_fwd_tc_supported(T, hd)) raise(1, "tcgen05 attention: head_dim 64 and seq_len % 128 == 0");
  const CUtensorMap tm = tma::make_2d_bf16(qkv, 3 * H * hd, B * T, 3 * H * hd, 64, 128);
  const CUtensorMap tkv = tma::make_2d_bf16(qkv, 3 * H * hd, B * T, 3 * H * hd, 64, FK);
  const size_t smem = sizeof(Smem) + 1024;
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    attr = true;
  }
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(hd));
  dim3 grid(static_cast<unsigned>(T / TQ), static_cast<unsigned>(B * H));
  long long* dbg = attn_fwd_debug_buffer();
  attn_fwd_tc_kernel<<<grid, kThreads, smem, s>>>(tm, tkv, static_cast<int>(T), static_cast<int>(H), o, lse,
                                                  scale_log2, dbg);
  CKF_LAUNCH_CHECK();
}

void attn_bwd_tc(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
                 size_t hd, bf16* dqkv, float* Dsum, cudaStream_t s, const float2* rope_tab) {
  if (!attn_fwd_tc_supported(T, hd)) raise(1, "tcgen05 attention: head_dim 64 and seq_len % 128 == 0");
  const size_t rows = B * T * H;
  dsum_kernel<<<static_cast<unsigned>((rows + 31) / 32), 256, 0, s>>>(o, dout, static_cast<int>(B), static_cast<int>(T),
                                                                     static_cast<int>(H), Dsum);
  CKF_LAUNCH_CHECK();
  const CUtensorMap tq = tma::make_2d_bf16(qkv, 3 * H * hd, B * T, 3 * H * hd, 64, 128);
  const CUtensorMap td = tma::make_2d_bf16(dout, H * hd, B * T, H * hd, 64, 128);
  const size_t smem_kv = sizeof(SmemKV) + 1024, smem_q = sizeof(SmemQ) + 1024;
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(attn_dkdv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_kv)));
    CKF_CUDA(cudaFuncSetAttribute(attn_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_q)));
    attr = true;
  }
  const float scale = 1.f / sqrtf(static_cast<float>(hd));
  static const int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  const int BH = static_cast<int>(B * H), units = static_cast<int>(T / TQ) * BH;
  const unsigned grid = static_cast<unsigned>(std::min(units, sms));
  static const bool pp = [] {  // CKF_ATTN_BWD=serial: the one-tile-in-flight kernels above
    const char* v = std::getenv("CKF_ATTN_BWD");
    return !(v && std::string(v) == "serial");
  }();
  if (pp && !rope_tab) {
    const CUtensorMap tq64 = tma::make_2d_bf16(qkv, 3 * H * hd, B * T, 3 * H * hd, 64, 64);
    const CUtensorMap td64 = tma::make_2d_bf16(dout, H * hd, B * T, H * hd, 64, 64);
    const size_t smem_kvp = sizeof(SmemKVpp) + 1024, smem_qp = sizeof(SmemQpp) + 1024;
    static bool attr_pp = false;
    if (!attr_pp) {
      CKF_CUDA(cudaFuncSetAttribute(attn_dkdv_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_kvp)));
      CKF_CUDA(cudaFuncSetAttribute(attn_dq_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_qp)));
      attr_pp = true;
    }
    attn_dkdv_pp_kernel<<<grid, kThreadsBwd, smem_kvp, s>>>(tq, tq64, td64, lse, Dsum, static_cast<int>(T),
                                                            static_cast<int>(H), BH, dqkv, scale, scale * kLog2e);
    CKF_LAUNCH_CHECK();
    attn_dq_pp_kernel<<<grid, kThreadsBwd, smem_qp, s>>>(tq, tq64, td, lse, Dsum, static_cast<int>(T),
                                                        static_cast<int>(H), BH, dqkv, scale, scale * kLog2e);
    CKF_LAUNCH_CHECK();
    return;
  }
  long long* dbg = attn_fwd_debug_buffer();
  attn_dkdv_tc_kernel<<<grid, kThreadsBwd, smem_kv, s>>>(tq, td, lse, Dsum, static_cast<int>(T), static_cast<int>(H), BH,
                                                         dqkv, scale, scale * kLog2e, rope_tab,
                                                         dbg ? dbg + 8 * 32768 : nullptr);
  CKF_LAUNCH_CHECK();
  attn_dq_tc_kernel<<<grid, kThreadsBwd, smem_q, s>>>(tq, td, lse, Dsum, static_cast<int>(T), static_cast<int>(H), BH,
                                                   dqkv, scale, scale * kLog2e, rope_tab);
  CKF_LAUNCH_CHECK();
}

}  // namespace ckf::llama
