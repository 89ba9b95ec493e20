// Causal attention on the 5th-generation tensor cores, head_dim 64 or 128.
//
// Forward: one CTA per (128-query tile, sequence x head) -- at head_dim 128 per PAIR of query
// tiles, each with its own softmax warp group and MMA issuer, sharing the K / V stages.  Q, K, V tiles arrive by TMA
// straight from the packed qkv activation (2-D tensor maps, boxes of 64 columns, 128-byte
// swizzle: K-major for Q and K, MN-major for V as the PV B operand; a 128-wide head is
// two such column chunks).  S = Q K^T accumulates in TMEM, the softmax warps turn it into
// P (one query row per thread, online max / sum with lazy rescaling), P goes back to
// swizzled shared memory as the A operand of O += P V, whose fp32 accumulator also lives
// in TMEM.
//
// Backward (dK dV kernel + dQ kernel, deterministic, no atomics): persistent over
// (tile, head) units longest-first, two inner tiles in flight (ping-pong softmax groups).
//
// Warp roles: forward (one query tile) 0 TMA producer + TMEM allocator, 1 MMA issuer, 2..5 softmax;
// forward (two query tiles) 0 producer, 1 / 3 MMA issuers, 2 allocator, 4..11 softmax; dK dV 0
// producer, 1 S / dP issuer, 2 allocator, 3 dV / dK issuer, 4..11 softmax.  MMA issuers run
// warp-converged with elect.sync (sm100.cuh umma_*_w).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "llama_kernels.h"
#include "sm100.cuh"

namespace ckf::llama {
namespace {

using namespace ckf::sm100;

constexpr int TQ = 128, TK = 128;
constexpr int kThreadsBwd = 384;  // backward: 8 softmax warps (2 groups x one per TMEM lane quarter)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2, common.cuh) and the 3-input max (FMNMX3):
// the softmax loops are issue-bound (a polynomial exp2 on the FMA pipe made them slower, so
// MUFU is not the limit), and these halve their FMA / add / max instruction counts.

// A [rows x HD] bf16 tile in shared memory as HD/64 K-major SW128 chunks of [rows][128 B]:
// TMA brings each 64-column chunk; UMMA K step k (16 columns) reads chunk k/4 at byte 32 (k%4).
template <int HD>
__device__ __forceinline__ void tma_tile(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int col, int row,
                                         int rows) {
#pragma unroll
  for (int c = 0; c < HD / 64; ++c) tma_load_2d(dst + c * rows * 128, map, bar, col + c * 64, row);
}
__device__ __forceinline__ uint32_t kmajor_k(uint32_t base, int rows, int k) {
  return base + static_cast<uint32_t>((k >> 2) * rows * 128 + (k & 3) * 32);
}

// One row of a head's gradient (HD fp32 accumulator columns at TMEM address trow) times mul ->
// bf16 at dst; with rope (pair-major cos/sin table [HD/2][T]) the inverse rotation of position
// pos is applied first, in fp32 (the RoPE backward fused into the epilogue: (j, j + HD/2) pairs,
// x1' = x1 c + x2 s, x2' = x2 c - x1 s -- the transpose of the forward rotation).
template <int HD>
__device__ __forceinline__ void store_head_row(uint32_t trow, float mul, __nv_bfloat16* dst, const float2* rope,
                                               int pos, int T) {
  auto st8 = [&](__nv_bfloat16* p, const float* v) {
    uint4 w;
    w.x = pack_bf16(v[0], v[1]);
    w.y = pack_bf16(v[2], v[3]);
    w.z = pack_bf16(v[4], v[5]);
    w.w = pack_bf16(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = w;
  };
  if (rope) {
#pragma unroll 1
    for (int c0 = 0; c0 < HD / 2; c0 += 32) {
      uint32_t a[32], b[32];
      tmem_ld32(trow + c0, a);
      tmem_ld32(trow + HD / 2 + c0, b);
      tmem_ld_wait();
      const float2* cs = rope + static_cast<size_t>(c0) * T + pos;
#pragma unroll
      for (int piece = 0; piece < 4; ++piece) {
        float y1[8], y2[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = 8 * piece + e;
          const float2 t = __ldg(cs + static_cast<size_t>(j) * T);
          const float x1 = __uint_as_float(a[j]) * mul, x2 = __uint_as_float(b[j]) * mul;
          y1[e] = x1 * t.x + x2 * t.y;
          y2[e] = x2 * t.x - x1 * t.y;
        }
        st8(dst + c0 + 8 * piece, y1);
        st8(dst + HD / 2 + c0 + 8 * piece, y2);
      }
    }
  } else {
#pragma unroll 1
    for (int c0 = 0; c0 < HD; c0 += 32) {
      uint32_t w32[32];
      tmem_ld32(trow + c0, w32);
      tmem_ld_wait();
#pragma unroll
      for (int piece = 0; piece < 4; ++piece) {
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(w32[8 * piece + e]) * mul;
        st8(dst + c0 + 8 * piece, v);
      }
    }
  }
}

// ---------------------------------------------------------------- forward
// 128 queries x 64-key tiles: S double-buffered in TMEM (2 x 64 columns) + O (HD columns).
// m is only raised when a tile's max exceeds it by more than kRescale (P stays <= 2^kRescale,
// exact in bf16 range); then the thread rescales its O row in TMEM after the previous P V.
constexpr int FK = 64;
constexpr uint32_t kPTile = TQ * FK * 2;  // 16 KiB: P [128 rows][128 B]
constexpr float kRescale = 8.f;
// exponential pairs (of 8) on the FMA pipe in the head_dim-64 forward (measured at [64, 1024, 16,
// 64]: 0 -> 347.5 us, 1 -> 336.0, 2 -> 339.3, 3 -> 359.6, 4 -> 395.7; head_dim 128 is fastest with 0)
constexpr int kFwdPolyDefault = 1;
// query tiles per forward CTA (FwdCfg), measured (profiles/r02_attention_fwd_ng_sweep.jsonl):
// head_dim 128: 1694 -> 1159 us at [16, 4096, 16, 128] with two (the single-tile CTA fits only
// once per SM: 4 softmax warps); head_dim 64: two single-tile CTAs per SM stay ahead (335 vs 379 us
// at [64, 1024, 16, 64])
template <int HD>
constexpr int kFwdNgDefault = HD == 128 ? 2 : 1;
// per-tile clock instrumentation of the forward (tools/attn_debug.py): compiled in only with
// -DCKF_ATTN_DEBUG_BUILD=1 (and CKF_ATTN_DEBUG=1 at run time), so the hot loop carries none of it
#ifndef CKF_ATTN_DEBUG_BUILD
#define CKF_ATTN_DEBUG_BUILD 0
#endif
constexpr bool kDbg = CKF_ATTN_DEBUG_BUILD != 0;
// bottleneck experiments on the dK dV kernel (debug builds only): 1 = no softmax math (P / dS
// constant), 2 = no MMAs issued (barriers still committed)
#ifndef CKF_ATTN_BWD_EXPERIMENT
#define CKF_ATTN_BWD_EXPERIMENT 0
#endif
constexpr int kBwdExp = CKF_ATTN_BWD_EXPERIMENT;
// dK dV MMA issue: 2 = two issuer warps (warp 1: S / dP of every tile as soon as its Q / dO stage
// and the group's S buffer allow; warp 3: the dV / dK accumulation in tile order), 1 = one warp
// interleaving both (an S waiting on a Q / dO load then held back the dV / dK of the tile before)
#ifndef CKF_ATTN_BWD_ISSUERS
#define CKF_ATTN_BWD_ISSUERS 2
#endif
// CKF_ATTN_P_ALIAS=1: two query tiles per CTA (hd 128) write P into the TMEM columns of the S it
// came from (the P V MMA reads it there; the next S into that buffer is issued after that P V)
#ifndef CKF_ATTN_P_ALIAS
#define CKF_ATTN_P_ALIAS 1
#endif
#ifndef CKF_ATTN_P_TMEM
#define CKF_ATTN_P_TMEM 1
#endif
constexpr int kBwdSplitDefault = 1;  // 2 measured no faster (1084.7 vs 1087.8 us at [64, 1024, 16, 64])  // exponential pairs (of 8) on the FMA pipe, forward

// NG query tiles per CTA (NG = 2: query tiles 2c and 2c+1 share every K / V tile the producer
// loads; two softmax warp groups, one per tile, each on its own S pair and O in TMEM, so the
// tensor core runs one group's S / P V while the other group is in its softmax).
template <int HD, int NG>
struct FwdCfg {
  static constexpr uint32_t kQ = TQ * HD * 2, kK = FK * HD * 2;
  // P aliased onto S in TMEM (two query tiles): no P buffers in shared memory, two more K / V stages
  static constexpr bool kPAlias = NG == 2 && CKF_ATTN_P_ALIAS;
  static constexpr int kKSt = HD == 64 ? 4 : (kPAlias ? 5 : 3), kVSt = HD == 64 ? 3 : (NG == 2 ? (kPAlias ? 5 : 3) : 2);
  // NG = 1: 104 KiB vs 144 KiB of shared memory; two hd-128 CTAs per SM with 2 K / 1 V stages (112 KiB)
  // measured 1.7x slower (1697 -> 2887 us at [16, 4096, 16, 128]): the single V stage serialises
  static constexpr int kMinBlocks = HD == 64 && NG == 1 ? 2 : 1;
  // one query tile: 6 warps -- producer + TMEM allocator (0), MMA issuer (1), softmax (2..5, TMEM lane
  // quarter = warp % 4) -- so two CTAs per SM get 170 registers per thread instead of 128 (no spills);
  // two tiles: producer (0), issuers (1, 3), allocator (2), softmax (4..11)
  static constexpr int kThreads = NG == 1 ? 192 : 128 + 128 * NG;
  static constexpr int kSoftWarp0 = NG == 1 ? 2 : 4, kAllocWarp = NG == 1 ? 0 : 2;
  // TMEM: group g's S pair at columns g*128 + {0, 64}, its O at NG*128 + g*HD
  static constexpr int kTmemCols = NG * 128 + NG * HD <= 256 ? 256 : 512;
  // S_{j+2} issued two tiles ahead (into the buffer the softmax has just loaded) when a third V
  // stage lets the producer run that far ahead
  static constexpr bool kEarly = kVSt >= 3;
  // P in TMEM (A operand of P V from tensor memory: no shared-memory round trip, no proxy fence):
  // columns 192 + 32 pb next to S pair 0-127 and O 128-191 -- head_dim 64, one query tile
  static constexpr bool kPTmem = HD == 64 && NG == 1 && CKF_ATTN_P_TMEM;
};

template <int HD, int NG>
struct Smem {
  using C = FwdCfg<HD, NG>;
  uint8_t q[NG][C::kQ];
  uint8_t k[C::kKSt][C::kK];
  uint8_t v[C::kVSt][C::kK];
  uint8_t p[C::kPTmem || C::kPAlias ? 1 : NG][C::kPTmem || C::kPAlias ? 1 : 2][C::kPTmem || C::kPAlias ? 16 : kPTile];
  uint64_t q_full;
  uint64_t k_full[C::kKSt], k_empty[C::kKSt], v_full[C::kVSt], v_empty[C::kVSt];
  uint64_t s_full[NG][2], s_free[NG][2], p_full[NG][2], p_free[NG][2];
  uint64_t o_full[NG], o_free[NG];
  // persistent CTAs: the unit ring (written by the producer, read by the issuers and softmax warps)
  // and the Q buffer's release by the unit's last S MMAs
  uint64_t unit_full[2], unit_empty[2], q_empty;
  int unit[2];
  uint32_t tmem;
};

__device__ __forceinline__ void tmem_st32_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// POLY: of every 8 exponential pairs of a softmax row chunk, POLY run on the FMA pipe
// (ex2_fma2), the rest on MUFU (CKF_ATTN_POLY selects; 0 = all MUFU)
template <int HD, int POLY, int NG>
__global__ void __launch_bounds__(FwdCfg<HD, NG>::kThreads, FwdCfg<HD, NG>::kMinBlocks)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_kv,
                       int T, int H, __nv_bfloat16* __restrict__ o, float* __restrict__ lse, float scale_log2,
                       int BH, int* __restrict__ ctr, long long* __restrict__ dbg) {
  using C = FwdCfg<HD, NG>;
  constexpr int KS = C::kKSt, VS = C::kVSt;
  extern __shared__ uint8_t smem_raw[];
  const long long t_start = clock64();
  Smem<HD, NG>& sm =
      *reinterpret_cast<Smem<HD, NG>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  // Work unit u = (sequence x head bh, query tile pair c): bh = u / nqu, heavy (late) query tiles
  // first within a sequence x head; NG = 2: tiles qb0 = 2c and 2c + 1.  ctr == nullptr: one unit
  // per CTA, u = (blockIdx.y, blockIdx.x).  Otherwise the CTAs are persistent and take units in
  // that same order from the counter (the CTA that draws the last past-the-end ticket resets it
  // for the next launch): each CTA loads the next unit's Q while its softmax finishes the current
  // one and keeps its TMEM allocation, instead of paying a CTA start per 128 queries.
  const int nqu = nqb / NG, nunits = nqu * BH;
  struct UnitPos {
    int qb0, bh, row0, h;
  };
  auto unit_pos = [&](int u) {
    UnitPos w;
    w.bh = u / nqu;
    w.qb0 = NG * (nqu - 1 - (u - w.bh * nqu));
    const int b = w.bh / H;
    w.h = w.bh - b * H;
    w.row0 = b * T;
    return w;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_kv);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.q_full, 1);
    // a K / V stage is released by every group's issuer (group 0 releases the last query tile's
    // two extra key tiles without reading them)
    for (int i = 0; i < KS; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], NG);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], NG);
    }
    for (int g = 0; g < NG; ++g) {
      for (int i = 0; i < 2; ++i) {
        mbar_init(&sm.s_full[g][i], 1);
        mbar_init(&sm.s_free[g][i], 4);
        mbar_init(&sm.p_full[g][i], 4);
        mbar_init(&sm.p_free[g][i], 1);
      }
      mbar_init(&sm.o_full[g], 1);
      mbar_init(&sm.o_free[g], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.unit_full[i], 1);
      mbar_init(&sm.unit_empty[i], 5 * NG);  // every issuer and softmax warp
    }
    mbar_init(&sm.q_empty, NG);
    fence_barrier_init();
  }
  if (warp == C::kAllocWarp) tmem_alloc<C::kTmemCols>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: per unit the Q tiles once (after the previous unit's last S
      // MMAs), then K_j and V_j (each exactly once); jj counts K / V tiles over the CTA's units
      int jj = 0;
      for (int k = 0;; ++k) {
        int u = -1;
        if (ctr) {
          const int t = atomicAdd(ctr, 1);
          if (t < nunits)
            u = t;
          else if (t == nunits + static_cast<int>(gridDim.x) - 1)
            atomicExch(ctr, 0);  // every CTA has drawn its last ticket: reset for the next launch
        } else if (k == 0) {
          u = static_cast<int>(blockIdx.y) * nqu + static_cast<int>(blockIdx.x);
        }
        mbar_wait(&sm.unit_empty[k & 1], ((k >> 1) & 1) ^ 1);
        sm.unit[k & 1] = u;
        mbar_arrive(&sm.unit_full[k & 1]);
        if (u < 0) break;
        const UnitPos w = unit_pos(u);
        const int nkb_last = 2 * (w.qb0 + NG - 1) + 2;  // causal: 64-key tiles of the last query tile
        const int qcol = w.h * HD, kcol = (H + w.h) * HD, vcol = (2 * H + w.h) * HD;
        mbar_wait(&sm.q_empty, (k & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.q_full, NG * C::kQ);
#pragma unroll
        for (int g = 0; g < NG; ++g) tma_tile<HD>(sm.q[g], &tm_qkv, &sm.q_full, qcol, w.row0 + (w.qb0 + g) * TQ, TQ);
        for (int j = 0; j < nkb_last; ++j, ++jj) {
          const int ks = jj % KS, vs = jj % VS;
          mbar_wait(&sm.k_empty[ks], ((jj / KS) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.k_full[ks], C::kK);
          tma_tile<HD>(sm.k[ks], &tm_kv, &sm.k_full[ks], kcol, w.row0 + j * FK, FK);
          mbar_wait(&sm.v_empty[vs], ((jj / VS) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.v_full[vs], C::kK);
          tma_tile<HD>(sm.v[vs], &tm_kv, &sm.v_full[vs], vcol, w.row0 + j * FK, FK);
        }
      }
    }
  } else if (warp == 1 || (NG == 2 && warp == 3)) {
    {  // whole warp; elect.sync issues (umma_*_w)
      // ---------------- MMA issuers, one per query tile (warp 1: group 0, warp 3: group 1): the
      // groups share the K / V stages (released by both issuers) but are otherwise independent,
      // so one group's softmax overlaps the other's MMAs as two CTAs per SM would.
      // S_{j+1} (or S_{j+2}) is issued before P_j is awaited.
      const int g = warp == 1 ? 0 : 1;
      constexpr uint32_t kIdS = idesc_bf16_f32(TQ, FK, false, false);  // S = Q K^T  (128 x 64)
      constexpr uint32_t kIdO = idesc_bf16_f32(TQ, HD, false, true);   // O += P V   (V MN-major)
      const uint32_t qa = smem_u32(sm.q[g]);
      // jj0: the producer's K / V tile count at this unit's start; tg: this group's tile count
      // (S / P buffers and their phases run on over the CTA's units)
      int jj0 = 0, tg = 0;
      for (int un = 0;; ++un) {
      mbar_wait(&sm.unit_full[un & 1], (un >> 1) & 1);
      const int u = sm.unit[un & 1];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.unit_empty[un & 1]);
      if (u < 0) break;
      const int qb0 = unit_pos(u).qb0;
      const int nkb = 2 * (qb0 + g) + 2, nkb_last = 2 * (qb0 + NG - 1) + 2;
      mbar_wait(&sm.q_full, un & 1);
      auto issue_s = [&](int j) {
        const int ks = (jj0 + j) % KS, sb = (tg + j) & 1;
        mbar_wait(&sm.k_full[ks], ((jj0 + j) / KS) & 1);
        if constexpr (!C::kPAlias) mbar_wait(&sm.s_free[g][sb], (((tg + j) >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sm.k[ks]);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_w(tmem + g * 128 + sb * FK, umma_desc_sw128(kmajor_k(qa, TQ, k), 16, 1024),
                    umma_desc_sw128(kmajor_k(ka, FK, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
        umma_commit_w(&sm.s_full[g][sb]);
        umma_commit_w(&sm.k_empty[ks]);
        if (j == nkb - 1) umma_commit_w(&sm.q_empty);  // the unit's last S: its Q buffer may be refilled
      };
      // S runs two tiles ahead of the softmax when a third V stage allows it: S_{j+2} goes into
      // S_j's TMEM buffer as soon as the softmax warps have loaded S_j (early in their tile j),
      // ahead of P_j V_j, so the next S is ready when the softmax finishes a tile instead of
      // queueing behind P V.  With two V stages S_{j+2} would wait for K_{j+2}, which the producer
      // loads only after P_{j-1} V_{j-1} freed a V stage -- there S_{j+1} is issued one tile ahead.
      // P aliased onto S: S_{j+2} reuses S_j's columns, which hold P_j until P_j V_j has read them,
      // so it is issued right after that P V (tcgen05 MMAs of one CTA run in issue order)
      constexpr bool kEarly = C::kEarly && !C::kPAlias;
      issue_s(0);
      if ((kEarly || C::kPAlias) && nkb > 1) issue_s(1);
      for (int j = 0; j < nkb; ++j) {
        if (kEarly && j + 2 < nkb) issue_s(j + 2);
        if (!kEarly && !C::kPAlias && j + 1 < nkb) issue_s(j + 1);
        const int pb = (tg + j) & 1, vs = (jj0 + j) % VS;
        mbar_wait(&sm.v_full[vs], ((jj0 + j) / VS) & 1);
        mbar_wait(&sm.p_full[g][pb], ((tg + j) >> 1) & 1);
        // the first P V of a unit overwrites O: the softmax warps have read the previous unit's O
        if (j == 0 && un > 0) mbar_wait(&sm.o_free[g], (un - 1) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(sm.v[vs]);
        if constexpr (C::kPTmem) {
#pragma unroll
          for (int k = 0; k < FK / 16; ++k)  // P from TMEM: 8 packed columns per 16 keys
            umma_bf16_ts_w(tmem + 128, tmem + 192 + pb * 32 + k * 8, umma_desc_sw128(va + k * 2048, FK * 128, 1024),
                           kIdO, (j > 0 || k > 0) ? 1u : 0u);  // k: the MMA's K step
        } else if constexpr (C::kPAlias) {
#pragma unroll
          for (int k = 0; k < FK / 16; ++k)  // P in the first 32 columns of its S buffer
            umma_bf16_ts_w(tmem + NG * 128 + g * HD, tmem + g * 128 + pb * FK + k * 8,
                           umma_desc_sw128(va + k * 2048, FK * 128, 1024), kIdO, (j > 0 || k > 0) ? 1u : 0u);
        } else {
          const uint32_t pa = smem_u32(sm.p[g][pb]);
#pragma unroll
          for (int k = 0; k < FK / 16; ++k)  // V MN-major: chunks of 64 hd columns FK*128 bytes apart
            umma_bf16_w(tmem + NG * 128 + g * HD, umma_desc_sw128(pa + k * 32, 16, 1024),
                        umma_desc_sw128(va + k * 2048, FK * 128, 1024), kIdO, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit_w(&sm.p_free[g][pb]);
        umma_commit_w(&sm.v_empty[vs]);
        if (C::kPAlias && j + 2 < nkb) issue_s(j + 2);
      }
      umma_commit_w(&sm.o_full[g]);
      // NG = 2: the second tile's two extra K / V tiles are released by group 0 too (once loaded,
      // so the arrival counts toward that use of the stage), or the next unit's loads would wait
      for (int j = nkb; j < nkb_last; ++j) {
        const int ks = (jj0 + j) % KS, vs = (jj0 + j) % VS;
        mbar_wait(&sm.k_full[ks], ((jj0 + j) / KS) & 1);
        umma_commit_w(&sm.k_empty[ks]);
        mbar_wait(&sm.v_full[vs], ((jj0 + j) / VS) & 1);
        umma_commit_w(&sm.v_empty[vs]);
      }
      jj0 += nkb_last;
      tg += nkb;
      }
    }
  } else if (warp >= C::kSoftWarp0) {
    // ---------------- softmax: one query row per thread, online with lazy rescaling
    const int g = (warp - C::kSoftWarp0) >> 2, wq = warp & 3;  // group, TMEM lane quarter (= warp % 4)
    const int r = wq * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t tS = trow + g * 128, tO = trow + NG * 128 + g * HD;
    long long w_s = 0, w_p = 0, t_first = 0;
    int tg = 0, nkb = 0;  // tg: this group's tile count over the CTA's units (S / P buffer phases)
    for (int un = 0;; ++un) {
    mbar_wait(&sm.unit_full[un & 1], (un >> 1) & 1);
    const int u = sm.unit[un & 1];
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.unit_empty[un & 1]);
    if (u < 0) break;
    const UnitPos w = unit_pos(u);
    const int qb = w.qb0 + g, q = qb * TQ + r, row0 = w.row0, h = w.h, bh = w.bh;
    nkb = 2 * qb + 2;
    float m = -INFINITY, l = 0.f;  // m: running max of S * scale_log2
    for (int j = 0; j < nkb; ++j) {
      const int jt = tg + j, sb = jt & 1, pb = jt & 1;
      const long long t0 = (kDbg && dbg) ? clock64() : 0;
      mbar_wait(&sm.s_full[g][sb], (jt >> 1) & 1);
      if (kDbg && dbg) {  // CKF_ATTN_DEBUG timings only
        const long long t1 = clock64();
        if (j == 0 && un == 0) t_first = t1 - t_start;
        w_s += t1 - t0;
      }
      tc_fence_after();
      uint32_t u[64];
      tmem_ld32(tS + sb * FK, *reinterpret_cast<uint32_t(*)[32]>(&u[0]));
      tmem_ld32(tS + sb * FK + 32, *reinterpret_cast<uint32_t(*)[32]>(&u[32]));
      tmem_ld_wait();
      if constexpr (!C::kPAlias) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[g][sb]);
      }
      const int kbase = j * FK;
      const int nvalid = min(FK, q - kbase + 1);  // keys <= q are visible (causal)
      const uint32_t prow = C::kPTmem || C::kPAlias ? 0u : smem_u32(sm.p[g][pb]) + r * 128;
      // P = 2^(S scale - mc) -> bf16 -> swizzled smem (32 keys at a time); returns the row sum
      // the causal mask only on the last two key tiles (j >= 2 qb: keys above some query of the
      // tile), a warp-uniform branch between two copies of the loop, not selects on every tile
      const bool diag = j >= nkb - 2;
      auto write_p_t = [&](auto mask_tag, float mc) -> float {
        constexpr bool kMask = decltype(mask_tag)::value;
        const f32x2 sc2 = f2(scale_log2, scale_log2), nm2 = f2(-mc, -mc);
        float lt = 0.f;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t w[16];
          f32x2 l2[2] = {0ull, 0ull};  // (+0.f, +0.f) pairs
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            const int tt = hf * 32 + t;
            const f32x2 xx = ffma2(f2(__uint_as_float(u[tt]), __uint_as_float(u[tt + 1])), sc2, nm2);
            float p0, p1;
            if ((t >> 1) % 8 < POLY) {
              f2split(ex2_fma2(xx), p0, p1);
            } else {
              float x0, x1;
              f2split(xx, x0, x1);
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            if (kMask) {
              p0 = tt < nvalid ? p0 : 0.f;
              p1 = tt + 1 < nvalid ? p1 : 0.f;
            }
            l2[(t >> 1) & 1] = fadd2(l2[(t >> 1) & 1], f2(p0, p1));
            w[t / 2] = pack_bf16(p0, p1);
          }
          float la, lb;
          f2split(fadd2(l2[0], l2[1]), la, lb);
          lt += la + lb;
          if constexpr (C::kPTmem) {
            tmem_st16(trow + 192 + pb * 32 + hf * 16, w);
          } else if constexpr (C::kPAlias) {
            tmem_st16(tS + sb * FK + hf * 16, w);  // over the S values this thread has loaded
          } else {
#pragma unroll
            for (int pc = 0; pc < 4; ++pc)
              st_shared_v4(prow + (((hf * 4 + pc) ^ (r & 7)) << 4), w[4 * pc], w[4 * pc + 1], w[4 * pc + 2],
                           w[4 * pc + 3]);
          }
        }
        return lt;
      };
      auto write_p = [&](float mc) -> float {
        return diag ? write_p_t(std::true_type{}, mc) : write_p_t(std::false_type{}, mc);
      };
      const long long t2 = (kDbg && dbg) ? clock64() : 0;
      mbar_wait(&sm.p_free[g][pb], ((jt >> 1) & 1) ^ 1);  // P V_{j-2} has read this P buffer
      if (kDbg && dbg) w_p += clock64() - t2;
      // Fast path (every tile after the first): P against the running max m with no max pass;
      // kept when the tile's row sum stays <= 2^16 (so every P <= 2^16, finite).  Otherwise --
      // a score above m + 16 in log2 units, or the first tile -- the tile is redone against its
      // own max with the lazy rescale of O and l (only when it exceeds m by > kRescale).
      float lt = 0.f;
      bool slow = j == 0;
      if (!slow) {
        lt = write_p(m);
        slow = __any_sync(0xffffffffu, !(lt <= 65536.f));
      }
      if (slow) {
        // row max of the visible scores: 4 independent 3-input max chains
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (nvalid >= FK) {
#pragma unroll
          for (int t = 0; t < FK; t += 2)
            mx4[(t >> 1) & 3] = fmax3(mx4[(t >> 1) & 3], __uint_as_float(u[t]), __uint_as_float(u[t + 1]));
        } else {
#pragma unroll
          for (int t = 0; t < FK; t += 2)
            mx4[(t >> 1) & 3] = fmax3(mx4[(t >> 1) & 3], t < nvalid ? __uint_as_float(u[t]) : -INFINITY,
                                      t + 1 < nvalid ? __uint_as_float(u[t + 1]) : -INFINITY);
        }
        const float mx = fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]) * scale_log2;
        // lazy rescale: only when this tile's max exceeds the running max by > kRescale
        const bool need = mx > m + kRescale;
        const float mn = need ? mx : m;
        const float alpha = need ? ex2(m - mn) : 1.f;  // m = -inf on the first tile -> 0
        if (__any_sync(0xffffffffu, need) && j > 0) {
          // the previous P V must have landed before this warp rewrites its O rows
          mbar_wait(&sm.p_free[g][(jt - 1) & 1], ((jt - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int hf = 0; hf < HD / 32; ++hf) {
            uint32_t ov[32];
            tmem_ld32(tO + hf * 32, ov);
            tmem_ld_wait();
#pragma unroll
            for (int t = 0; t < 32; ++t) ov[t] = __float_as_uint(__uint_as_float(ov[t]) * alpha);
            tmem_st32(tO + hf * 32, ov);
          }
          tmem_st32_wait();
        }
        l *= alpha;
        m = mn;
        lt = write_p(m);
      }
      l += lt;
      if constexpr (C::kPTmem || C::kPAlias)
        tmem_st_wait();  // P in TMEM before the MMA reads it
      else
        fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[g][pb]);
    }
    // ---------------- epilogue: O / l -> bf16, lse; then O is free for the next unit's P V
    mbar_wait(&sm.o_full[g], un & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const size_t ldo = static_cast<size_t>(H) * HD;
    __nv_bfloat16* orow = o + (static_cast<size_t>(row0) + q) * ldo + static_cast<size_t>(h) * HD;
#pragma unroll
    for (int hf = 0; hf < HD / 32; ++hf) {
      uint32_t u[32];
      tmem_ld32(tO + hf * 32, u);
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
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.o_free[g]);
    tg += nkb;
    }
    if (kDbg && dbg && !ctr && threadIdx.x == C::kSoftWarp0 * 32) {
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
  if (warp == C::kAllocWarp) tmem_free<C::kTmemCols>(tmem);
}

// ---------------------------------------------------------------- backward
// D[bh*T + q] = sum_c dO[q, c] O[q, c]   (HD/8 lanes per (token, head), 16-byte loads)
template <int HD>
__global__ void dsum_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout, int B, int T,
                            int H, float* __restrict__ D) {
  constexpr int LP = HD / 8;  // lanes per row
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  const long long row = i / LP;
  const int part = static_cast<int>(i % LP);
  const bool live = row < static_cast<long long>(B) * T * H;
  float acc = 0.f;
  if (live) {
    const size_t off = static_cast<size_t>(row) * HD + 8 * part;  // o / dout are [tok][H][HD]: row = tok * H + h
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
  for (int s = LP / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (live && part == 0) {
    const long long tok = row / H;
    const int h = static_cast<int>(row % H);
    const int b = static_cast<int>(tok / T), q = static_cast<int>(tok % T);
    D[(static_cast<size_t>(b) * H + h) * T + q] = acc;
  }
}

// Both backward kernels are persistent (one CTA per SM) over work units sorted longest-first,
// with 64-wide inner tiles and TWO tiles in flight per CTA: two S/dP TMEM buffers (128
// columns each) and two groups of 4 softmax warps (group b owns every tile of parity b, one
// TMEM lane quarter per warp).  While group b turns S(i) into P / dS, the tensor core runs
// group 1-b's S(i+1) and the dV / dK (dQ) MMAs of tile i-1.  The unit operands (K/V or Q/dO)
// and the TMEM accumulator sets are double-buffered where they fit (head_dim 64; head_dim 128
// keeps one of each in the dK dV kernel), and a unit's epilogue runs one tile late,
// overlapping the next unit.  Tile / unit counters run across units, so every mbarrier keeps a
// single phase sequence.
// Persistent backward kernels: each CTA walks pairs of units of the same (sequence, head) -- the
// longest (index pi) then the shortest (index n-1-pi) -- so every pair has the same total length
// (load balance without a longest-first order across heads) and the units that share operand
// tiles (the K tiles of dQ, the Q / dO tiles of dK dV) run at the same time.  Unit ids keep the u = idx * BH + bh encoding (idx 0 = longest).
struct UnitIter {
  int s, half;
};
__device__ __forceinline__ bool next_unit(UnitIter& it, int n, int BH, int& u) {
  const int npairs = (n + 1) / 2;
  while (it.s < npairs * BH) {
    // sequence x head major: the pairs of one (sequence, head) run side by side on neighbouring
    // CTAs, so each K (dQ) / Q, dO (dK dV) tile comes from DRAM about once
    const int bh = it.s / npairs, pi = it.s - bh * npairs;
    const int idx = it.half ? n - 1 - pi : pi;
    const bool valid = !(it.half && n - 1 - pi == pi);  // odd n: the middle unit once
    if (it.half) {
      it.half = 0;
      it.s += static_cast<int>(gridDim.x);
    } else {
      it.half = 1;
    }
    if (valid) {
      u = idx * BH + bh;
      return true;
    }
  }
  return false;
}

constexpr int PT = 64;                 // inner tile: queries (dK/dV kernel) or keys (dQ kernel)
constexpr uint32_t kPB = TQ * PT * 2;  // 16 KiB: P^T / dS^T [128 rows][64 cols] bf16, one SW128 chunk

// Stored dS^T, causal tiles only: key block j (64 keys) keeps query blocks t = 2 (j / 2) .. n64 - 1
// (from its 128-key unit's diagonal on), rows of one sequence x head in key-block order:
//   tile(bh, j, t) = bh * ds_tiles(n64) + ds_row(n64, j) + t - 2 (j / 2)
__host__ __device__ __forceinline__ int ds_row(int n64, int j) {
  const int p = j >> 1;
  return 2 * p * (n64 - p + 1) + (j & 1) * (n64 - 2 * p);
}
__host__ __device__ __forceinline__ int ds_tiles(int n64) { return n64 * n64 / 2 + n64; }

template <int HD>
struct BwdCfg {
  static constexpr uint32_t kUnit = TK * HD * 2;   // 128-row unit operand tile
  static constexpr uint32_t kInner = PT * HD * 2;  // 64-row inner tile
  static constexpr int kNU = HD == 64 ? 2 : 1;     // unit operand buffers (dK dV kernel)
  static constexpr int kSt = HD == 64 ? 5 : 3;     // inner-tile stages (dK dV kernel)
  static constexpr int kNAcc = HD == 64 ? 2 : 1;   // dV|dK accumulator sets (2 x HD columns each)
  static constexpr int kNUq = HD == 64 ? 2 : 1;    // unit operand buffers (dQ kernel)
  static constexpr int kStq = HD == 64 ? 5 : 3;    // inner-tile stages (dQ kernel)
};

template <int HD>
struct SmemKVpp {
  using C = BwdCfg<HD>;
  uint8_t k[C::kNU][C::kUnit], v[C::kNU][C::kUnit];  // unit operands (128 keys)
  uint8_t q[C::kSt][C::kInner], d_o[C::kSt][C::kInner];
  uint8_t p[2][kPB], ds[2][kPB];  // per softmax group
  float lse[C::kSt][PT], dsum[C::kSt][PT];
  uint64_t kv_full[C::kNU], kv_empty[C::kNU], qd_full[C::kSt], qd_empty[C::kSt], s_full[2], s_free[2], pd_full[2],
      pd_free[2], acc_full[C::kNAcc], acc_free[C::kNAcc];
  uint32_t tmem;
};

// Unit u = (key tile kb, sequence x head bh), kb-major: kb = 0 (longest) first.
//   S^T = K Q^T, dP^T = V dO^T (TMEM) -> P^T = exp(S^T - lse), dS^T = P^T (dP^T - D) (softmax,
//   row = key) -> dV += P^T dO, dK += dS^T Q (TMEM accumulators, B operands MN-major)
// SPLIT: softmax warps per TMEM lane quarter per group -- 2 splits each key row's 64 queries
// between two warps (32 each): P and dS are elementwise given lse / D, so the halves never
// communicate, and twice the warps per SM sub-partition hide the latency of the per-thread
// chains (the single-warp softmax issued one instruction every few cycles).
template <int HD, int POLY, int SPLIT>
__global__ void __launch_bounds__(128 + 256 * SPLIT, 1)
    attn_dkdv_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv128, const __grid_constant__ CUtensorMap tm_qkv64,
                        const __grid_constant__ CUtensorMap tm_do64, const __grid_constant__ CUtensorMap tm_dst,
                        int store_ds, const float* __restrict__ lse,
                        const float* __restrict__ D, int T, int H, int BH, __nv_bfloat16* __restrict__ dqkv,
                        float scale, float scale_log2, const float2* __restrict__ rope, long long* __restrict__ dbg) {
  using C = BwdCfg<HD>;
  constexpr int NU = C::kNU, ST = C::kSt, NA = C::kNAcc;
  constexpr bool kTwoIss = CKF_ATTN_BWD_ISSUERS == 2;
  // CKF_ATTN_DEBUG timings (compiled in only with -DCKF_ATTN_DEBUG_BUILD=1): [0] tiles, [1] softmax
  // wait S, [2] wait pd_free, [3] compute, [4] epilogue, [5] total, [8] MMA issue_s (+ its waits),
  // [9] acc_free wait, [10] pd_full wait -- softmax numbers from warp 4 (group 0, lane quarter 0)
  const long long t_start = kDbg ? clock64() : 0;
  long long tw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  extern __shared__ uint8_t smem_raw[];
  SmemKVpp<HD>& sm =
      *reinterpret_cast<SmemKVpp<HD>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int nunits = nqb * BH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv128);
    tma_prefetch(&tm_qkv64);
    tma_prefetch(&tm_do64);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < NU; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], 4 * SPLIT);
      mbar_init(&sm.pd_full[i], 4 * SPLIT);
      mbar_init(&sm.pd_free[i], 1);
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 8 * SPLIT);
    }
    for (int i = 0; i < ST; ++i) {
      mbar_init(&sm.qd_full[i], 1);
      mbar_init(&sm.qd_empty[i], kTwoIss ? 2 : 1);  // two issuers: released by both (S/dP and dV/dK)
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // S^T[b] cols 128b..+63, dP^T[b] 128b+64..; accumulator set a: dV at 256 + 2 HD a, dK + HD
  const uint32_t tmem = sm.tmem;

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lu = 0;
      UnitIter it_{static_cast<int>(blockIdx.x), 0};
      for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
        const int kb = u / BH, bh = u - kb * BH, b = bh / H, h = bh - b * H;
        const int row0 = b * T;
        const int kbuf = lu % NU;
        mbar_wait(&sm.kv_empty[kbuf], ((lu / NU) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.kv_full[kbuf], 2 * C::kUnit);
        tma_tile<HD>(sm.k[kbuf], &tm_qkv128, &sm.kv_full[kbuf], (H + h) * HD, row0 + kb * TK, TK);
        tma_tile<HD>(sm.v[kbuf], &tm_qkv128, &sm.kv_full[kbuf], (2 * H + h) * HD, row0 + kb * TK, TK);
        const int ntiles = 2 * (nqb - kb);
        for (int i = 0; i < ntiles; ++i, ++g) {
          const int st = g % ST;
          mbar_wait(&sm.qd_empty[st], ((g / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.qd_full[st], 2 * C::kInner + 2 * PT * 4);
          const int q0 = kb * TK + i * PT;
          tma_tile<HD>(sm.q[st], &tm_qkv64, &sm.qd_full[st], h * HD, row0 + q0, PT);
          tma_tile<HD>(sm.d_o[st], &tm_do64, &sm.qd_full[st], h * HD, row0 + q0, PT);
          const size_t qo = static_cast<size_t>(bh) * T + q0;
          bulk_load(sm.lse[st], lse + qo, PT * 4, &sm.qd_full[st]);
          bulk_load(sm.dsum[st], D + qo, PT * 4, &sm.qd_full[st]);
        }
      }
    }
  } else if (kTwoIss && (warp == 1 || warp == 3)) {
    // two issuer warps (whole warp each; elect.sync issues).  Warp 1: S^T = K Q^T and dP^T = V dO^T
    // of every tile into its group's buffer, as soon as the tile's Q / dO stage is loaded and the
    // group's softmax has read the buffer's previous tile; it releases the K / V unit buffer.
    // Warp 3: dV += P^T dO, dK += dS^T Q in tile order (deterministic accumulation).  A Q / dO
    // stage is free once both have read it.
    constexpr uint32_t kIdS = idesc_bf16_f32(TK, PT, false, false);  // [keys x 64 q], K = hd
    constexpr uint32_t kIdA = idesc_bf16_f32(TK, HD, false, true);   // [keys x hd], K = 64 q, B MN-major
    int g = 0, lu = 0;
    UnitIter it_{static_cast<int>(blockIdx.x), 0};
    if (warp == 1) {
      for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
        const int ntiles = 2 * (nqb - u / BH);
        const int kbuf = lu % NU;
        mbar_wait(&sm.kv_full[kbuf], (lu / NU) & 1);
        const uint32_t ka = smem_u32(sm.k[kbuf]), va = smem_u32(sm.v[kbuf]);
        for (int i = 0; i < ntiles; ++i) {
          const long long ti = kDbg ? clock64() : 0;
          const int gi = g + i, st = gi % ST, bb = gi & 1;
          mbar_wait(&sm.qd_full[st], (gi / ST) & 1);
          mbar_wait(&sm.s_free[bb], ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
          const uint32_t sd = tmem + static_cast<uint32_t>(bb * 128);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            if constexpr (kBwdExp == 2) continue;
            umma_bf16_w(sd, umma_desc_sw128(kmajor_k(ka, TK, k), 16, 1024),
                        umma_desc_sw128(kmajor_k(qa, PT, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
            umma_bf16_w(sd + 64, umma_desc_sw128(kmajor_k(va, TK, k), 16, 1024),
                        umma_desc_sw128(kmajor_k(oa, PT, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit_w(&sm.s_full[bb]);
          umma_commit_w(&sm.qd_empty[st]);
          if (kDbg) tw[0] += clock64() - ti;
        }
        umma_commit_w(&sm.kv_empty[kbuf]);
        g += ntiles;
      }
    } else {
      for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
        const int ntiles = 2 * (nqb - u / BH);
        const int aset = lu % NA;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(aset * 2 * HD);
        const long long ta = kDbg ? clock64() : 0;
        mbar_wait(&sm.acc_free[aset], ((lu / NA) & 1) ^ 1);
        if (kDbg) tw[1] += clock64() - ta;
        for (int i = 0; i < ntiles; ++i) {
          const int gi = g + i, st = gi % ST, bb = gi & 1;
          const long long tp = kDbg ? clock64() : 0;
          mbar_wait(&sm.pd_full[bb], (gi >> 1) & 1);
          if (kDbg) tw[2] += clock64() - tp;
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
          const uint32_t pa = smem_u32(sm.p[bb]), da = smem_u32(sm.ds[bb]);
#pragma unroll
          for (int k = 0; k < PT / 16; ++k) {  // B MN-major: HD/64 chunks of [64 q][128 B], PT*128 apart
            if constexpr (kBwdExp == 2) continue;
            umma_bf16_w(acc, umma_desc_sw128(pa + k * 32, 16, 1024), umma_desc_sw128(oa + k * 2048, PT * 128, 1024),
                        kIdA, (i > 0 || k > 0) ? 1u : 0u);
            umma_bf16_w(acc + HD, umma_desc_sw128(da + k * 32, 16, 1024),
                        umma_desc_sw128(qa + k * 2048, PT * 128, 1024), kIdA, (i > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit_w(&sm.pd_free[bb]);
          umma_commit_w(&sm.qd_empty[st]);
        }
        umma_commit_w(&sm.acc_full[aset]);
        g += ntiles;
      }
    }
    if (kDbg && dbg && lane == 0) {
      long long* d = dbg + 16 * blockIdx.x;
      if (warp == 1) d[8] = tw[0];
      if (warp == 3) {
        d[9] = tw[1];
        d[10] = tw[2];
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop; elect.sync picks the issuing lane (umma_*_w)
      constexpr uint32_t kIdS = idesc_bf16_f32(TK, PT, false, false);  // [keys x 64 q], K = hd
      constexpr uint32_t kIdA = idesc_bf16_f32(TK, HD, false, true);   // [keys x hd], K = 64 q, B MN-major
      int g = 0, lu = 0;
      UnitIter it_{static_cast<int>(blockIdx.x), 0};
      for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
        const int ntiles = 2 * (nqb - u / BH);
        const int kbuf = lu % NU, aset = lu % NA;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(aset * 2 * HD);
        mbar_wait(&sm.kv_full[kbuf], (lu / NU) & 1);
        const uint32_t ka = smem_u32(sm.k[kbuf]), va = smem_u32(sm.v[kbuf]);
        auto issue_s = [&](int gi) {  // S^T = K Q^T, dP^T = V dO^T of global tile gi into buffer gi & 1
          const long long ti = kDbg ? clock64() : 0;
          const int st = gi % ST, bb = gi & 1;
          mbar_wait(&sm.qd_full[st], (gi / ST) & 1);
          mbar_wait(&sm.s_free[bb], ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
          const uint32_t sd = tmem + static_cast<uint32_t>(bb * 128);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            if constexpr (kBwdExp == 2) continue;
            umma_bf16_w(sd, umma_desc_sw128(kmajor_k(ka, TK, k), 16, 1024),
                      umma_desc_sw128(kmajor_k(qa, PT, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
            umma_bf16_w(sd + 64, umma_desc_sw128(kmajor_k(va, TK, k), 16, 1024),
                      umma_desc_sw128(kmajor_k(oa, PT, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit_w(&sm.s_full[bb]);
          if (kDbg) tw[0] += clock64() - ti;
        };
        // S/dP run LA tiles ahead of the dV/dK MMAs.  LA = 3 (five Q/dO stages, head_dim 64):
        // tile i+3 goes into tile i+1's S/dP buffer as soon as the OTHER group's softmax has read
        // it, before this iteration waits for tile i's P / dS -- with LA = 2 it was queued behind
        // tile i's dV/dK and the next softmax waited on it (ncu: long-scoreboard at s_full).
        // LA = 2 needs four stages (with two, tile i+2 reuses the stage tile i's dV/dK still
        // reads; with three its load waits on tile i-1's MMAs: 13 % slower at hd 128).
        constexpr int LA = ST >= 5 ? 3 : ST >= 4 ? 2 : 0;
        issue_s(g);
        issue_s(g + 1);
        if (LA >= 3 && ntiles > 2) issue_s(g + 2);
        const long long ta = kDbg ? clock64() : 0;
        mbar_wait(&sm.acc_free[aset], ((lu / NA) & 1) ^ 1);
        if (kDbg) tw[1] += clock64() - ta;
        for (int i = 0; i < ntiles; ++i) {
          const int gi = g + i, st = gi % ST, bb = gi & 1;
          if constexpr (LA >= 2)
            if (i + LA < ntiles) issue_s(gi + LA);
          const long long tp = kDbg ? clock64() : 0;
          mbar_wait(&sm.pd_full[bb], (gi >> 1) & 1);
          if (kDbg) tw[2] += clock64() - tp;
          tc_fence_after();
          const uint32_t qa = smem_u32(sm.q[st]), oa = smem_u32(sm.d_o[st]);
          const uint32_t pa = smem_u32(sm.p[bb]), da = smem_u32(sm.ds[bb]);
#pragma unroll
          for (int k = 0; k < PT / 16; ++k) {  // B MN-major: HD/64 chunks of [64 q][128 B], PT*128 apart
            if constexpr (kBwdExp == 2) continue;
            umma_bf16_w(acc, umma_desc_sw128(pa + k * 32, 16, 1024), umma_desc_sw128(oa + k * 2048, PT * 128, 1024),
                      kIdA, (i > 0 || k > 0) ? 1u : 0u);
            umma_bf16_w(acc + HD, umma_desc_sw128(da + k * 32, 16, 1024),
                      umma_desc_sw128(qa + k * 2048, PT * 128, 1024), kIdA, (i > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit_w(&sm.pd_free[bb]);
          umma_commit_w(&sm.qd_empty[st]);
          if constexpr (ST < 4)
            if (i + 2 < ntiles) issue_s(gi + 2);
        }
        umma_commit_w(&sm.acc_full[aset]);
        umma_commit_w(&sm.kv_empty[kbuf]);
        g += ntiles;
      }
      if (kDbg && dbg && lane == 0) {
        long long* d = dbg + 16 * blockIdx.x;
        d[8] = tw[0];
        d[9] = tw[1];
        d[10] = tw[2];
      }
    }
  } else if (warp >= 4) {
    // sw = grp * 4 SPLIT + half * 4 + quarter
    const int sw = warp - 4, quarter = sw & 3, half = (sw >> 2) % SPLIT, grp = sw / (4 * SPLIT);
    constexpr int QW = PT / SPLIT;  // queries of a tile per softmax thread
    const int r = quarter * 32 + lane;  // key row within the unit
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t pbase = smem_u32(sm.p[grp]), dbase = smem_u32(sm.ds[grp]);
    const size_t ld = static_cast<size_t>(3) * H * HD;
    // unit epilogue (group 0 -> dV, group 1 -> dK x scale), run after this group's first tile of
    // the next unit so the accumulator set has long been complete
    auto epilogue = [&](int eu, int elu) {
      const int ekb = eu / BH, ebh = eu - ekb * BH, eb = ebh / H, eh = ebh - eb * H;
      const int aset = elu % NA;
      mbar_wait(&sm.acc_full[aset], (elu / NA) & 1);
      tc_fence_after();
      __nv_bfloat16* dst = dqkv + (static_cast<size_t>(eb) * T + ekb * TK + r) * ld +
                           static_cast<size_t>(grp ? (H + eh) * HD : (2 * H + eh) * HD);
      const float mul = grp ? scale : 1.f;
      if constexpr (SPLIT == 1) {  // dK with the inverse RoPE of key position ekb * TK + r when rope is given
        store_head_row<HD>(trow + 256 + aset * 2 * HD + grp * HD, mul, dst, grp ? rope : nullptr, ekb * TK + r, T);
      } else {
#pragma unroll 1
      for (int c0 = half * (HD / SPLIT); c0 < (half + 1) * (HD / SPLIT); c0 += 32) {
        uint32_t w32[32];
        tmem_ld32(trow + 256 + aset * 2 * HD + grp * HD + c0, w32);
        tmem_ld_wait();
#pragma unroll
        for (int piece = 0; piece < 4; ++piece) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(w32[8 * piece + 0]) * mul, __uint_as_float(w32[8 * piece + 1]) * mul);
          w.y = pack_bf16(__uint_as_float(w32[8 * piece + 2]) * mul, __uint_as_float(w32[8 * piece + 3]) * mul);
          w.z = pack_bf16(__uint_as_float(w32[8 * piece + 4]) * mul, __uint_as_float(w32[8 * piece + 5]) * mul);
          w.w = pack_bf16(__uint_as_float(w32[8 * piece + 6]) * mul, __uint_as_float(w32[8 * piece + 7]) * mul);
          reinterpret_cast<uint4*>(dst + c0)[piece] = w;
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
    };
    int pend_u = -1, pend_lu = 0;
    int g = 0, lu = 0;
    UnitIter it_{static_cast<int>(blockIdx.x), 0};
    for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
      const int ntiles = 2 * (nqb - u / BH);
      for (int i = grp; i < ntiles; i += 2) {
        const int gi = g + i, st = gi % ST;
        const long long t0 = kDbg ? clock64() : 0;
        mbar_wait(&sm.s_full[grp], (gi >> 1) & 1);
        mbar_wait(&sm.qd_full[st], (gi / ST) & 1);  // (complete) lse / D of this tile visible
        const long long t1 = kDbg ? clock64() : 0;
        if (kDbg) {
          tw[0] += 1;
          tw[1] += t1 - t0;
        }
        tc_fence_after();
        uint32_t us[QW], ud[QW];
#pragma unroll
        for (int c = 0; c < QW; c += 32) {
          tmem_ld32(trow + grp * 128 + half * QW + c, *reinterpret_cast<uint32_t(*)[32]>(&us[c]));
          tmem_ld32(trow + grp * 128 + 64 + half * QW + c, *reinterpret_cast<uint32_t(*)[32]>(&ud[c]));
        }
        tmem_ld_wait();
        if (kDbg) tw[5] += clock64() - t1;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[grp]);
        // P^T / dS^T are computed into packed registers while this group's previous dV / dK MMAs
        // may still be reading the shared buffers; the wait for them comes just before the stores
        uint32_t pkp[QW / 2], pkd[QW / 2];
        const uint32_t rowoff = static_cast<uint32_t>(r * 128);
        const uint32_t la_ = smem_u32(&sm.lse[st][0]), da_ = smem_u32(&sm.dsum[st][0]);
#pragma unroll
        for (int lg = 0; lg < QW / 8; ++lg) {  // 8 queries at a time: P^T, dS^T -> bf16 -> packed registers
          if constexpr (kBwdExp == 1) {
#pragma unroll
            for (int e = 0; e < 4; ++e) pkp[4 * lg + e] = pkd[4 * lg + e] = us[8 * lg + e] ^ ud[8 * lg + e];
            continue;
          }
          const int g8 = half * (QW / 8) + lg;
          const uint4 la = ld_shared_v4(la_ + 32 * g8), lb = ld_shared_v4(la_ + 32 * g8 + 16);
          const uint4 da4 = ld_shared_v4(da_ + 32 * g8), db4 = ld_shared_v4(da_ + 32 * g8 + 16);
          const float lq[8] = {__uint_as_float(la.x), __uint_as_float(la.y), __uint_as_float(la.z),
                               __uint_as_float(la.w), __uint_as_float(lb.x), __uint_as_float(lb.y),
                               __uint_as_float(lb.z), __uint_as_float(lb.w)};
          const float dq8[8] = {__uint_as_float(da4.x), __uint_as_float(da4.y), __uint_as_float(da4.z),
                                __uint_as_float(da4.w), __uint_as_float(db4.x), __uint_as_float(db4.y),
                                __uint_as_float(db4.z), __uint_as_float(db4.w)};
          float pv[8], dv[8];
          const f32x2 sc2 = f2(scale_log2, scale_log2), nl2 = f2(-kLog2e, -kLog2e), neg2 = f2(-1.f, -1.f);
#pragma unroll
          for (int e = 0; e < 8; e += 2) {  // pairs: P = 2^(S scale - lse log2e), dS = P (dP - D)
            const f32x2 xx = ffma2(f2(__uint_as_float(us[8 * lg + e]), __uint_as_float(us[8 * lg + e + 1])), sc2,
                                   fmul2(f2(lq[e], lq[e + 1]), nl2));
            if ((g8 * 4 + e / 2) % 8 < POLY) {  // this pair's exponentials on the FMA pipe
              f2split(ex2_fma2(xx), pv[e], pv[e + 1]);
            } else {
              float x0, x1;
              f2split(xx, x0, x1);
              pv[e] = ex2(x0);
              pv[e + 1] = ex2(x1);
            }
            f2split(fmul2(f2(pv[e], pv[e + 1]),
                          ffma2(f2(dq8[e], dq8[e + 1]), neg2,
                                f2(__uint_as_float(ud[8 * lg + e]), __uint_as_float(ud[8 * lg + e + 1])))),
                    dv[e], dv[e + 1]);
          }
          if (i < 2) {  // diagonal: query kb*128 + 64 i + c sees key kb*128 + r iff 64 i + c >= r
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (PT * i + 8 * g8 + e < r) pv[e] = dv[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            pkp[4 * lg + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
            pkd[4 * lg + e] = pack_bf16(dv[2 * e], dv[2 * e + 1]);
          }
        }
        // then the wait for this group's previous dV / dK MMAs (they read P / dS) and the previous dS^T
        // store (it reads this warp's slab), then the stores (storing each 8-query group as computed,
        // after an earlier wait, measured slower in the kernel: DESIGN.md §4.2)
        const long long t2 = kDbg ? clock64() : 0;
        mbar_wait(&sm.pd_free[grp], ((gi >> 1) & 1) ^ 1);
        if (store_ds) {
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        const long long t3 = kDbg ? clock64() : 0;
#pragma unroll
        for (int lg = 0; lg < QW / 8; ++lg) {
          const int g8 = half * (QW / 8) + lg;
          const uint32_t off = rowoff + ((g8 ^ (r & 7)) << 4);
          st_shared_v4(pbase + off, pkp[4 * lg], pkp[4 * lg + 1], pkp[4 * lg + 2], pkp[4 * lg + 3]);
          st_shared_v4(dbase + off, pkd[4 * lg], pkd[4 * lg + 1], pkd[4 * lg + 2], pkd[4 * lg + 3]);
        }
        if (kDbg) {
          tw[2] += t3 - t2;
          tw[3] += t2 - t1;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sm.pd_full[grp]);
          if (store_ds) {  // this warp's 32 key rows of dS^T -> its [64 keys x 64 queries] tile for the dQ GEMM
            const int kb = u / BH, bh = u - kb * BH, n64 = T / PT;
            const int j = kb * 2 + (quarter >> 1);  // 64-key block; 64-query block t = 2 kb + i
            tma_store_2d(&tm_dst, reinterpret_cast<const uint8_t*>(sm.ds[grp]) + quarter * 32 * 128, 0,
                         (bh * ds_tiles(n64) + ds_row(n64, j) + i) * PT + (quarter & 1) * 32);
            bulk_commit();
          }
        }
        if (kDbg) tw[6] += clock64() - t3;  // store phase (P / dS to smem, fence, arrive, dS^T TMA store)
        if (i == grp && pend_u >= 0) {
          const long long t4 = kDbg ? clock64() : 0;
          epilogue(pend_u, pend_lu);
          if (kDbg) tw[4] += clock64() - t4;
          pend_u = -1;
        }
      }
      g += ntiles;
      pend_u = u;
      pend_lu = lu;
    }
    if (pend_u >= 0) epilogue(pend_u, pend_lu);
    if (store_ds && lane == 0) bulk_wait_all();
    if (kDbg && dbg && warp == 4 && lane == 0) {
      long long* d = dbg + 16 * blockIdx.x;
      for (int k = 0; k < 5; ++k) d[k] = tw[k];
      d[5] = clock64() - t_start;
      d[6] = tw[5];
      d[7] = tw[6];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<512>(tmem);
}

template <int HD>
struct SmemQpp {  // dQ kernel
  using C = BwdCfg<HD>;
  uint8_t q[C::kNUq][C::kUnit], d_o[C::kNUq][C::kUnit];  // unit operands (128 queries)
  uint8_t k[C::kStq][C::kInner], v[C::kStq][C::kInner];  // 64-key tiles
  uint8_t ds[2][kPB];                                    // per softmax group
  float lse[C::kNUq][TQ], dsum[C::kNUq][TQ];
  uint64_t qd_full[C::kNUq], qd_empty[C::kNUq], kv_full[C::kStq], kv_empty[C::kStq], s_full[2], s_free[2],
      ds_full[2], ds_free[2], acc_full[2], acc_free[2];
  uint32_t tmem;
};

// Unit u = (query tile qb, sequence x head bh), longest first; inner tiles of 64 keys.
//   S = Q K^T, dP = dO V^T (TMEM) -> dS = P (dP - D) (softmax, row = query) -> dQ += dS K
template <int HD, int POLY>
__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_dq_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv128, const __grid_constant__ CUtensorMap tm_qkv64,
                      const __grid_constant__ CUtensorMap tm_do128, const float* __restrict__ lse,
                      const float* __restrict__ D, int T, int H, int BH, __nv_bfloat16* __restrict__ dqkv, float scale,
                      float scale_log2) {
  using C = BwdCfg<HD>;
  constexpr int NU = C::kNUq, ST = C::kStq;
  extern __shared__ uint8_t smem_raw[];
  SmemQpp<HD>& sm = *reinterpret_cast<SmemQpp<HD>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int nunits = nqb * BH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv128);
    tma_prefetch(&tm_qkv64);
    tma_prefetch(&tm_do128);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < NU; ++i) {
      mbar_init(&sm.qd_full[i], 1);
      mbar_init(&sm.qd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], 4);
      mbar_init(&sm.ds_full[i], 4);
      mbar_init(&sm.ds_free[i], 1);
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 8);
    }
    for (int i = 0; i < ST; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S[b] cols 128b..+63, dP[b] 128b+64..; dQ set a: 256 + HD a

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        const int qi = u / BH, bh = u - qi * BH, b = bh / H, h = bh - b * H;
        const int qb = nqb - 1 - qi, row0 = b * T;
        const int qbuf = lu % NU;
        mbar_wait(&sm.qd_empty[qbuf], ((lu / NU) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.qd_full[qbuf], 2 * C::kUnit + 2 * TQ * 4);
        tma_tile<HD>(sm.q[qbuf], &tm_qkv128, &sm.qd_full[qbuf], h * HD, row0 + qb * TQ, TQ);
        tma_tile<HD>(sm.d_o[qbuf], &tm_do128, &sm.qd_full[qbuf], h * HD, row0 + qb * TQ, TQ);
        const size_t qo = static_cast<size_t>(bh) * T + qb * TQ;
        bulk_load(sm.lse[qbuf], lse + qo, TQ * 4, &sm.qd_full[qbuf]);
        bulk_load(sm.dsum[qbuf], D + qo, TQ * 4, &sm.qd_full[qbuf]);
        const int ntiles = 2 * (qb + 1);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int st = g % ST;
          mbar_wait(&sm.kv_empty[st], ((g / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.kv_full[st], 2 * C::kInner);
          tma_tile<HD>(sm.k[st], &tm_qkv64, &sm.kv_full[st], (H + h) * HD, row0 + j * PT, PT);
          tma_tile<HD>(sm.v[st], &tm_qkv64, &sm.kv_full[st], (2 * H + h) * HD, row0 + j * PT, PT);
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
        const int qbuf = lu % NU, aset = lu & 1;
        const uint32_t acc = tmem + 256 + static_cast<uint32_t>(aset * HD);
        mbar_wait(&sm.qd_full[qbuf], (lu / NU) & 1);
        const uint32_t qa = smem_u32(sm.q[qbuf]), oa = smem_u32(sm.d_o[qbuf]);
        auto issue_s = [&](int gj) {  // S = Q K^T, dP = dO V^T of global tile gj into buffer gj & 1
          const int st = gj % ST, bb = gj & 1;
          mbar_wait(&sm.kv_full[st], (gj / ST) & 1);
          mbar_wait(&sm.s_free[bb], ((gj >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sm.k[st]), va = smem_u32(sm.v[st]);
          const uint32_t sd = tmem + static_cast<uint32_t>(bb * 128);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            umma_bf16(sd, umma_desc_sw128(kmajor_k(qa, TQ, k), 16, 1024),
                      umma_desc_sw128(kmajor_k(ka, PT, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
            umma_bf16(sd + 64, umma_desc_sw128(kmajor_k(oa, TQ, k), 16, 1024),
                      umma_desc_sw128(kmajor_k(va, PT, k), 16, 1024), kIdS, k > 0 ? 1u : 0u);
          }
          umma_commit(&sm.s_full[bb]);
        };
        constexpr int LA = ST >= 5 ? 3 : ST >= 4 ? 2 : 0;  // S/dP lookahead (see dK dV)
        issue_s(g);
        issue_s(g + 1);
        if (LA >= 3 && ntiles > 2) issue_s(g + 2);
        mbar_wait(&sm.acc_free[aset], ((lu >> 1) & 1) ^ 1);
        for (int j = 0; j < ntiles; ++j) {
          const int gj = g + j, st = gj % ST, bb = gj & 1;
          if constexpr (LA >= 2)
            if (j + LA < ntiles) issue_s(gj + LA);
          mbar_wait(&sm.ds_full[bb], (gj >> 1) & 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sm.k[st]), da = smem_u32(sm.ds[bb]);
#pragma unroll
          for (int k = 0; k < PT / 16; ++k)
            umma_bf16(acc, umma_desc_sw128(da + k * 32, 16, 1024), umma_desc_sw128(ka + k * 2048, PT * 128, 1024),
                      kIdQ, (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&sm.ds_free[bb]);
          umma_commit(&sm.kv_empty[st]);
          if constexpr (ST < 4)
            if (j + 2 < ntiles) issue_s(gj + 2);
        }
        umma_commit(&sm.acc_full[aset]);
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
    // unit epilogue (dQ x scale; group b writes columns [b HD/2, (b+1) HD/2)), one tile late
    auto epilogue = [&](int eu, int elu) {
      const int eqi = eu / BH, ebh = eu - eqi * BH, eb = ebh / H, eh = ebh - eb * H;
      const int eq = (nqb - 1 - eqi) * TQ + r;
      const int aset = elu & 1;
      mbar_wait(&sm.acc_full[aset], (elu >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* qrow = dqkv + (static_cast<size_t>(eb) * T + eq) * ld + static_cast<size_t>(eh * HD);
#pragma unroll 1
      for (int c0 = grp * (HD / 2); c0 < (grp + 1) * (HD / 2); c0 += 32) {
        uint32_t w32[32];
        tmem_ld32(trow + 256 + aset * HD + c0, w32);
        tmem_ld_wait();
#pragma unroll
        for (int piece = 0; piece < 4; ++piece) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(w32[8 * piece + 0]) * scale, __uint_as_float(w32[8 * piece + 1]) * scale);
          w.y = pack_bf16(__uint_as_float(w32[8 * piece + 2]) * scale, __uint_as_float(w32[8 * piece + 3]) * scale);
          w.z = pack_bf16(__uint_as_float(w32[8 * piece + 4]) * scale, __uint_as_float(w32[8 * piece + 5]) * scale);
          w.w = pack_bf16(__uint_as_float(w32[8 * piece + 6]) * scale, __uint_as_float(w32[8 * piece + 7]) * scale);
          reinterpret_cast<uint4*>(qrow + c0)[piece] = w;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
    };
    int pend_u = -1, pend_lu = 0;
    int g = 0, lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      const int qb = nqb - 1 - u / BH, ntiles = 2 * (qb + 1);
      const int qbuf = lu % NU;
      mbar_wait(&sm.qd_full[qbuf], (lu / NU) & 1);  // lse / D of the unit's queries
      float l2, dq;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(l2) : "r"(smem_u32(&sm.lse[qbuf][r])));
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(dq) : "r"(smem_u32(&sm.dsum[qbuf][r])));
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
        uint32_t pkd[32];  // dS computed before the wait for this group's previous dQ MMA (see dK dV)
        const uint32_t rowoff = static_cast<uint32_t>(r * 128);
        const bool diag = j >= 2 * qb;  // keys 64 j + c vs query qb*128 + r: visible iff 64 j + c <= 128 qb + r
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {
          float dv[8];
          const f32x2 sc2 = f2(scale_log2, scale_log2), nl2 = f2(-l2, -l2), nd2 = f2(-dq, -dq);
#pragma unroll
          for (int e = 0; e < 8; e += 2) {  // pairs: dS = 2^(S scale - lse log2e) (dP - D)
            const f32x2 xx =
                ffma2(f2(__uint_as_float(us[8 * g8 + e]), __uint_as_float(us[8 * g8 + e + 1])), sc2, nl2);
            f32x2 pp;
            if ((g8 * 4 + e / 2) % 8 < POLY) {  // this pair's exponentials on the FMA pipe
              pp = ex2_fma2(xx);
            } else {
              float x0, x1;
              f2split(xx, x0, x1);
              pp = f2(ex2(x0), ex2(x1));
            }
            f2split(fmul2(pp, fadd2(f2(__uint_as_float(ud[8 * g8 + e]), __uint_as_float(ud[8 * g8 + e + 1])), nd2)),
                    dv[e], dv[e + 1]);
          }
          if (diag) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (PT * j + 8 * g8 + e > TQ * qb + r) dv[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) pkd[4 * g8 + e] = pack_bf16(dv[2 * e], dv[2 * e + 1]);
        }
        mbar_wait(&sm.ds_free[grp], ((gj >> 1) & 1) ^ 1);
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8)
          st_shared_v4(dbase + rowoff + ((g8 ^ (r & 7)) << 4), pkd[4 * g8], pkd[4 * g8 + 1], pkd[4 * g8 + 2],
                       pkd[4 * g8 + 3]);
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


// dQ from the stored dS^T (attn_dkdv_pp_kernel, store_ds): dQ[q, :] = scale sum_key dS^T[key, q] K[key, :]
// -- a causal batched GEMM with no S / dP recompute and no exponentials.  Persistent over units
// (query tile qb, sequence x head bh) longest first; 64-key inner tiles: A = dS^T tile (MN-major,
// two [64 keys][64 q] SW128 chunks), B = K tile (MN-major, HD/64 [64 keys][64 hd] chunks) by TMA
// into a 6-deep ring; dQ accumulates in TMEM (two accumulator sets, HD columns each), epilogue
// warps 4..7 scale, round and store while the next unit runs.
template <int HD>
struct SmemDQ {
  static constexpr int kSt = 6;
  uint8_t a[kSt][2 * 8192];
  uint8_t b[kSt][PT * HD * 2];
  uint64_t full[kSt], empty[kSt], acc_full[2], acc_free[2];
  uint32_t tmem;
};

template <int HD>
__global__ void __launch_bounds__(256, 1)
    attn_dq_gemm_kernel(const __grid_constant__ CUtensorMap tm_dst, const __grid_constant__ CUtensorMap tm_qkv64,
                        int T, int H, int BH, __nv_bfloat16* __restrict__ dqkv, float scale,
                        const float2* __restrict__ rope) {
  using SM = SmemDQ<HD>;
  constexpr int ST = SM::kSt;
  extern __shared__ uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ, nunits = nqb * BH;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_dst);
    tma_prefetch(&tm_qkv64);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_free[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<2 * HD>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      UnitIter it_{static_cast<int>(blockIdx.x), 0};
      for (int u = 0; next_unit(it_, nqb, BH, u);) {
        const int qi = u / BH, bh = u - qi * BH, b = bh / H, h = bh - b * H;
        const int qb = nqb - 1 - qi, ntiles = 2 * (qb + 1);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int st = g % ST;
          mbar_wait(&sm.empty[st], ((g / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.full[st], 2 * 8192 + PT * HD * 2);
          // dS^T tiles (j, 2qb) and (j, 2qb + 1), adjacent in the causal layout (2qb >= 2 (j / 2))
          const int n64 = T / PT, tile = bh * ds_tiles(n64) + ds_row(n64, j) + 2 * qb - 2 * (j >> 1);
          tma_load_2d(sm.a[st], &tm_dst, &sm.full[st], 0, tile * PT);
          tma_load_2d(sm.a[st] + 8192, &tm_dst, &sm.full[st], 0, (tile + 1) * PT);
          tma_tile<HD>(sm.b[st], &tm_qkv64, &sm.full[st], (H + h) * HD, b * T + j * PT, PT);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp; elect.sync issues (umma_*_w)
      constexpr uint32_t kId = idesc_bf16_f32(TQ, HD, true, true);
      int g = 0, lu = 0;
      UnitIter it_{static_cast<int>(blockIdx.x), 0};
      for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
        const int qb = nqb - 1 - u / BH, ntiles = 2 * (qb + 1), aset = lu & 1;
        mbar_wait(&sm.acc_free[aset], ((lu >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + static_cast<uint32_t>(aset * HD);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int st = g % ST;
          mbar_wait(&sm.full[st], (g / ST) & 1);
          tc_fence_after();
          const uint32_t aa = smem_u32(sm.a[st]), ba = smem_u32(sm.b[st]);
#pragma unroll
          for (int k = 0; k < PT / 16; ++k)
            umma_bf16_w(acc, umma_desc_sw128(aa + k * 2048, 8192, 1024), umma_desc_sw128(ba + k * 2048, PT * 128, 1024),
                      kId, (j > 0 || k > 0) ? 1u : 0u);
          umma_commit_w(&sm.empty[st]);
        }
        umma_commit_w(&sm.acc_full[aset]);
      }
    }
  } else if (warp >= 4) {
    const int quarter = warp - 4, r = quarter * 32 + lane;
    const size_t ld = static_cast<size_t>(3) * H * HD;
    int lu = 0;
    UnitIter it_{static_cast<int>(blockIdx.x), 0};
      for (int u = 0; next_unit(it_, nqb, BH, u); ++lu) {
      const int qi = u / BH, bh = u - qi * BH, b = bh / H, h = bh - b * H;
      const int q = (nqb - 1 - qi) * TQ + r, aset = lu & 1;
      mbar_wait(&sm.acc_full[aset], (lu >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* qrow = dqkv + (static_cast<size_t>(b) * T + q) * ld + static_cast<size_t>(h) * HD;
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(aset * HD);
      store_head_row<HD>(trow, scale, qrow, rope, q, T);  // (inverse RoPE of query position q when given)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_free[aset]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<2 * HD>(tmem);
}

// dS^T scratch for the stored-dS backward: B H ds_tiles(T / 64) 64 x 64 bf16 tiles per launch chunk
// (grown on demand)
bf16* dst_buffer(size_t elems) {
  static bf16* buf = nullptr;
  static size_t cap = 0;
  if (elems > cap) {
    if (buf) CKF_CUDA(cudaFree(buf));
    CKF_CUDA(cudaMalloc(&buf, elems * sizeof(bf16)));
    cap = elems;
    ++alloc_epoch();
  }
  return buf;
}

int num_sms_attn() {
  static const int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return sms;
}

// the persistent forward's unit counters (zero between launches: the kernel resets its own), per
// device: a ring of 256 taken in turn, so forwards launched on different streams at once use
// different counters
int* attn_fwd_counter() {
  constexpr int kRing = 256;
  static int* ctr[64] = {};
  static std::atomic<unsigned> next[64];
  int dev = 0;
  CKF_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) raise(1, "attention: device index out of range");
  if (!ctr[dev]) {
    CKF_CUDA(cudaMalloc(&ctr[dev], kRing * sizeof(int)));
    CKF_CUDA(cudaMemset(ctr[dev], 0, kRing * sizeof(int)));
    ++alloc_epoch();
  }
  return ctr[dev] + next[dev].fetch_add(1, std::memory_order_relaxed) % kRing;
}

template <int HD, int NG>
void fwd_launch_ng(const bf16* qkv, size_t B, size_t T, size_t H, bf16* o, float* lse, int poly, cudaStream_t s) {
  const CUtensorMap tm = tma::make_2d_bf16(qkv, 3 * H * HD, B * T, 3 * H * HD, 64, 128);
  const CUtensorMap tkv = tma::make_2d_bf16(qkv, 3 * H * HD, B * T, 3 * H * HD, 64, FK);
  const size_t smem = sizeof(Smem<HD, NG>) + 1024;
  auto kern = poly >= 4 ? attn_fwd_tc_kernel<HD, 4, NG>
              : poly == 3 ? attn_fwd_tc_kernel<HD, 3, NG>
              : poly == 2 ? attn_fwd_tc_kernel<HD, 2, NG>
              : poly == 1 ? attn_fwd_tc_kernel<HD, 1, NG> : attn_fwd_tc_kernel<HD, 0, NG>;
  static bool attr[5] = {false, false, false, false, false};
  const int pi = std::min(std::max(poly, 0), 4);
  if (!attr[pi]) {
    CKF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr[pi] = true;
  }
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(HD));
  const int nqu = static_cast<int>(T / (TQ * NG)), BH = static_cast<int>(B * H);
  // persistent CTAs; CKF_ATTN_FWD_PERSIST=0: one CTA per unit
  static const bool persist_env = [] {
    const char* v = std::getenv("CKF_ATTN_FWD_PERSIST");
    return !(v && v[0] == '0');
  }();
  long long* dbg = attn_fwd_debug_buffer();
  int* ctr = persist_env && !dbg ? attn_fwd_counter() : nullptr;
  const int units = nqu * BH;
  const dim3 grid = ctr ? dim3(static_cast<unsigned>(std::min(units, FwdCfg<HD, NG>::kMinBlocks * num_sms_attn())))
                        : dim3(static_cast<unsigned>(nqu), static_cast<unsigned>(BH));
  kern<<<grid, FwdCfg<HD, NG>::kThreads, smem, s>>>(tm, tkv, static_cast<int>(T), static_cast<int>(H), o, lse,
                                                   scale_log2, BH, ctr, dbg);
  CKF_LAUNCH_CHECK();
}

template <int HD>
void fwd_launch(const bf16* qkv, size_t B, size_t T, size_t H, bf16* o, float* lse, cudaStream_t s) {
  static const int poly = [] {
    const char* v = std::getenv("CKF_ATTN_POLY");
    return v ? std::atoi(v) : (HD == 64 ? kFwdPolyDefault : 0);
  }();
  // CKF_ATTN_FWD_NG=1|2: query tiles per CTA (2 needs seq_len % 256 == 0)
  static const int ng = [] {
    const char* v = std::getenv("CKF_ATTN_FWD_NG");
    return v ? std::atoi(v) : kFwdNgDefault<HD>;
  }();
  if (ng >= 2 && T % (2 * TQ) == 0)
    fwd_launch_ng<HD, 2>(qkv, B, T, H, o, lse, poly, s);
  else
    fwd_launch_ng<HD, 1>(qkv, B, T, H, o, lse, poly, s);
}

template <int HD>
void bwd_launch(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
                bf16* dqkv, float* Dsum, bool rope, bool d_ready, cudaStream_t s) {
  const size_t rows = B * T * H;
  if (!d_ready) {
    dsum_kernel<HD><<<static_cast<unsigned>((rows * (HD / 8) + 255) / 256), 256, 0, s>>>(
        o, dout, static_cast<int>(B), static_cast<int>(T), static_cast<int>(H), Dsum);
    CKF_LAUNCH_CHECK();
  }
  // CKF_ATTN_BWD_SPLIT=1|2: softmax warps per TMEM lane quarter per group in the dK dV kernel
  // (CKF_ATTN_BWD_POLY: FMA-pipe exponential pairs of 8 in the backward -- measured no gain, so
  // only the all-MUFU kernels are built: profiles/r02_attention_bwd_poly_sweep.jsonl)
  static const int split = [] {
    const char* v = std::getenv("CKF_ATTN_BWD_SPLIT");
    return v ? std::atoi(v) : kBwdSplitDefault;
  }();
  // dQ from the dS^T the dK dV kernel stores (one GEMM pass, no recompute) unless CKF_ATTN_DQ=recompute
  // selects the dQ kernel that recomputes S, dP and dS (the split-2 dK dV kernel stores no dS^T)
  static const bool stored_ds = [] {
    const char* v = std::getenv("CKF_ATTN_DQ");
    return !(v && std::string(v) == "recompute") && split < 2;
  }();
  auto kkv = split >= 2 ? attn_dkdv_pp_kernel<HD, 0, 2> : attn_dkdv_pp_kernel<HD, 0, 1>;
  const int kv_threads = 128 + 256 * (split >= 2 ? 2 : 1);
  auto kq = attn_dq_pp_kernel<HD, 0>;
  auto kg = attn_dq_gemm_kernel<HD>;
  const size_t smem_kv = sizeof(SmemKVpp<HD>) + 1024, smem_q = sizeof(SmemQpp<HD>) + 1024,
               smem_g = sizeof(SmemDQ<HD>) + 1024;
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(kkv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_kv)));
    CKF_CUDA(cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_q)));
    CKF_CUDA(cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_g)));
    attr = true;
  }
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  long long* dbg = attn_fwd_debug_buffer();
  // the RoPE backward of dq / dk in the dK and dQ-GEMM epilogues (otherwise a separate pass below)
  const bool rope_fused = rope && split < 2 && stored_ds;
  const float2* rtab = rope_fused ? rope_table_pair_major(T, HD, s) : nullptr;
  // sequences per pass: the dS^T scratch (B_c H ds_tiles tiles) stays within ~2.5 GB -- each pass
  // pays a partial last wave in both kernels, so few passes (profiles/r02_attention_ds_chunk_sweep.jsonl:
  // hd 128 at [16, 4096, 16, 128] 3,970 us in 8 passes, 3,462 in 2, 3,494 in 1)
  const size_t tiles_seq = H * static_cast<size_t>(ds_tiles(static_cast<int>(T / PT)));
  const size_t per_seq = tiles_seq * PT * PT * sizeof(bf16);
  static const size_t ds_bytes = [] {  // CKF_ATTN_DS_BYTES: the dS^T scratch budget per pass
    const char* v = std::getenv("CKF_ATTN_DS_BYTES");
    return v ? static_cast<size_t>(std::atoll(v)) : static_cast<size_t>(2500000000ull);
  }();
  const size_t bc = stored_ds ? std::max<size_t>(1, std::min<size_t>(B, ds_bytes / per_seq)) : B;
  bf16* dst = stored_ds ? dst_buffer(bc * tiles_seq * PT * PT) : nullptr;
  const size_t ld = 3 * H * HD;
  for (size_t b0 = 0; b0 < B; b0 += bc) {
    const size_t nb = std::min(bc, B - b0);
    const bf16* q_c = qkv + b0 * T * ld;
    const bf16* do_c = dout + b0 * T * H * HD;
    bf16* dq_c = dqkv + b0 * T * ld;
    const float* lse_c = lse + b0 * H * T;
    const float* D_c = Dsum + b0 * H * T;
    const CUtensorMap tq = tma::make_2d_bf16(q_c, ld, nb * T, ld, 64, 128);
    const CUtensorMap tq64 = tma::make_2d_bf16(q_c, ld, nb * T, ld, 64, 64);
    const CUtensorMap td = tma::make_2d_bf16(do_c, H * HD, nb * T, H * HD, 64, 128);
    const CUtensorMap td64 = tma::make_2d_bf16(do_c, H * HD, nb * T, H * HD, 64, 64);
    // dS^T as contiguous [64 keys][64 queries] tiles (8 KiB each; causal tiles only, tile (bh, key
    // block j, query block t) at row 64 ds_tile(...) of a [* x 64] matrix, ds_row above): 32-row slabs
    // stored by the dK dV warps, whole tiles loaded by dQ -- every transfer is one contiguous run of DRAM
    const size_t ds_rows = nb * tiles_seq * PT;
    const CUtensorMap tds32 = stored_ds ? tma::make_2d_bf16(dst, 64, ds_rows, 64, 64, 32) : tq;
    const CUtensorMap tds64 = stored_ds ? tma::make_2d_bf16(dst, 64, ds_rows, 64, 64, 64) : tq;
    const int BH = static_cast<int>(nb * H);
    // unit pairs (next_unit): one per CTA slot
    const int pairs = static_cast<int>((T / TQ + 1) / 2) * BH;
    const unsigned grid = static_cast<unsigned>(std::min(pairs, num_sms_attn()));
    kkv<<<grid, kv_threads, smem_kv, s>>>(tq, tq64, td64, tds32, stored_ds ? 1 : 0, lse_c, D_c, static_cast<int>(T),
                                          static_cast<int>(H), BH, dq_c, scale, scale * kLog2e, rtab,
                                          dbg ? dbg + 8 * 32768 : nullptr);
    CKF_LAUNCH_CHECK();
    if (stored_ds)
      kg<<<grid, 256, smem_g, s>>>(tds64, tq64, static_cast<int>(T), static_cast<int>(H), BH, dq_c, scale, rtab);
    else
      kq<<<grid, kThreadsBwd, smem_q, s>>>(tq, tq64, td, lse_c, D_c, static_cast<int>(T), static_cast<int>(H), BH, dq_c,
                                           scale, scale * kLog2e);
    CKF_LAUNCH_CHECK();
  }
  if (rope && !rope_fused) llama::rope(dqkv, B * T, T, H * HD, H, 1, s);
}

}  // namespace

bool attn_fwd_tc_supported(size_t T, size_t hd) { return (hd == 64 || hd == 128) && T % TQ == 0; }

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
  if (!attn_fwd_tc_supported(T, hd)) raise(1, "tcgen05 attention: head_dim 64 or 128 and seq_len % 128 == 0");
  if (hd == 64)
    fwd_launch<64>(qkv, B, T, H, o, lse, s);
  else
    fwd_launch<128>(qkv, B, T, H, o, lse, s);
}

void attn_bwd_tc(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
                 size_t hd, bf16* dqkv, float* Dsum, cudaStream_t s, bool rope_inverse, bool d_ready) {
  if (!attn_fwd_tc_supported(T, hd)) raise(1, "tcgen05 attention: head_dim 64 or 128 and seq_len % 128 == 0");
  if (hd == 64)
    bwd_launch<64>(qkv, o, lse, dout, B, T, H, dqkv, Dsum, rope_inverse, d_ready, s);
  else
    bwd_launch<128>(qkv, o, lse, dout, B, T, H, dqkv, Dsum, rope_inverse, d_ready, s);
}

}  // namespace ckf::llama
