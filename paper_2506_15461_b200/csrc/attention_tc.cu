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
#include "common.cuh"
#include "llama_kernels.h"
#include "sm100.cuh"

namespace ckf::llama {
namespace {

using namespace ckf::sm100;

constexpr int TQ = 128, TK = 128, HD = 64;
constexpr int kThreads = 256;
constexpr uint32_t kTile = TQ * HD * 2;      // 16 KiB: one 128 x 64 bf16 tile
constexpr uint32_t kPBuf = TQ * TK * 2;      // 32 KiB: P as [2 K-chunks][128 rows][128 B]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct Smem {
  // 1024-aligned tiles first
  uint8_t q[kTile];
  uint8_t k[2][kTile];
  uint8_t v[2][kTile];
  uint8_t p[2][kPBuf];
  uint64_t q_full;
  uint64_t kv_full[2], kv_empty[2];
  uint64_t s_full[2], s_free[2];
  uint64_t p_full[2], p_free[2];
  uint64_t o_full;
  uint32_t tmem;
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, int T, int H, __nv_bfloat16* __restrict__ o,
                       float* __restrict__ lse, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = T / TQ;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);  // heavy (late) query tiles first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int nkb = qb + 1;  // causal: key tiles 0..qb
  const int row0 = b * T;
  const int qcol = h * HD, kcol = (H + h) * HD, vcol = (2 * H + h) * HD;

  if (warp == 0 && lane == 0) tma_prefetch(&tm_qkv);
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], 4);
      mbar_init(&sm.p_full[i], 4);
      mbar_init(&sm.p_free[i], 1);
    }
    mbar_init(&sm.o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;  // S[0] cols 0-127, S[1] 128-255, O 256-319

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: Q once; K (pass 1) then K+V (pass 2) per key tile
      mbar_arrive_expect_tx(&sm.q_full, kTile);
      tma_load_2d(sm.q, &tm_qkv, &sm.q_full, qcol, row0 + qb * TQ);
      int c = 0;
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = 0; j < nkb; ++j, ++c) {
          const int st = c & 1;
          mbar_wait(&sm.kv_empty[st], ((c >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.kv_full[st], pass ? 2 * kTile : kTile);
          tma_load_2d(sm.k[st], &tm_qkv, &sm.kv_full[st], kcol, row0 + j * TK);
          if (pass) tma_load_2d(sm.v[st], &tm_qkv, &sm.kv_full[st], vcol, row0 + j * TK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t kIdS = idesc_bf16_f32(TQ, TK, false, false);  // S = Q K^T
      constexpr uint32_t kIdO = idesc_bf16_f32(TQ, HD, false, true);   // O += P V (V MN-major)
      mbar_wait(&sm.q_full, 0);
      const uint32_t qa = smem_u32(sm.q);
      int c = 0;  // kv loads consumed == S tiles produced
      auto issue_s = [&](int cc) {
        const int st = cc & 1, sb = cc & 1;
        mbar_wait(&sm.kv_full[st], (cc >> 1) & 1);
        mbar_wait(&sm.s_free[sb], ((cc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sm.k[st]);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + sb * TK, umma_desc_sw128(qa + k * 32, 16, 1024), umma_desc_sw128(ka + k * 32, 16, 1024),
                    kIdS, k > 0 ? 1u : 0u);
        umma_commit(&sm.s_full[sb]);
      };
      // pass 1: S tiles only (the softmax warps reduce them to the row log-sum-exp)
      for (int j = 0; j < nkb; ++j, ++c) {
        issue_s(c);
        umma_commit(&sm.kv_empty[c & 1]);
      }
      // pass 2: S_{j+1} is issued before waiting for P_j so softmax and MMA overlap
      const int c0 = c;
      issue_s(c0);
      for (int j = 0; j < nkb; ++j) {
        const int cc = c0 + j;
        if (j + 1 < nkb) issue_s(cc + 1);
        const int pb = j & 1;
        mbar_wait(&sm.p_full[pb], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(sm.p[pb]);
        const uint32_t va = smem_u32(sm.v[cc & 1]);
#pragma unroll
        for (int k = 0; k < TK / 16; ++k)
          umma_bf16(tmem + 256, umma_desc_sw128(pa + (k >> 2) * (TQ * 128) + (k & 3) * 32, 16, 1024),
                    umma_desc_sw128(va + k * 2048, 8192, 1024), kIdO, (j > 0 || k > 0) ? 1u : 0u);
        umma_commit(&sm.p_free[pb]);
        umma_commit(&sm.kv_empty[cc & 1]);
      }
      umma_commit(&sm.o_full);
    }
  } else if (warp >= 4) {
    // ---------------- softmax: one query row per thread
    const int r = (warp - 4) * 32 + lane;
    const int q = qb * TQ + r;
    const uint32_t trow = tmem + (static_cast<uint32_t>((warp - 4) * 32) << 16);
    float m = -INFINITY, l = 0.f;
    int c = 0;
    auto load_s = [&](int cc, float (&s)[TK]) {
      const int sb = cc & 1;
      mbar_wait(&sm.s_full[sb], (cc >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int k4 = 0; k4 < TK / 32; ++k4) {
        uint32_t u[32];
        tmem_ld32(trow + sb * TK + k4 * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t) s[k4 * 32 + t] = __uint_as_float(u[t]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.s_free[sb]);
    };
    float s[TK];
    for (int j = 0; j < nkb; ++j, ++c) {
      load_s(c, s);
      float mx = -INFINITY;
#pragma unroll
      for (int t = 0; t < TK; ++t) {
        float x = s[t] * scale_log2;
        if (j == qb && j * TK + t > q) x = -INFINITY;
        s[t] = x;
        mx = fmaxf(mx, x);
      }
      const float mn = fmaxf(m, mx);
      float acc = 0.f;
#pragma unroll
      for (int t = 0; t < TK; ++t) acc += exp2f(s[t] - mn);
      l = l * exp2f(m - mn) + acc;
      m = mn;
    }
    const float lse2 = m + log2f(l);
    for (int j = 0; j < nkb; ++j, ++c) {
      load_s(c, s);
      const int pb = j & 1;
      mbar_wait(&sm.p_free[pb], ((j >> 1) & 1) ^ 1);
      const uint32_t prow = smem_u32(sm.p[pb]) + r * 128;
#pragma unroll
      for (int ch = 0; ch < TK / 64; ++ch) {
#pragma unroll
        for (int piece = 0; piece < 8; ++piece) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t = ch * 64 + piece * 8 + 2 * e;
            float p0 = exp2f(s[t] * scale_log2 - lse2), p1 = exp2f(s[t + 1] * scale_log2 - lse2);
            if (j == qb) {
              if (j * TK + t > q) p0 = 0.f;
              if (j * TK + t + 1 > q) p1 = 0.f;
            }
            w[e] = pack_bf16(p0, p1);
          }
          st_shared_v4(prow + ch * (TQ * 128) + ((piece ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[pb]);
    }
    // ---------------- epilogue: O (already normalised) -> bf16, lse
    mbar_wait(&sm.o_full, 0);
    tc_fence_after();
    const size_t ldo = static_cast<size_t>(H) * HD;
    __nv_bfloat16* orow = o + (static_cast<size_t>(row0) + q) * ldo + static_cast<size_t>(h) * HD;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t u[32];
      tmem_ld32(trow + 256 + half * 32, u);
      tmem_ld_wait();
#pragma unroll
      for (int piece = 0; piece < 4; ++piece) {
        uint4 v;
        v.x = pack_bf16(__uint_as_float(u[8 * piece + 0]), __uint_as_float(u[8 * piece + 1]));
        v.y = pack_bf16(__uint_as_float(u[8 * piece + 2]), __uint_as_float(u[8 * piece + 3]));
        v.z = pack_bf16(__uint_as_float(u[8 * piece + 4]), __uint_as_float(u[8 * piece + 5]));
        v.w = pack_bf16(__uint_as_float(u[8 * piece + 6]), __uint_as_float(u[8 * piece + 7]));
        reinterpret_cast<uint4*>(orow + half * 32)[piece] = v;
      }
    }
    lse[static_cast<size_t>(bh) * T + q] = lse2 * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_free<512>(tmem);
}

}  // namespace

bool attn_fwd_tc_supported(size_t T, size_t hd) { return hd == HD && T % TQ == 0; }

void attn_fwd_tc(const bf16* qkv, size_t B, size_t T, size_t H, size_t hd, bf16* o, float* lse, cudaStream_t s) {
  if (!attn_fwd_tc_supported(T, hd)) raise(1, "tcgen05 attention: head_dim 64 and seq_len % 128 == 0");
  const CUtensorMap tm = tma::make_2d_bf16(qkv, 3 * H * hd, B * T, 3 * H * hd, 64, 128);
  const size_t smem = sizeof(Smem) + 1024;
  static bool attr = false;
  if (!attr) {
    CKF_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    attr = true;
  }
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(hd));
  dim3 grid(static_cast<unsigned>(T / TQ), static_cast<unsigned>(B * H));
  attn_fwd_tc_kernel<<<grid, kThreads, smem, s>>>(tm, static_cast<int>(T), static_cast<int>(H), o, lse, scale_log2);
  CKF_LAUNCH_CHECK();
}

}  // namespace ckf::llama
