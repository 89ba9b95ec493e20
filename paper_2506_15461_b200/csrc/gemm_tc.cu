// bf16 tensor-core GEMM for sm_100a: TMA -> shared memory (128-B swizzle)
// -> tcgen05.mma (fp32 accumulators in TMEM) -> tcgen05.ld epilogue.
//
// Replaces the reference's four row-major GEMMs (kernels_serial.cpp:13-61)
// on the bf16 throughput path.  Every operand layout the stage forward /
// backward needs is a template switch instead of a transpose:
//   A K-major  = stored [M][lda]   A MN-major = stored [K][lda] (A^T)
//   B K-major  = stored [N][ldb]   B MN-major = stored [K][ldb]
//   forward  Y  = X W      A=X K-major,   B=W[K,N] MN-major
//   dgrad    dX = dY W^T   A=dY K-major,  B=W[K,N] K-major  (as [N'][K'])
//   wgrad    dW += X^T dY  A=X MN-major,  B=dY MN-major     (epilogue += fp32)
//
// Persistent, warp-specialised (one CTA per SM):
//   warp 0      TMA producer, kStages-deep smem ring (warp-converged, elect.sync issues; one lane
//               for the weight gradients)
//   warp 1      MMA issuer (warp-converged, elect.sync issues): 128 x BN x 16 tcgen05.mma, commits
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulators)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns, fused store /
//               fp32 accumulate, so tile i's epilogue overlaps tile i+1's MMAs.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm_tc.h"
#include "sm100.cuh"

namespace ckf {

// ------------------------------------------------------------------ tensor maps (host)
namespace tma {
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CKF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) raise(6, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace

CUtensorMap make_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                         uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 2) & 15))
    raise(1, "TMA operands need 16-byte aligned base and row pitch (ld % 8 == 0 for bf16)");
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(6, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

CUtensorMap make_2d_f32(const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                        uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 4) & 15))
    raise(1, "TMA fp32 operands need 16-byte aligned base and row pitch (ld % 4 == 0)");
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(6, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

CUtensorMap make_3d_bf16(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld1, uint64_t ld2,
                         uint32_t box0, uint32_t box1) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {ld1 * 2, ld2 * 2};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld1 * 2) & 15) || ((ld2 * 2) & 15))
    raise(1, "TMA operands need 16-byte aligned base and pitches");
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(6, "cuTensorMapEncodeTiled (3d) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}
}  // namespace tma

namespace tc {
namespace {

using namespace ckf::sm100;

constexpr int BM = 128, BK = 64, UK = 16;
// Epilogue warps: 8 (two per TMEM lane quarter, each on half of the tile's columns) for the
// CTA-pair LM head + loss epilogue; 4 elsewhere -- the plain bf16 store included
// (CKF_GEMM_BF16_EW8=1 gives it 8): its 32 KiB less staging buys a sixth operand stage, which the
// MMA warp's full-stage waits needed (QKV forward 144.5 -> 140.8 us, O dgrad 52.4 -> 50.9 us at
// the 500M shapes, same-box A/B; tools/gemm_debug.py)
// kSwiGLUBwd: g/u chunks in flight per epilogue warp (each a 2 x 4 KiB buffer pair); one ahead
// frees a fifth operand stage but measured slower (296.0 -> 301.4 us at [32,768 x 4,096 x 1,024])
#ifndef CKF_SWB_AHEAD
#define CKF_SWB_AHEAD 2
#endif
#ifndef CKF_GEMM_BF16_EW8
#define CKF_GEMM_BF16_EW8 0
#endif
__host__ __device__ constexpr int epi_warps(int epi, int ncta) {
  return ((CKF_GEMM_BF16_EW8 && (epi == kStoreBF16 || epi == kBF16Dsum)) || epi == kXentFwd) && ncta == 2 ? 8 : 4;
}
__host__ __device__ constexpr int gemm_threads(int epi, int ncta) { return 128 + 32 * epi_warps(epi, ncta); }
constexpr uint32_t kAStage = BM * BK * 2;  // 16 KiB
constexpr uint32_t kStageBufBytes = 4096;  // per epilogue warp, x2: [32 rows][128 B] TMA-store staging

struct Params {
  long long* dbg;  // CKF_GEMM_DEBUG=1: per-CTA phase cycles [producer empty-wait, mma full-wait, mma tempty-wait,
                   // epilogue tfull-wait, total] (tools/gemm_debug.py)
  int M, N, K;
  float alpha;
  int nm, nn, tiles, nk;
  int splits, kb_per_split, units;
  int* flags;    // split-K: 4 counters per half-tile (co-resident: stored, reduced; otherwise one per
                 // lane quarter), self-resetting
  int coresident;  // split-K units all in flight at once (waiting reduction) or not (last-arriver)
  float* ws;     // split-K partial tiles: [units][BM][BN] fp32
  float* C;      // split-K: fp32 C (row pitch ldc) the reduced tile is added into
  int ldc;
  const float2* rope_tab;  // fused RoPE (bf16 epilogue): heads of rope_hd (64 or 128) columns below rope_cols
  int rope_T, rope_cols, rope_hd;
  int f;                   // kSwiGLU / kSwiGLUBwd: ffn width (column offset of the up half)
  const __nv_bfloat16* gu; // kSwiGLUBwd: [M x 2f] gate/up activations (row pitch 2f)
  const float* row_scale;  // kStoreF32: per-row scale instead of alpha
  const int* gate;         // no work when *gate == 0
  const __nv_bfloat16* dsum_o;  // kStoreBF16: D = rowsum(bf16(C) . O) per head (gemm_tc.h)
  float* dsum_out;
  int dsum_T, dsum_hd;
  XentArgs xent;           // kXentFwd
};

// ordered-int encoding of a float (monotonic under signed int compare) for atomicMax
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2eF = 1.4426950408889634f;
constexpr float kXentGuardExp = 5.184705528587072e21f;  // exp(kXentGuard)

template <int BN, int EPI, int NCTA>
struct Cfg {
  // kSwiGLUBwd trades operand stages for 6 epilogue buffers per warp (two g/u prefetch pairs and
  // the dg/du staging pair).
  // NCTA = 2 (CTA pair): each CTA holds BN/2 columns of B, so a stage is 32 KiB at BN = 256.
  static constexpr int kEW = epi_warps(EPI, NCTA);
  static constexpr int kEpiBufs = EPI == kSwiGLUBwd ? 2 * CKF_SWB_AHEAD + 2 : 2;
  static constexpr uint32_t kBStage = (BN / NCTA) * BK * 2;
  static constexpr uint32_t kStageBytes = kAStage + kBStage;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr uint32_t kEpiBytes = kEW * kEpiBufs * kStageBufBytes;
  // as many operand stages as fit next to the epilogue staging (<= 227 KiB per CTA), at most 6
  static constexpr int kStages = (232448 - 1024 - 256 - static_cast<int>(kEpiBytes)) / static_cast<int>(kStageBytes) > 6
                                     ? 6
                                     : (232448 - 1024 - 256 - static_cast<int>(kEpiBytes)) / static_cast<int>(kStageBytes);
  static constexpr size_t kSmem = 1024 /*align slack*/ + kStages * kStageBytes + kEpiBytes + 256 /*barriers*/;
};

// Persistent work unit -> (tile, split, k-block range).  Units are split-major so
// split s of a tile always has a larger index than split s-1 (deadlock-free ordering).
struct Unit {
  int mb, nb, tile, split, kb0, kb1;
};
// Tiles are rastered in bands of kRasterM M-tiles: within a band the M index runs
// fastest, then N.  The ~148 tiles in flight then share a few A row-blocks and a
// few B column-blocks, so each operand tile comes from HBM once and is re-read
// from L2 (a plain M-fastest order over M = 65,536 tokens re-streams A from HBM
// once per N-tile).
constexpr int kRasterM = 16;
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
  Unit w;
  w.split = u / p.tiles;
  w.tile = u % p.tiles;
  const int band = w.tile / (kRasterM * p.nn);
  const int in_band = w.tile - band * kRasterM * p.nn;
  const int rows = min(kRasterM, p.nm - band * kRasterM);
  w.mb = band * kRasterM + in_band % rows;
  w.nb = in_band / rows;
  w.kb0 = w.split * p.kb_per_split;
  w.kb1 = min(p.nk, w.kb0 + p.kb_per_split);
  return w;
}

// NCTA = 2: CTA-pair (cluster of 2) tiles of 256 x BN: each CTA stages 128 rows of A and
// BN/2 columns of B, the leader issues tcgen05.mma.cta_group::2 (M = 256), both CTAs hold
// their 128 x BN accumulator rows in TMEM and run their own epilogue.
template <int BN, bool A_MN, bool B_MN, int EPI, int NCTA>
__global__ void __launch_bounds__(gemm_threads(EPI, NCTA), 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_ws, Params p) {
  using C = Cfg<BN, EPI, NCTA>;
  constexpr int ST = C::kStages;
  constexpr uint32_t IDESC = idesc_bf16_f32(BM * NCTA, BN, A_MN, B_MN);
  constexpr int BNC = BN / NCTA;  // B columns staged by this CTA
  const uint32_t rank = NCTA == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int u0 = static_cast<int>(blockIdx.x) / NCTA, ustep = static_cast<int>(gridDim.x) / NCTA;
  const long long t_start_ = p.dbg ? clock64() : 0;
  long long dw[4] = {0, 0, 0, 0};
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * kAStage;
  uint8_t* sEpi = smem + ST * C::kStageBytes;  // 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + C::kEpiBytes);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint64_t* lbar = tempty + 2;  // kSwiGLUBwd: per epilogue warp, one load barrier per g/u buffer pair
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lbar + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmap_a);
    tma_prefetch(&tmap_b);
    tma_prefetch(&tmap_c);
    if (p.splits > 1 || EPI == kSwiGLU || EPI == kSwiGLUBwd) tma_prefetch(&tmap_ws);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], C::kEW * NCTA);  // the leader's counts both CTAs' epilogue warps
    }
    for (int i = 0; i < 8; ++i) mbar_init(&lbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (NCTA == 2)
      tmem_alloc_2sm<C::kTmemCols>(tmem_slot);
    else
      tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (NCTA == 2)
    cluster_sync_all();  // barriers of both CTAs initialised before any cross-CTA signal
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the set-up above overlaps the previous kernel's tail;
  // nothing global is read or written before the previous grid has fully completed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // gated launch (a rerun decided on the device): every role sees zero units
  const int units = (p.gate && *reinterpret_cast<const volatile int*>(p.gate) == 0) ? 0 : p.units;

  if (warp == 0) {
    // the whole warp runs the producer loop (elect.sync issues) except for the weight gradients
    // (A MN-major), whose split-K epilogue shares the SM sub-partition with this warp: there one
    // lane runs it (measured: wgrad families 5-20 % slower with a converged producer, the others
    // 1-2 % faster)
#ifndef CKF_GEMM_WARP_PRODUCER
#define CKF_GEMM_WARP_PRODUCER 1
#endif
    constexpr bool kWP = CKF_GEMM_WARP_PRODUCER == 2 || (CKF_GEMM_WARP_PRODUCER == 1 && !A_MN);
    if (kWP || lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u0; u < units; u += ustep) {
        const Unit w = unit_of(p, u);
        const int arow = w.mb * BM * NCTA + static_cast<int>(rank) * BM;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          const long long w0_ = p.dbg ? clock64() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (p.dbg) dw[0] += clock64() - w0_;
          uint8_t* a = sA + stage * kAStage;
          uint8_t* b = sB + stage * C::kBStage;
          // NCTA = 2: the leader's full barrier counts both CTAs' bytes; both CTAs' loads complete on it
          const uint32_t fb = NCTA == 2 ? mapa_shared(&full[stage], 0) : smem_u32(&full[stage]);
          if (leader) {
            if constexpr (kWP)
              mbar_arrive_expect_tx_w(&full[stage], NCTA * C::kStageBytes);
            else
              mbar_arrive_expect_tx(&full[stage], NCTA * C::kStageBytes);
          }
          auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1) {
            if constexpr (NCTA == 2 && kWP)
              tma_load_2d_pair_w(dst, map, fb, c0, c1);
            else if constexpr (NCTA == 2)
              tma_load_2d_pair(dst, map, fb, c0, c1);
            else if constexpr (kWP)
              tma_load_2d_w(dst, map, &full[stage], c0, c1);
            else
              tma_load_2d(dst, map, &full[stage], c0, c1);
          };
          if constexpr (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) load(a + c * 8192, &tmap_a, arow + c * 64, kb * BK);
          } else {
            load(a, &tmap_a, kb * BK, arow);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int c = 0; c < BNC / 64; ++c) {
              const int cc = static_cast<int>(rank) * BNC + c * 64;  // column within the BN-wide tile
              int col = w.nb * BN + cc;
              if constexpr (EPI == kSwiGLU)  // accumulator columns [0, BN/2) = gate, [BN/2, BN) = up
                col = cc < BN / 2 ? w.nb * (BN / 2) + cc : p.f + w.nb * (BN / 2) + cc - BN / 2;
              load(b + c * 8192, &tmap_b, col, kb * BK);
            }
          } else {
            load(b, &tmap_b, kb * BK, w.nb * BN + static_cast<int>(rank) * BNC);
          }
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (the pair's leader issues for both CTAs): the whole warp runs
      // the loop (descriptors in uniform registers), elect.sync picks the issuing lane
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = u0; u < units; u += ustep) {
        const Unit w = unit_of(p, u);
        const long long w1_ = p.dbg ? clock64() : 0;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        if (p.dbg) dw[2] += clock64() - w1_;
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          const long long w2_ = p.dbg ? clock64() : 0;
          mbar_wait(&full[stage], phase);
          if (p.dbg) dw[1] += clock64() - w2_;
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kAStage);
          const uint32_t b0 = smem_u32(sB + stage * C::kBStage);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a0 + k * 2048, 8192, 1024) : umma_desc_sw128(a0 + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b0 + k * 2048, 8192, 1024) : umma_desc_sw128(b0 + k * 32, 16, 1024);
            if constexpr (NCTA == 2)
              umma_bf16_2sm_w(d, ad, bd, IDESC, (kb > w.kb0 || k > 0) ? 1u : 0u);
            else
              umma_bf16_w(d, ad, bd, IDESC, (kb > w.kb0 || k > 0) ? 1u : 0u);
          }
          if constexpr (NCTA == 2)
            umma_commit_2sm_w(&empty[stage], 0x3);
          else
            umma_commit_w(&empty[stage]);
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (NCTA == 2)
          umma_commit_2sm_w(&tfull[acc], 0x3);
        else
          umma_commit_w(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> swizzled smem -> TMA store / reduce-add
    constexpr int EH = C::kEW / 4;  // column slices per lane quarter
    const int ew = warp - 4;
    const int q = ew & 3;   // TMEM lane quarter (warp % 4)
    const int eh = ew >> 2;  // column slice of this warp
    uint8_t* stg = sEpi + ew * C::kEpiBufs * kStageBufBytes;
    int acc = 0, sbuf = 0;
    uint32_t acc_phase = 0;
    constexpr int CW = EPI == kStoreF32 || EPI == kAccF32 ? 32 : 64;  // columns per 128-byte staged row
    // one [32 rows x 64 bf16] chunk (packed pairs) -> swizzled staging -> TMA store
    auto store_bf16_chunk = [&](const uint32_t* pk, const CUtensorMap* map, int x, int y) {
      uint8_t* sb = stg + sbuf * kStageBufBytes;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      const uint32_t row = smem_u32(sb) + lane * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j) st_shared_v4(row + ((j ^ (lane & 7)) << 4), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (y < p.M) tma_store_2d(map, sb, x, y);
        bulk_commit();
      }
      sbuf ^= 1;
    };
    // the accumulator buffer goes back to the MMA issuer (the leader's barrier in a CTA pair)
    auto release_acc = [&](int a) {
      if constexpr (NCTA == 2)
        mbar_arrive_cluster(mapa_shared(&tempty[a], 0));
      else
        mbar_arrive(&tempty[a]);
    };
    // first output row of this warp's 32 accumulator lanes
    auto row0_of = [&](const Unit& wu) { return wu.mb * BM * NCTA + static_cast<int>(rank) * BM + q * 32; };
    int cc = 0;               // kSwiGLUBwd: chunk counter of this warp's stream
    // kSwiGLUBwd (lane 0): chunk k of this warp's stream = (unit uu, 64-column chunk c) -> pair k & 1
    constexpr int kSWA = CKF_SWB_AHEAD;
    auto swb_prefetch = [&](int k, int uu, int c) {
      const Unit w2 = unit_of(p, uu);
      uint8_t* gb = stg + (k % kSWA) * 2 * kStageBufBytes;
      uint64_t* bar = &lbar[q * 2 + (k % kSWA)];
      const int n0 = w2.nb * BN + c * 64, y = row0_of(w2);
      mbar_arrive_expect_tx(bar, 2 * kStageBufBytes);
      tma_load_2d(gb, &tmap_ws, bar, n0, y);
      tma_load_2d(gb + kStageBufBytes, &tmap_ws, bar, p.f + n0, y);
    };
    bool first_unit = true;
    for (int u = u0; u < units; u += ustep) {
      const Unit w = unit_of(p, u);
      if constexpr (EPI == kSwiGLUBwd) {
        if (first_unit && lane == 0) {  // the first g/u chunks in flight before the accumulator is ready
          for (int k = 0; k < kSWA; ++k) swb_prefetch(k, u, k);
        }
        first_unit = false;
      }
      const long long w3_ = p.dbg ? clock64() : 0;
      mbar_wait(&tfull[acc], acc_phase);
      if (p.dbg) dw[3] += clock64() - w3_;
      tc_fence_after();
      const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
      const int m0 = row0_of(w);
      if constexpr (EPI == kXentFwd) {
        // LM head + cross-entropy (gemm_tc.h): this thread's row is m0 + lane; e = 2^(l log2e - c log2e)
        const int mrow = m0 + lane;
        const bool rok = mrow < p.M;
        const int lab = rok ? __ldg(p.xent.labels + mrow) : -1;
        const float cr = rok ? fmaxf(__ldg(p.xent.c + mrow), ord2f(p.xent.vmax[mrow])) : 0.f;
        const f32x2 lg2 = f2(kLog2eF, kLog2eF), ncl = f2(-cr * kLog2eF, -cr * kLog2eF);
        float ps = 0.f;
#pragma unroll 1
        for (int c0 = eh * (BN / EH); c0 < (eh + 1) * (BN / EH); c0 += 64) {
          uint32_t r[64];
          tmem_ld32(trow + c0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32(trow + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_ld_wait();
          if (c0 + 64 >= (eh + 1) * (BN / EH)) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(acc);
          }
          const int n0 = w.nb * BN + c0;
          const int yo = lab - n0;
          if (static_cast<unsigned>(yo) < 64u) {  // the label column is in this chunk: its exact fp32 logit
            float v = 0.f;
#pragma unroll
            for (int j = 0; j < 64; ++j) v = j == yo ? __uint_as_float(r[j]) : v;
            p.xent.ly[mrow] = v;
          }
          const int nval = p.N - n0;  // columns of this chunk inside the vocabulary
          uint32_t pk[32];
          f32x2 s2[2] = {0ull, 0ull};
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float e0, e1;
            f2split(ffma2(f2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), lg2, ncl), e0, e1);
            e0 = ex2_approx(e0);
            e1 = ex2_approx(e1);
            if (nval < 64) {
              e0 = 2 * j < nval ? e0 : 0.f;
              e1 = 2 * j + 1 < nval ? e1 : 0.f;
            }
            s2[j & 1] = fadd2(s2[j & 1], f2(e0, e1));
            pk[j] = pack_bf16(e0, e1);
          }
          float sa, sb;
          f2split(fadd2(s2[0], s2[1]), sa, sb);
          const float sc = sa + sb;
          ps += sc;
          if (rok && !(sc <= kXentGuardExp)) {  // a logit too far above the shift (rare): flag a rerun
            float lm = -INFINITY;
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < nval) lm = fmaxf(lm, __uint_as_float(r[j]));
            atomicMax(p.xent.vmax + mrow, f2ord(lm));
            *p.xent.flag = 1;
          }
          if (p.xent.store) store_bf16_chunk(pk, &tmap_c, n0, m0);
        }
        if (rok) p.xent.psum[static_cast<size_t>(w.nb * EH + eh) * p.M + mrow] = ps;
      } else if constexpr (EPI == kSwiGLU) {
        // gate columns [c0, c0+64) and the matching up columns [BN/2 + c0, ...)
#pragma unroll 1
        for (int c0 = eh * (BN / 2 / EH); c0 < (eh + 1) * (BN / 2 / EH); c0 += 64) {
          uint32_t g[64], v[64];
          tmem_ld32(trow + c0, *reinterpret_cast<uint32_t(*)[32]>(&g[0]));
          tmem_ld32(trow + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&g[32]));
          tmem_ld32(trow + BN / 2 + c0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
          tmem_ld32(trow + BN / 2 + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
          tmem_ld_wait();
          if (c0 + 64 >= (eh + 1) * (BN / 2 / EH)) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(acc);
          }
          const int n0 = w.nb * (BN / 2) + c0;
          uint32_t pk[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) pk[j] = pack_bf16(__uint_as_float(g[2 * j]), __uint_as_float(g[2 * j + 1]));
          store_bf16_chunk(pk, &tmap_c, n0, m0);
#pragma unroll
          for (int j = 0; j < 32; ++j) {  // g := bf16(g) as float (what the unfused kernel reads back)
            g[2 * j] = pk[j] << 16;
            g[2 * j + 1] = pk[j] & 0xffff0000u;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) pk[j] = pack_bf16(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
          store_bf16_chunk(pk, &tmap_c, p.f + n0, m0);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float g0 = __uint_as_float(g[2 * j]), g1 = __uint_as_float(g[2 * j + 1]);
            const float u0 = __uint_as_float(pk[j] << 16), u1 = __uint_as_float(pk[j] & 0xffff0000u);
            float a0, a1;
            f2split(swiglu_fwd2(f2(g0, g1), f2(u0, u1)), a0, a1);
            pk[j] = pack_bf16(a0, a1);
          }
          store_bf16_chunk(pk, &tmap_ws, n0, m0);
        }
      } else if constexpr (EPI == kSwiGLUBwd) {
        // g/u chunks arrive by TMA TWO chunks ahead of the math into a ring of two buffer pairs
        // (chunk cc of the warp's stream uses pair cc & 1): the math reads a pair into registers and
        // it is refilled at once with chunk cc + 2; dg/du leave through a separate staging pair by
        // TMA store.  Two chunks (16 KiB) of loads in flight per warp: the epilogue moves 8 B per
        // output element.  da = dY Wd^T never leaves the SM.  Measured at the 500M shape [32,768 x 4,096
        // x 1,024]: 304 us at one chunk ahead (single CTAs) -> 293 us (pairs, two ahead); the plain
        // dgrad is 192 us; without the g/u loads 245 us, without the dg/du stores 255 us; stores
        // straight from registers (no staging) 369 us.
        constexpr int NCH = BN / 64;
        static_assert(NCH >= 2, "kSwiGLUBwd: two chunks per tile at least");
        uint8_t* ob = stg + 2 * kSWA * kStageBufBytes;  // dg / du staging pair
#pragma unroll 1
        for (int c = 0; c < NCH; ++c, ++cc) {
          const int n0 = w.nb * BN + c * 64;
          uint32_t r[64];
          tmem_ld32(trow + c * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32(trow + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_ld_wait();
          if (c + 1 == NCH) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(acc);
          }
          mbar_wait(&lbar[q * 2 + (cc % kSWA)], (cc / kSWA) & 1);
          uint8_t* gb = stg + (cc % kSWA) * 2 * kStageBufBytes;
          const uint32_t ga = smem_u32(gb) + lane * 128, ua = ga + kStageBufBytes;
          uint4 gq[8], uq[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t off = (j ^ (lane & 7)) << 4;
            gq[j] = ld_shared_v4(ga + off);
            uq[j] = ld_shared_v4(ua + off);
          }
          __syncwarp();
          if (lane == 0) {  // refill this pair with chunk cc + kSWA (generic reads ordered before the async write)
            const int c2 = c + kSWA < NCH ? c + kSWA : c + kSWA - NCH;
            const int u2 = c + kSWA < NCH ? u : u + ustep;
            if (u2 < units) {
              fence_proxy_async();
              swb_prefetch(cc + kSWA, u2, c2);
            }
          }
          uint32_t pg[32], pu[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t gw[4] = {gq[j].x, gq[j].y, gq[j].z, gq[j].w}, uw[4] = {uq[j].x, uq[j].y, uq[j].z, uq[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              // da rounded to bf16 exactly as the unfused path stores it, then swiglu_bwd's arithmetic
              const uint32_t dpk = pack_bf16(__uint_as_float(r[8 * j + 2 * e]), __uint_as_float(r[8 * j + 2 * e + 1]));
              float dg0, du0, dg1, du1;
              f32x2 dg2, du2;
              swiglu_bwd2(f2(__uint_as_float(gw[e] << 16), __uint_as_float(gw[e] & 0xffff0000u)),
                          f2(__uint_as_float(uw[e] << 16), __uint_as_float(uw[e] & 0xffff0000u)),
                          f2(__uint_as_float(dpk << 16), __uint_as_float(dpk & 0xffff0000u)), dg2, du2);
              f2split(dg2, dg0, dg1);
              f2split(du2, du0, du1);
              pg[4 * j + e] = pack_bf16(dg0, dg1);
              pu[4 * j + e] = pack_bf16(du0, du1);
            }
          }
          if (lane == 0) bulk_wait_read<0>();  // the previous chunk's stores have left the staging pair
          __syncwarp();
          const uint32_t oa = smem_u32(ob) + lane * 128, oua = oa + kStageBufBytes;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t off = (j ^ (lane & 7)) << 4;
            st_shared_v4(oa + off, pg[4 * j], pg[4 * j + 1], pg[4 * j + 2], pg[4 * j + 3]);
            st_shared_v4(oua + off, pu[4 * j], pu[4 * j + 1], pu[4 * j + 2], pu[4 * j + 3]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (m0 < p.M && n0 < p.N) {
              tma_store_2d(&tmap_c, ob, n0, m0);
              tma_store_2d(&tmap_c, ob + kStageBufBytes, p.f + n0, m0);
            }
            bulk_commit();
          }
        }
      } else if (EPI == kStoreBF16 && p.rope_tab && p.rope_hd == 128 && w.nb * BN < p.rope_cols) {
        // fused RoPE on 128-column heads: the warp's slice is whole heads; pairs (j, j+64) are the
        // two 64-column chunks of a head, rotated in fp32 and stored as two bf16 chunks
        const float2* cs = p.rope_tab + (m0 + lane) % p.rope_T;  // pair-major: coalesced per j
#pragma unroll 1
        for (int c0 = eh * (BN / EH); c0 < (eh + 1) * (BN / EH); c0 += 128) {
          uint32_t ra[64], rb[64];
          tmem_ld32(trow + c0, *reinterpret_cast<uint32_t(*)[32]>(&ra[0]));
          tmem_ld32(trow + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&ra[32]));
          tmem_ld32(trow + c0 + 64, *reinterpret_cast<uint32_t(*)[32]>(&rb[0]));
          tmem_ld32(trow + c0 + 96, *reinterpret_cast<uint32_t(*)[32]>(&rb[32]));
          tmem_ld_wait();
          if (c0 + 128 >= (eh + 1) * (BN / EH)) {  // last chunks loaded: hand the accumulator back early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(acc);
          }
          uint32_t pa[32], pb[32];
#pragma unroll
          for (int j = 0; j < 64; j += 2) {
            const float2 t0 = cs[static_cast<size_t>(j) * p.rope_T], t1 = cs[static_cast<size_t>(j + 1) * p.rope_T];
            const float x10 = __uint_as_float(ra[j]), x20 = __uint_as_float(rb[j]);
            const float x11 = __uint_as_float(ra[j + 1]), x21 = __uint_as_float(rb[j + 1]);
            pa[j / 2] = pack_bf16((x10 * t0.x - x20 * t0.y) * p.alpha, (x11 * t1.x - x21 * t1.y) * p.alpha);
            pb[j / 2] = pack_bf16((x20 * t0.x + x10 * t0.y) * p.alpha, (x21 * t1.x + x11 * t1.y) * p.alpha);
          }
          const int n0 = w.nb * BN + c0;
          store_bf16_chunk(pa, &tmap_c, n0, m0);
          store_bf16_chunk(pb, &tmap_c, n0 + 64, m0);
        }
      } else {
      float rsc = p.alpha;  // kStoreF32 with a per-row scale: this lane's row
      if (EPI == kStoreF32 && p.row_scale) rsc = m0 + lane < p.M ? __ldg(p.row_scale + m0 + lane) : 0.f;
      float dacc = 0.f;  // D epilogue: the running dot of the current head
#pragma unroll 1
      for (int c0 = eh * (BN / EH); c0 < (eh + 1) * (BN / EH); c0 += CW) {
        uint32_t r[CW];
        if constexpr (CW == 64) {
          uint32_t (&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
          uint32_t (&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
          tmem_ld32(trow + c0, r0);
          tmem_ld32(trow + c0 + 32, r1);
        } else {
          uint32_t (&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
          tmem_ld32(trow + c0, r0);
        }
        tmem_ld_wait();
        if constexpr (EPI == kStoreBF16) {
          // fused RoPE: this 64-column chunk is one head of q or k; rotate (j, j+32) in fp32
          if (p.rope_tab && w.nb * BN + c0 < p.rope_cols) {
            const float2* cs = p.rope_tab + (m0 + lane) % p.rope_T;  // pair-major: coalesced per j
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float2 t = cs[static_cast<size_t>(j) * p.rope_T];
              const float x1 = __uint_as_float(r[j]), x2 = __uint_as_float(r[j + 32]);
              r[j] = __float_as_uint(x1 * t.x - x2 * t.y);
              r[j + 32] = __float_as_uint(x2 * t.x + x1 * t.y);
            }
          }
        }
        if (c0 + CW >= (eh + 1) * (BN / EH)) {  // last chunk loaded: hand the accumulator back early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(acc);
        }
        uint8_t* sb = stg + sbuf * kStageBufBytes;
        if (lane == 0) bulk_wait_read<1>();  // the staging buffer used two stores ago is free
        __syncwarp();
        const uint32_t row = smem_u32(sb) + lane * 128;
        // D epilogue: this row's O for the chunk's 64 columns (8 x 16 B in flight; loading them one
        // chunk ahead measured slower: the extra live registers spill)
        const bool dsum = EPI == kBF16Dsum && m0 + lane < p.M;
        uint4 ov[EPI == kBF16Dsum ? 8 : 1];
        if (EPI == kBF16Dsum && dsum) {
          const uint4* op = reinterpret_cast<const uint4*>(p.dsum_o + static_cast<size_t>(m0 + lane) * p.N + w.nb * BN + c0);
#pragma unroll
          for (int j = 0; j < (EPI == kBF16Dsum ? 8 : 1); ++j) ov[j] = __ldg(op + j);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t a, b, c, d;
          if constexpr (EPI == kStoreBF16 || EPI == kBF16Dsum) {
            a = pack_bf16(__uint_as_float(r[8 * j + 0]) * p.alpha, __uint_as_float(r[8 * j + 1]) * p.alpha);
            b = pack_bf16(__uint_as_float(r[8 * j + 2]) * p.alpha, __uint_as_float(r[8 * j + 3]) * p.alpha);
            c = pack_bf16(__uint_as_float(r[8 * j + 4]) * p.alpha, __uint_as_float(r[8 * j + 5]) * p.alpha);
            d = pack_bf16(__uint_as_float(r[8 * j + 6]) * p.alpha, __uint_as_float(r[8 * j + 7]) * p.alpha);
            if (EPI == kBF16Dsum && dsum) {  // bf16(dO) . O in fp32, the dsum kernel's operands
              const uint4 o4 = ov[EPI == kBF16Dsum ? j : 0];
              const uint32_t dq[4] = {a, b, c, d}, oq[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                dacc = fmaf(__uint_as_float(dq[e] << 16), __uint_as_float(oq[e] << 16), dacc);
                dacc = fmaf(__uint_as_float(dq[e] & 0xffff0000u), __uint_as_float(oq[e] & 0xffff0000u), dacc);
              }
            }
          } else {
            a = __float_as_uint(__uint_as_float(r[4 * j + 0]) * rsc);
            b = __float_as_uint(__uint_as_float(r[4 * j + 1]) * rsc);
            c = __float_as_uint(__uint_as_float(r[4 * j + 2]) * rsc);
            d = __float_as_uint(__uint_as_float(r[4 * j + 3]) * rsc);
          }
          st_shared_v4(row + ((j ^ (lane & 7)) << 4), a, b, c, d);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const int n0 = w.nb * BN + c0;
          if (p.splits > 1) {
            // split-K: this split's partial tile goes to its workspace slot (plain store)
            // (CTA pair: each CTA's 128-row half-tile is its own slot)
            tma_store_2d(&tmap_ws, sb, c0, ((w.split * p.tiles + w.tile) * NCTA + static_cast<int>(rank)) * BM + q * 32);
          } else if (n0 < p.N && m0 < p.M) {
            if constexpr (EPI == kAccF32)
              tma_reduce_add_2d(&tmap_c, sb, n0, m0);
            else
              tma_store_2d(&tmap_c, sb, n0, m0);
          }
          bulk_commit();
        }
        sbuf ^= 1;
        if (EPI == kBF16Dsum && ((w.nb * BN + c0 + CW) % p.dsum_hd) == 0) {  // head complete
          const int mrow = m0 + lane;
          if (mrow < p.M) {
            const int hh = (w.nb * BN + c0 + CW) / p.dsum_hd - 1, H = p.N / p.dsum_hd;
            const int b = mrow / p.dsum_T, q = mrow - b * p.dsum_T;
            p.dsum_out[(static_cast<size_t>(b) * H + hh) * p.dsum_T + q] = dacc;
          }
          dacc = 0.f;
        }
      }
      }  // generic epilogues
      if (EPI == kAccF32 && p.splits > 1) {  // (split-K runs only with the accumulate epilogue)
        const int ht = w.tile * NCTA + static_cast<int>(rank);  // half-tile of a CTA pair
        // sums partial rows [r_lo, r_hi) of this half-tile over the splits, in split order, into C:
        // float4 slots, lanes along the columns (coalesced); kP slots per lane in flight at once --
        // C first, then each split's partials -- so the reduction is bandwidth- rather than
        // latency-bound.  Sum order per element as always: ((p0 + p1) + p2 ...) + C, deterministic.
        auto reduce_rows = [&](int r_lo, int r_hi) {
          constexpr int kP = 8, kQ = BN / 4;
          const int nslot = (r_hi > r_lo ? r_hi - r_lo : 0) * kQ;
          const size_t ws_base = (static_cast<size_t>(w.tile) * NCTA + rank) * BM;
          const size_t ws_split = static_cast<size_t>(p.tiles) * NCTA * BM * BN;  // floats between splits
          for (int base = lane; base < nslot; base += 32 * kP) {
            float4 o[kP], acc4[kP];
            float4* dst[kP];
            size_t wofs[kP];
            bool ok[kP];
#pragma unroll
            for (int i = 0; i < kP; ++i) {
              const int idx = base + 32 * i;
              const int rr = r_lo + idx / kQ, c = (idx % kQ) * 4;
              const int m = w.mb * BM * NCTA + static_cast<int>(rank) * BM + rr;
              const int n = w.nb * BN + c;
              ok[i] = idx < nslot && m < p.M && n < p.N;
              dst[i] = reinterpret_cast<float4*>(p.C + static_cast<size_t>(ok[i] ? m : 0) * p.ldc + (ok[i] ? n : 0));
              wofs[i] = (ws_base + rr) * BN + c;
              if (ok[i]) o[i] = *dst[i];
            }
#pragma unroll 1
            for (int sp = 0; sp < p.splits; ++sp) {
              float4 t[kP];
#pragma unroll
              for (int i = 0; i < kP; ++i)
                if (ok[i]) t[i] = __ldcg(reinterpret_cast<const float4*>(p.ws + sp * ws_split + wofs[i]));
#pragma unroll
              for (int i = 0; i < kP; ++i)
                if (ok[i]) {
                  if (sp == 0) {
                    acc4[i] = t[i];
                  } else {
                    acc4[i].x += t[i].x;
                    acc4[i].y += t[i].y;
                    acc4[i].z += t[i].z;
                    acc4[i].w += t[i].w;
                  }
                }
            }
#pragma unroll
            for (int i = 0; i < kP; ++i)
              if (ok[i]) {
                o[i].x += acc4[i].x;
                o[i].y += acc4[i].y;
                o[i].z += acc4[i].z;
                o[i].w += acc4[i].w;
                *dst[i] = o[i];
              }
          }
        };
        if (p.coresident) {
          // All units co-resident (units <= CTAs in flight): 1) every warp publishes its stored
          // partial rows, 2) once all 4*splits warps of the tile have, the tile's rows are shared
          // out among them and each reduces its share.
          int* stored = p.flags + 4 * ht;
          int* reduced = stored + 1;
          const int nwarps = C::kEW * p.splits;
          if (lane == 0) {
            bulk_wait_all();  // this warp's partial rows have landed in the workspace
            fence_proxy_async_global();
            __threadfence();
            atomicAdd(stored, 1);
            while (ld_acquire(stored) < nwarps) __nanosleep(32);
          }
          __syncwarp();
          const int wid = w.split * C::kEW + ew;
          const int per = (BM + nwarps - 1) / nwarps;
          reduce_rows(wid * per, min(BM, (wid + 1) * per));
          __syncwarp();
          if (lane == 0) {
            __threadfence();
            if (atomicAdd(reduced, 1) == nwarps - 1) {  // last one out resets the tile's counters
              atomicExch(stored, 0);
              atomicExch(reduced, 0);
            }
          }
          __syncwarp();
        } else {
          // More units than CTAs in flight (split counts chosen for wave balance): no waiting --
          // the LAST of the tile's `splits` warps of this lane quarter (the arrival that completes
          // the count) reduces the quarter's 32 rows; the others move on.  Same sums, same order.
          int* cnt = p.flags + 4 * ht + q;
          int last = 0;
          if (lane == 0) {
            bulk_wait_all();
            fence_proxy_async_global();
            __threadfence();
            last = atomicAdd(cnt, 1) == p.splits - 1 ? 1 : 0;
            __threadfence();
          }
          last = __shfl_sync(0xffffffffu, last, 0);
          if (last) {
            reduce_rows(q * 32, q * 32 + 32);
            __syncwarp();
            if (lane == 0) atomicExch(cnt, 0);
          }
          __syncwarp();
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  if (p.dbg && lane == 0) {
    long long* d = p.dbg + 8 * blockIdx.x;
    if (warp == 0) d[0] = dw[0];
    if (warp == 1) {
      d[1] = dw[1];
      d[2] = dw[2];
    }
    if (warp == 4) {
      d[3] = dw[3];
      d[4] = clock64() - t_start_;
    }
  }
  tc_fence_before();
  if constexpr (NCTA == 2) {
    cluster_sync_all();  // the leader's MMAs into the peer's TMEM are complete
    tc_fence_after();
    if (warp == 2) tmem_free_2sm<C::kTmemCols>(tmem_base);
  } else {
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_free<C::kTmemCols>(tmem_base);
  }
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : kNumSMs;
  }();
  return n;
}

}  // namespace
long long* gemm_debug_buffer() {
  static long long* b = [] {
    long long* x = nullptr;
    if (std::getenv("CKF_GEMM_DEBUG")) {
      CKF_CUDA(cudaMalloc(&x, 8 * sizeof(long long) * 1024));
      CKF_CUDA(cudaMemset(x, 0, 8 * sizeof(long long) * 1024));
    }
    return x;
  }();
  return b;
}
namespace {

float* split_workspace(size_t bytes) {
  static float* ws = nullptr;
  static size_t cap = 0;
  if (bytes > cap) {
    if (ws) CKF_CUDA(cudaFree(ws));
    cap = std::max<size_t>(bytes, 32u << 20);
    CKF_CUDA(cudaMalloc(&ws, cap));
    ++alloc_epoch();
  }
  return ws;
}

int* split_flags(size_t n) {
  // two self-resetting counters per output tile (zero between launches)
  static int* flags = nullptr;
  static size_t cap = 0;
  static int dev = -1;
  int cur = 0;
  CKF_CUDA(cudaGetDevice(&cur));
  if (n > cap || cur != dev) {
    if (flags && cur == dev) CKF_CUDA(cudaFree(flags));
    cap = std::max<size_t>(n, 4096);
    CKF_CUDA(cudaMalloc(&flags, cap * sizeof(int)));
    ++alloc_epoch();
    CKF_CUDA(cudaMemset(flags, 0, cap * sizeof(int)));
    dev = cur;
  }
  return flags;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int NCTA>
void launch_t(const GemmDesc& g, int splits, cudaStream_t s) {
  using C = Cfg<BN, EPI, NCTA>;
  const CUtensorMap ta = A_MN ? tma::make_2d_bf16(g.A, g.M, g.K, g.lda, 64, 64)
                              : tma::make_2d_bf16(g.A, g.K, g.M, g.lda, 64, BM);
  const CUtensorMap tb = B_MN ? tma::make_2d_bf16(g.B, g.N, g.K, g.ldb, 64, 64)
                              : tma::make_2d_bf16(g.B, g.K, g.N, g.ldb, 64, BN / NCTA);
  const bool c_bf16 = EPI == kStoreBF16 || EPI == kBF16Dsum || EPI == kSwiGLU || EPI == kSwiGLUBwd || EPI == kXentFwd;
  // kSwiGLUBwd: C = dgu [M x 2f] although the GEMM's N is f
  const CUtensorMap tcm = c_bf16 ? tma::make_2d_bf16(g.C, EPI == kSwiGLUBwd ? 2 * g.N : g.N, g.M, g.ldc, 64, 32)
                                 : tma::make_2d_f32(g.C, g.N, g.M, g.ldc, 32, 32);
  Params p;
  p.dbg = gemm_debug_buffer();
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.alpha = g.alpha;
  p.nm = (g.M + BM * NCTA - 1) / (BM * NCTA);  // (pair) tiles along M
  p.nn = (g.N + BN - 1) / BN;
  p.tiles = p.nm * p.nn;
  p.nk = (g.K + BK - 1) / BK;
  p.splits = std::max(1, std::min(splits, p.nk));
  p.kb_per_split = (p.nk + p.splits - 1) / p.splits;
  p.splits = (p.nk + p.kb_per_split - 1) / p.kb_per_split;  // no empty split
  p.units = p.tiles * p.splits;
  if (p.splits > 1 && (EPI != kAccF32 || g.N % 4 != 0)) p.splits = 1, p.units = p.tiles, p.kb_per_split = p.nk;
  // co-resident: every unit in flight at once (units <= CTAs or CTA pairs) -> the waiting,
  // shared reduction; otherwise the last-arriver reduction per lane quarter
  p.coresident = p.units <= num_sms() / NCTA ? 1 : 0;
  p.flags = p.splits > 1 ? split_flags(4 * static_cast<size_t>(p.tiles) * NCTA) : nullptr;
  p.ws = p.splits > 1 ? split_workspace(static_cast<size_t>(p.units) * NCTA * BM * BN * sizeof(float)) : nullptr;
  p.C = static_cast<float*>(g.C);
  p.ldc = g.ldc;
  p.rope_tab = g.rope_tab;
  p.rope_T = g.rope_T;
  p.rope_cols = g.rope_cols;
  p.rope_hd = g.rope_hd;
  p.f = EPI == kSwiGLU ? g.N / 2 : g.N;
  p.gu = EPI == kSwiGLUBwd ? static_cast<const __nv_bfloat16*>(g.aux) : nullptr;
  p.row_scale = g.row_scale;
  p.gate = g.gate;
  p.xent = g.xent;
  p.dsum_o = g.dsum_o;
  p.dsum_out = g.dsum_out;
  p.dsum_T = g.dsum_T;
  p.dsum_hd = g.dsum_hd;
  if (EPI == kBF16Dsum && (!g.dsum_o || !g.dsum_out || g.dsum_T <= 0 || (g.dsum_hd != 64 && g.dsum_hd != 128) ||
                   g.N % g.dsum_hd != 0 || g.M % g.dsum_T != 0 || g.rope_tab || (BN * 4 / C::kEW) % g.dsum_hd != 0))
    raise(1, "gemm_bf16: the D epilogue needs the bf16 store, 64/128-column heads aligned to the epilogue slices, no RoPE");
  if (EPI == kXentFwd && (!g.xent.labels || !g.xent.c || !g.xent.vmax || !g.xent.psum || !g.xent.ly || !g.xent.flag))
    raise(1, "gemm_bf16: the cross-entropy epilogue needs labels, c, vmax, psum, ly and flag");
  if (g.row_scale && EPI != kStoreF32) raise(1, "gemm_bf16: row_scale needs the fp32 store epilogue");
  if constexpr (EPI == kSwiGLU || EPI == kSwiGLUBwd) {
    if (!g.aux) raise(1, "gemm_bf16: the SwiGLU epilogues need aux");
    if (EPI == kSwiGLU && (g.N % BN != 0 || (g.N / 2) % (BN / 2) != 0))
      raise(1, "gemm_bf16: fused SwiGLU needs 2f % BN == 0");
    if (EPI == kSwiGLUBwd && (g.N % 64 != 0 || g.ldc != 2 * g.N || (reinterpret_cast<uintptr_t>(g.aux) & 15)))
      raise(1, "gemm_bf16: fused SwiGLU backward needs f % 64 == 0, ldc == 2f, 16-byte aligned gu");
  }
  if (g.rope_tab && (EPI != kStoreBF16 || g.rope_T <= 0 || g.rope_cols % 64 || (g.rope_hd != 64 && g.rope_hd != 128)))
    raise(1, "gemm_bf16: fused RoPE needs the bf16 epilogue and 64- or 128-column heads");
  if (g.rope_tab && g.rope_hd == 128 && (g.rope_cols % BN != 0 || (BN / C::kEW * 4) % 128 != 0))
    raise(1, "gemm_bf16: 128-column RoPE heads need rope_cols % BN == 0 and 128-column epilogue slices");
  const CUtensorMap twm = p.splits > 1    ? tma::make_2d_f32(p.ws, BN, static_cast<uint64_t>(p.units) * NCTA * BM, BN, 32, 32)
                          : EPI == kSwiGLU    ? tma::make_2d_bf16(g.aux, g.N / 2, g.M, g.ldaux, 64, 32)
                          : EPI == kSwiGLUBwd ? tma::make_2d_bf16(g.aux, 2 * g.N, g.M, g.ldaux, 64, 32)
                                              : tcm;
  auto kern = gemm_kernel<BN, A_MN, B_MN, EPI, NCTA>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    CKF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::kSmem)));
    attr_set = true;
  }
  const int grid = NCTA * std::min(p.units, num_sms() / NCTA);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(gemm_threads(EPI, NCTA));
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // NCTA = 2: the CTA pair shares one TPC
  attr[0].val.clusterDim.x = NCTA;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = [] {  // CKF_PDL=0: plain stream-ordered launches (A/B timing)
    const char* v = std::getenv("CKF_PDL");
    return !(v && v[0] == '0');
  }();
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  CKF_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, twm, p));
  CKF_LAUNCH_CHECK();
}

template <int BN, int NCTA>
void dispatch_bn(const GemmDesc& g, int splits, cudaStream_t s) {
#define CKF_GEMM_CASE(AM, BMN, E) \
  if (g.a_mn == AM && g.b_mn == BMN && g.epi == E) return launch_t<BN, AM, BMN, E, NCTA>(g, splits, s);
#define CKF_GEMM_EPIS(AM, BMN) CKF_GEMM_CASE(AM, BMN, kStoreBF16) CKF_GEMM_CASE(AM, BMN, kStoreF32) CKF_GEMM_CASE(AM, BMN, kAccF32)
  CKF_GEMM_EPIS(false, false)
  CKF_GEMM_EPIS(false, true)
  CKF_GEMM_EPIS(true, false)
  CKF_GEMM_EPIS(true, true)
  CKF_GEMM_CASE(false, true, kSwiGLU)
  CKF_GEMM_CASE(false, false, kSwiGLUBwd)
  CKF_GEMM_CASE(false, false, kBF16Dsum)
  if constexpr (BN == 256 && NCTA == 2) {  // the partial-sum layout assumes 256-wide pair tiles, 8 warps
    CKF_GEMM_CASE(false, true, kXentFwd)
  }
#undef CKF_GEMM_EPIS
#undef CKF_GEMM_CASE
  raise(1, "gemm_bf16: unsupported epilogue");
}

}  // namespace

int pick_bn(int M, int N) {
  const int sms = num_sms();
  auto cost = [&](int bn) {
    const long tiles = static_cast<long>((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    const long waves = (tiles + sms - 1) / sms;
    return waves * (bn + 48);  // per-tile time ~ BN columns of MMA + fixed prologue/epilogue
  };
  return cost(128) < cost(256) ? 128 : 256;
}

void gemm_bf16(const GemmDesc& g0, cudaStream_t s) {
  if (g0.M <= 0 || g0.N <= 0 || g0.K <= 0) return;
  GemmDesc g = g0;
  if (g.dsum_o) {  // the D epilogue is its own instantiation (bf16 store + D)
    if (g.epi != kStoreBF16) raise(1, "gemm_bf16: dsum_o needs the bf16 store epilogue");
    g.epi = kBF16Dsum;
  }
  if (g.ldc % 4 != 0 && (g.epi == kStoreF32 || g.epi == kAccF32)) raise(1, "gemm_bf16: fp32 C needs ldc % 4 == 0");
  if (reinterpret_cast<uintptr_t>(g.C) % 16) raise(1, "gemm_bf16: C must be 16-byte aligned");
  if (g.ldc % 8 != 0 && (g.epi == kStoreBF16 || g.epi == kBF16Dsum || g.epi == kSwiGLU || g.epi == kSwiGLUBwd))
    raise(1, "gemm_bf16: bf16 C needs ldc % 8 == 0");
  if (g.epi == kXentFwd) {
    if (g.a_mn || !g.b_mn || g.splits > 1) raise(1, "gemm_bf16: the cross-entropy epilogue needs A K-major, B MN-major");
    return dispatch_bn<256, 2>(g, 1, s);
  }
  int bn = g.bn ? g.bn : pick_bn(g.M, g.N);
  // Split-K (deterministic workspace reduction) only for the fp32-accumulate (weight-gradient)
  // epilogue, and only when no tile width fills the GPU: measured on B200
  // (profiles/r01_gemm_splitk_sweep.jsonl), a >= ~100-tile grid beats any split.
  int splits = g.splits;
  static const int env_splits = [] {  // tuning override (tools/gemm_splits.py), 0 = heuristic
    const char* v = std::getenv("CKF_GEMM_SPLITS");
    return v ? std::atoi(v) : 0;
  }();
  if (splits <= 0 && env_splits > 0) splits = env_splits;
  static const bool pair_ok = [] {  // CKF_GEMM_PAIR=0: single-CTA tiles only
    const char* v = std::getenv("CKF_GEMM_PAIR");
    return !(v && v[0] == '0');
  }();
  // weight gradients (fp32 accumulate, M = fan_in small, K = tokens long): CTA-pair 256 x 256
  // tiles split along K until the 74 pairs are busy (4x the MMA work per staged byte of the
  // single-CTA 128 x 128 split tiles)
  const bool pair_wgrad = pair_ok && !g.bn && g.epi == kAccF32 && g.M >= 2 * BM && g.M <= 4096;
  static const int wg_bn = [] {  // CKF_GEMM_WG_BN=128: 256 x 128 pair tiles for the weight gradients
    const char* v = std::getenv("CKF_GEMM_WG_BN");
    return v && std::atoi(v) == 128 ? 128 : 256;
  }();
  if (pair_wgrad) bn = wg_bn;
  if (splits <= 0 && pair_wgrad) {
    // split count by wave balance over the 74 pairs: time ~ ceil(tiles * s / pairs) / s of a tile
    // plus a per-split reduction term (e.g. QKV wgrad at d = 1024: 48 pair tiles -> s = 3, 144
    // units in two waves = 0.67 tile times instead of 1.0 with 26 pairs idle)
    const int pairs = num_sms() / 2, nk = (g.K + BK - 1) / BK;
    const int pt = ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + bn - 1) / bn);
    static const double red_cost = [] {
      const char* v = std::getenv("CKF_GEMM_SPLIT_COST");
      return v ? std::atof(v) : 0.04;
    }();
    double best = 1e30;
    splits = 1;
    // only a grid that leaves pairs idle is split: a multi-wave grid pays the reduction traffic for
    // nothing (measured: gate/up wgrad, 128 pair tiles, 4 splits 427.9 us vs 388.8 unsplit)
    for (int sk = 1; sk <= 16 && nk / sk >= 4 && pt < pairs; ++sk) {
      const double waves = static_cast<double>((pt * sk + pairs - 1) / pairs);
      const double t = waves / sk + (sk > 1 ? red_cost * sk : 0.0);
      if (t < best - 1e-9) {
        best = t;
        splits = sk;
      }
    }
  }
  if (splits <= 0) {
    splits = 1;
    if (g.epi == kAccF32) {
      const int sms = num_sms();
      const int nm = (g.M + BM - 1) / BM;
      const int t256 = nm * ((g.N + 255) / 256), t128 = nm * ((g.N + 127) / 128);
      const int nk = (g.K + BK - 1) / BK;
      if (!g.bn && t256 * 3 >= sms * 2) {
        bn = 256;
      } else if (!g.bn && t128 * 3 >= sms * 2) {
        bn = 128;
      } else {
        const int tiles = nm * ((g.N + bn - 1) / bn);
        if (tiles * 2 <= sms) splits = std::max(1, std::min({sms / tiles, nk / 4, 16}));
      }
    }
  }
  if (splits > 1 && g.epi != kAccF32) raise(1, "gemm_bf16: split-K needs the fp32 accumulate epilogue");
  // CTA pairs (256 x 256 tiles, cta_group::2) when the output is tiled without split-K: each SM
  // stages half the B bytes per MMA FLOP in a 6-deep ring.  Measured on B200
  // (profiles/r01_gemm_pair_vs_single.jsonl): +3-4 % on the stage GEMMs; single CTAs stay ahead
  // for the fused SwiGLU epilogues and for N <= 512 with very short or very long K.
  // The SwiGLU forward (gate/up GEMM, 128 x 256 single-CTA tiles are operand-bandwidth bound:
  // 96 B / clk / SM of A + B at the tensor peak) runs as CTA pairs too -- B multicast, 6 operand
  // stages: 481.7 -> 424.6 us at [32,768 x 8,192 x 1,024] (500M).  The backward epilogue
  // (g / u in, dg / du out: 8 B per element) is HBM-bound; as a CTA pair it keeps 4 operand stages
  // next to its 6 epilogue buffers per warp (two g/u chunks in flight per warp).
  // CKF_GEMM_SWIGLU_PAIR=0 / 1: single CTAs for both / for the backward only.
  static const int swiglu_pair = [] {
    const char* v = std::getenv("CKF_GEMM_SWIGLU_PAIR");
    return v ? std::atoi(v) : 2;
  }();
  const bool swiglu_single = (g.epi == kSwiGLU && swiglu_pair == 0) || (g.epi == kSwiGLUBwd && swiglu_pair != 2);
  const bool pair_shape = pair_wgrad || (!swiglu_single && splits <= 1 &&
                                         !(g.N <= 512 && (g.K <= 512 || g.K >= 16384)));
  if (bn == 128 && pair_wgrad)
    dispatch_bn<128, 2>(g, splits, s);
  else if (bn == 128)
    dispatch_bn<128, 1>(g, splits, s);
  else if (pair_ok && pair_shape && g.M >= 2 * BM)
    dispatch_bn<256, 2>(g, splits, s);
  else
    dispatch_bn<256, 1>(g, splits, s);
}

}  // namespace tc
}  // namespace ckf
