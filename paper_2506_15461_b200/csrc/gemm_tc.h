// Host API of the sm_100a bf16 tensor-core GEMM (gemm_tc.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ckf::tc {

// kSwiGLU (forward gate/up GEMM, B MN-major): output N = 2f columns [gate | up]; each
//   tile computes matching gate and up columns, stores both (bf16, C = gu) and the
//   activation a = silu(g) * u (bf16, aux [M x f], ld ldaux) from the bf16-rounded g, u.
// kSwiGLUBwd (down-projection dgrad da = dh Wd^T, N = f): da never leaves the SM; the
//   epilogue reads g, u from aux = gu [M x 2f] and stores dgu = [dg | du] (bf16, C, ldc 2f).
//   Both are element-for-element the unfused swiglu_fwd / swiglu_bwd kernels.
// kXentFwd (LM head forward, A = xn K-major, B = E_inv MN-major, N = V; CTA pairs, 256-wide
//   tiles, 8 epilogue warps): the logits never leave the SM.  Per row i with shift c_i
//   (xent.c, max'ed with the decoded xent.vmax) the epilogue forms e = exp(l - c_i) in fp32,
//   stores Q = bf16(e) into C when xent.store (the loss gradient up to a row scale, see
//   head_xent.cu), writes the fp32 partial row sum of e of each 128-column half tile to
//   xent.psum[(nb * 2 + half) * M + i], the fp32 logit of the label column to xent.ly[i], and
//   -- when a logit exceeds c_i + kXentGuard -- raises xent.flag and atomically maxes the
//   row's logit into xent.vmax (ordered-int encoding) so a gated rerun can use the true max.
// kBF16Dsum: kStoreBF16 plus the attention backward's D (dsum_* below); selected internally when
// dsum_o is set, a separate instantiation so the other bf16-store GEMMs keep their registers
enum Epi { kStoreBF16 = 0, kStoreF32 = 1, kAccF32 = 2, kSwiGLU = 3, kSwiGLUBwd = 4, kXentFwd = 5, kBF16Dsum = 6 };
constexpr float kXentGuard = 50.f;
// number of per-row partial sums kXentFwd writes for a vocabulary of V columns
inline int xent_partials(int V) { return 2 * ((V + 255) / 256); }
struct XentArgs {
  const int* labels = nullptr;  // [M] label column of each row
  const float* c = nullptr;     // [M] per-row shift
  int* vmax = nullptr;          // [M] ordered-int max of guard-violating logits (sentinel = none)
  float* psum = nullptr;        // [xent_partials(N) x M]
  float* ly = nullptr;          // [M] label logit
  int* flag = nullptr;          // set to 1 on a guard violation
  int store = 1;                // store Q (training) or not (loss only)
};

// C[M,N] (epi) alpha * op(A) op(B), bf16 operands, fp32 accumulation.
//   a_mn = false: A stored [M][lda] (K contiguous); true: A stored [K][lda] (M contiguous)
//   b_mn = false: B stored [N][ldb] (K contiguous); true: B stored [K][ldb] (N contiguous)
//   epi: kStoreBF16 (C bf16), kStoreF32 (C fp32), kAccF32 (C fp32 +=)
struct GemmDesc {
  int M = 0, N = 0, K = 0;
  const __nv_bfloat16* A = nullptr;
  int lda = 0;
  bool a_mn = false;
  const __nv_bfloat16* B = nullptr;
  int ldb = 0;
  bool b_mn = false;
  void* C = nullptr;
  int ldc = 0;
  int epi = kStoreBF16;
  float alpha = 1.0f;
  int bn = 0;      // 0 = heuristic (128 or 256)
  int splits = 0;  // split-K factor; 0 = heuristic (kAccF32 only; ordered, deterministic)
  // fused rotary embedding (kStoreBF16 only): columns [0, rope_cols) are 64-wide heads whose
  // (j, j+32) pairs are rotated by rope_tab[j * rope_T + row % rope_T] = (cos, sin) (the
  // pair-major table: a warp's 32 consecutive rows read 32 adjacent entries)
  // rope_hd = 128: heads of 128 columns, pairs (j, j+64) spanning two 64-column chunks of one
  // epilogue warp's slice (rope_cols % 256 == 0)
  const float2* rope_tab = nullptr;
  int rope_T = 0, rope_cols = 0, rope_hd = 64;
  void* aux = nullptr;  // kSwiGLU: a (written); kSwiGLUBwd: gu (read)
  int ldaux = 0;
  // kStoreF32: per-row output scale (C[i,:] = row_scale[i] * acc) instead of alpha
  const float* row_scale = nullptr;
  // kStoreBF16 only: the attention backward's D = rowsum(dO . O) per (row, head) from the bf16-rounded
  // output (C = dO of the O-projection dgrad) and dsum_o (O, [M x N], row pitch N): heads of
  // dsum_hd (64 or 128) columns; D[(b * H + h) * T + q] for row = b * T + q, H = N / dsum_hd
  const __nv_bfloat16* dsum_o = nullptr;
  float* dsum_out = nullptr;
  int dsum_T = 0, dsum_hd = 64;
  // launch gate: when non-null the kernel reads *gate after its predecessor finished and does no
  // work if it is 0 (a rerun that a device flag decides, without a host round trip)
  const int* gate = nullptr;
  XentArgs xent;
};

void gemm_bf16(const GemmDesc& g, cudaStream_t s);
long long* gemm_debug_buffer();  // non-null with CKF_GEMM_DEBUG=1
int pick_bn(int M, int N);

}  // namespace ckf::tc
