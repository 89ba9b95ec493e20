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
enum Epi { kStoreBF16 = 0, kStoreF32 = 1, kAccF32 = 2, kSwiGLU = 3, kSwiGLUBwd = 4 };

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
  const float2* rope_tab = nullptr;
  int rope_T = 0, rope_cols = 0;
  void* aux = nullptr;  // kSwiGLU: a (written); kSwiGLUBwd: gu (read)
  int ldaux = 0;
};

void gemm_bf16(const GemmDesc& g, cudaStream_t s);
long long* gemm_debug_buffer();  // non-null with CKF_GEMM_DEBUG=1
int pick_bn(int M, int N);

}  // namespace ckf::tc
