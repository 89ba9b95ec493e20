// CUDA-core GEMM for the fp64 reference-parity and fp32 parity precisions.
//
// Replaces the reference's four row-major GEMMs (kernels_serial.cpp:13-61):
//   gemm_nn     C  = A B        (ta=0, tb=0, accumulate=0)
//   gemm_nn_acc C += A B        (ta=0, tb=0, accumulate=1)
//   gemm_nt_acc C += A B^T      (ta=0, tb=1, accumulate=1)
//   gemm_tn_acc C += A^T B      (ta=1, tb=0, accumulate=1)
// Tensor cores cannot deliver fp32/fp64 parity (SURVEY §7 hard part 3), so
// these run on the FMA pipes; the bf16 throughput path is gemm_tc.cu.
// 64x64 output tile per CTA, 16-deep K slices staged through shared memory,
// 4x4 register micro-tile per thread.  Deterministic: fixed K order per output.
#include "common.cuh"
#include "kernels.h"

namespace ckf::k {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int ta, int tb, size_t M, size_t N, size_t K,
                                                        const T* __restrict__ A, size_t lda,
                                                        const T* __restrict__ B, size_t ldb, T* __restrict__ C,
                                                        size_t ldc, int accumulate) {
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  const size_t m0 = static_cast<size_t>(blockIdx.y) * BM, n0 = static_cast<size_t>(blockIdx.x) * BN;
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (size_t k0 = 0; k0 < K; k0 += BK) {
    // A slice: BM x BK elements, 4 per thread
#pragma unroll
    for (int r = 0; r < (BM * BK) / 256; ++r) {
      const int e = tid + r * 256;
      int mm, kk;
      if (ta) {  // A stored [K, M]: consecutive threads walk m
        kk = e / BM;
        mm = e % BM;
      } else {   // A stored [M, K]: consecutive threads walk k
        mm = e / BK;
        kk = e % BK;
      }
      const size_t gm = m0 + mm, gk = k0 + kk;
      T val = T(0);
      if (gm < M && gk < K) val = ta ? A[gk * lda + gm] : A[gm * lda + gk];
      As[kk][mm] = val;
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / 256; ++r) {
      const int e = tid + r * 256;
      int nn, kk;
      if (tb) {  // B stored [N, K]
        nn = e / BK;
        kk = e % BK;
      } else {   // B stored [K, N]
        kk = e / BN;
        nn = e % BN;
      }
      const size_t gn = n0 + nn, gk = k0 + kk;
      T val = T(0);
      if (gn < N && gk < K) val = tb ? B[gn * ldb + gk] : B[gk * ldb + gn];
      Bs[kk][nn] = val;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][tr + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tc + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const size_t gm = m0 + tr + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const size_t gn = n0 + tc + 16 * j;
      if (gn >= N) continue;
      T* c = C + gm * ldc + gn;
      *c = accumulate ? *c + acc[i][j] : acc[i][j];
    }
  }
}

}  // namespace

template <typename T>
void gemm_simt(bool ta, bool tb, size_t M, size_t N, size_t K, const T* A, size_t lda, const T* B, size_t ldb,
               T* C, size_t ldc, bool accumulate, cudaStream_t s) {
  if (M == 0 || N == 0) return;
  if (K == 0) {
    if (!accumulate)
      for (size_t r = 0; r < M; ++r) CKF_CUDA(cudaMemsetAsync(C + r * ldc, 0, N * sizeof(T), s));
    return;
  }
  dim3 grid(static_cast<unsigned>((N + BN - 1) / BN), static_cast<unsigned>((M + BM - 1) / BM));
  gemm_simt_kernel<T><<<grid, 256, 0, s>>>(ta ? 1 : 0, tb ? 1 : 0, M, N, K, A, lda, B, ldb, C, ldc,
                                           accumulate ? 1 : 0);
  CKF_LAUNCH_CHECK();
}

template void gemm_simt<double>(bool, bool, size_t, size_t, size_t, const double*, size_t, const double*, size_t,
                                double*, size_t, bool, cudaStream_t);
template void gemm_simt<float>(bool, bool, size_t, size_t, size_t, const float*, size_t, const float*, size_t,
                               float*, size_t, bool, cudaStream_t);

}  // namespace ckf::k
