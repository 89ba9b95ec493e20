// Internal launcher API of the engine's CUDA kernels (C++; not part of the C-ABI).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ckf {

// Device scratch for deterministic two-pass reductions: pass 1 writes one
// partial per CTA (fixed grid for a given n), pass 2 folds them in index order.
struct ReduceScratch {
  double* partials = nullptr;  // >= kMaxReduceBlocks doubles
  static constexpr int kMaxReduceBlocks = 1184;  // 8 x 148
};

namespace k {

enum Act { kTanh = 0, kRelu = 1, kIdentity = 2 };

template <typename T> void uniform(T* out, size_t n, uint64_t key, double lo, double hi, uint64_t first_counter,
                                   cudaStream_t s);
template <typename T> void act_fwd(int act, const T* in, T* out, size_t n, cudaStream_t s);
template <typename T> void act_bwd(int act, const T* z, const T* dz, T* da, size_t n, cudaStream_t s);
template <typename T> void add_inplace(T* x, const T* y, size_t n, cudaStream_t s);
template <typename T> void axpy(double alpha, const T* x, T* y, size_t n, cudaStream_t s);
template <typename T> void scale(double alpha, T* x, size_t n, cudaStream_t s);
template <typename T> void fill(T* x, double v, size_t n, cudaStream_t s);
template <typename A, typename B> void convert(const A* in, B* out, size_t n, cudaStream_t s);

// sum(x^2) / sum((x-y)^2) -> *out (device double), deterministic
template <typename T> void sum_squares(const T* x, size_t n, double* out, ReduceScratch& sc, cudaStream_t s);
template <typename T> void sum_sq_diff(const T* x, const T* y, size_t n, double* out, ReduceScratch& sc,
                                       cudaStream_t s);

// mean squared error (kernels_serial.cpp:146-161); dpred optional; *loss device double
template <typename T> void mse_loss_grad(const T* pred, const T* target, size_t rows, size_t cols, T* dpred,
                                         double* loss, ReduceScratch& sc, cudaStream_t s);
// mean softmax cross-entropy over rows (kernels_serial.cpp:163-185); labels as int32
template <typename T> void xent_loss_grad(const T* logits, const int* labels, size_t rows, size_t cols,
                                          T* dlogits, double* loss, ReduceScratch& sc, cudaStream_t s);

// fused Adam + omega (see ckf_adam_device in include/ckf.h)
template <typename T> void adam(T* w, T* m, T* v, T* g, __nv_bfloat16* w_bf16, size_t n, double lr, double bc1,
                                double bc2, double grad_scale, bool zero_grad, double* omega, ReduceScratch& sc,
                                cudaStream_t s);

// out = (op*wp + on*wn)/(op+on) (recovery.cpp:57-73); optional ||out_old-out_new||^2
template <typename T> void recover(const T* wp, const T* wn, T* out, size_t n, double op, double on,
                                   double* old_sq, ReduceScratch& sc, cudaStream_t s);
// Averaged-moment policy (trainer.cpp:263-269): out = weighted_or_uniform(op, on, a, b)
template <typename T> void weighted_or_uniform(const T* a, const T* b, T* out, size_t n, double op, double on,
                                               cudaStream_t s);

// One streaming pass that makes a failed stage ready (trainer.cpp:230-276 for the
// neighbour-average family): w = (op*Wp + on*Wn)/(op+on) (recovery.cpp:57-73; op = on = 1
// for the uniform baseline), Adam moments Fresh (zero) or Averaged (omega-weighted, the
// weighted_or_uniform policy of trainer.cpp:263-269), gradient accumulator zeroed, bf16
// shadow refreshed, and optionally ||w_old - w_new||^2 (trainer.cpp:278-279) from the same
// read.  wp / wn / mp / mn / vp / vn may be PEER pointers (another GPU's HBM mapped through
// CUDA IPC / peer access): the same kernel pulls the neighbours over NVLink.
template <typename T>
struct StageRecovery {
  const T *wp = nullptr, *wn = nullptr;                        // neighbour weights
  const T *mp = nullptr, *mn = nullptr, *vp = nullptr, *vn = nullptr;  // neighbour moments (Averaged)
  T *w = nullptr, *m = nullptr, *v = nullptr, *g = nullptr;   // the failed stage
  __nv_bfloat16* wlp = nullptr;                                 // its bf16 shadow (may be null)
  size_t n = 0;
  double op = 1.0, on = 1.0;   // weight omegas (degenerate 0,0 -> uniform, recovery.cpp:63-68)
  bool averaged = false;       // moments: false = Fresh (zero), true = omega-weighted
  double mop = 0.0, mon = 0.0; // moment weights (the neighbours' omegas)
  double* old_sq = nullptr;    // optional ||w_old - w_new||^2 (device double)
};
template <typename T> void recover_stage(const StageRecovery<T>& r, ReduceScratch& sc, cudaStream_t s);

// Peer-memory stage transfers (the IPC transport of the plan-driven pipeline): the sender's
// stream copies a microbatch buffer into the receiver's mailbox (peer HBM over NVLink), then
// flag_signal stores `value` into the receiver's flag with system-scope release semantics; the
// receiver's stream runs flag_wait, which spins (acquire) until the flag reaches `value`.
void flag_signal(uint64_t* flag, uint64_t value, cudaStream_t s);
void flag_wait(const uint64_t* flag, uint64_t value, cudaStream_t s);

// NaN poison (simulated loss of a stage's GPU state)
template <typename T> void poison(T* x, size_t n, cudaStream_t s);

// generic row-major GEMM on CUDA cores (fp64 / fp32 parity paths):
//   C[M,N] = beta*C + op(A) op(B); op(A) = A[M,K] (ta=0) or A^T with A[K,M] (ta=1);
//   op(B) = B[K,N] (tb=0) or B^T with B[N,K] (tb=1).  beta in {0,1}.
template <typename T> void gemm_simt(bool ta, bool tb, size_t M, size_t N, size_t K, const T* A, size_t lda,
                                     const T* B, size_t ldb, T* C, size_t ldc, bool accumulate, cudaStream_t s);

}  // namespace k
}  // namespace ckf
