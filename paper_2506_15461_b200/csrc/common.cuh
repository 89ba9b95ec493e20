// Shared device/host helpers for the B200 CheckFree engine (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace ckf {

// ---------------------------------------------------------------- errors
// Internal C++ errors; the C-ABI layer (capi.cu) maps them to CKF_E_* codes.
struct Error : std::runtime_error {
  int code;
  long iteration;
  Error(int c, const std::string& m, long it = -1) : std::runtime_error(m), code(c), iteration(it) {}
};

// Bumped whenever a device buffer that a captured CUDA graph could reference is
// (re)allocated (engine workspace slots, GEMM split-K scratch, RoPE tables): a graph
// captured under another epoch is stale.
inline long& alloc_epoch() {
  static long e = 0;
  return e;
}

[[noreturn]] inline void raise(int code, const std::string& msg, long it = -1) { throw Error(code, msg, it); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    raise(6, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")");
}
#define CKF_CUDA(x) ::ckf::cuda_check((x), #x, __FILE__, __LINE__)
// Every launch site is followed by CKF_LAUNCH_CHECK(); it also counts the
// launches of this library's own kernels (the evidence behind gpu_launches).
long& launch_counter();
#define CKF_LAUNCH_CHECK()                                                          \
  do {                                                                              \
    ++::ckf::launch_counter();                                                      \
    ::ckf::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);    \
  } while (0)

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// ---------------------------------------------------------------- counter RNG
// SplitMix64 finaliser and the counter generator of include/ckfree/rng.hpp:10-44,
// evaluated on the device.  Integer arithmetic is exact; the affine
// lo + (hi-lo)*u uses explicit round-to-nearest ops so nvcc cannot contract it
// into an FMA -> bit-exact with the x86-64 reference.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t derive_key(uint64_t seed, uint64_t a = 0, uint64_t b = 0,
                                                        uint64_t c = 0) {
  uint64_t h = mix64(seed ^ 0x6a09e667f3bcc909ULL);
  h = mix64(h ^ a);
  h = mix64(h ^ b);
  return mix64(h ^ c);
}

// SwiGLU element math shared by the standalone kernels (llama_kernels.cu) and the
// fused GEMM epilogues (gemm_tc.cu), so both produce the same bits.  Branch-free
// (approximate reciprocal): the fused epilogue issues it from one warp per SM
// sub-partition and needs the ILP.
__device__ __forceinline__ float swiglu_sig(float g) { return __fdividef(1.f, 1.f + __expf(-g)); }
__device__ __forceinline__ float swiglu_fwd1(float g, float u) { return g * swiglu_sig(g) * u; }
// d = dL/da; writes dL/dg, dL/du
__device__ __forceinline__ void swiglu_bwd1(float g, float u, float d, float& dg, float& du) {
  const float sg = swiglu_sig(g);
  dg = d * u * sg * (1.f + g * (1.f - sg));
  du = d * g * sg;
}

__device__ __forceinline__ double counter_uniform_at(uint64_t key, uint64_t counter, double lo, double hi) {
  const uint64_t bits = mix64(key + counter * 0x9e3779b97f4a7c15ULL);
  const double u = __dmul_rn(static_cast<double>(bits >> 11), 0x1.0p-53);
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}

// ---------------------------------------------------------------- dtype traits
template <typename T> struct Num;
template <> struct Num<double> {
  static __device__ __forceinline__ double from_d(double x) { return x; }
  static __device__ __forceinline__ double to_d(double x) { return x; }
};
template <> struct Num<float> {
  static __device__ __forceinline__ float from_d(double x) { return static_cast<float>(x); }
  static __device__ __forceinline__ double to_d(float x) { return static_cast<double>(x); }
};

// ---------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree); result valid in thread 0.
template <typename T, int kThreads>
__device__ __forceinline__ T block_sum(T v) {
  __shared__ T red[kThreads / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = 0;
  if (w == 0) {
    r = l < kThreads / 32 ? red[l] : T(0);
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

inline unsigned grid_for(size_t n, int per_block, int cap = kNumSMs * 16) {
  size_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > static_cast<size_t>(cap)) g = cap;
  return static_cast<unsigned>(g);
}

}  // namespace ckf
