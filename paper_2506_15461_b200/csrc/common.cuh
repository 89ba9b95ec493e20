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
// Packed fp32x2 arithmetic of sm_100 (FFMA2 / FADD2 / FMUL2: two IEEE fp32 operations per
// instruction, each lane rounding exactly like its scalar counterpart) and the 3-input max.
using f32x2 = unsigned long long;
__device__ __forceinline__ f32x2 f2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2split(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA / ALU pipes -- the MUFU offload of FlashAttention-4: the softmax of
// a head_dim-64 tile needs one exponential per 256 MMA FLOPs, which at 16 MUFU results / clk / SM
// caps the tensor pipe near half of its peak, while the issue slots have room.  x = j + f with
// j = rint(x) (the 1.5 * 2^23 trick), 2^f by a degree-3 minimax polynomial on [-0.5, 0.5]
// (relative error 7.5e-5, below a bf16 half-ulp of 2e-3), 2^j added into the exponent field.
// x is clamped at -125 (the result is then ~2^-125, zero for a bf16 probability).
__device__ __forceinline__ f32x2 ex2_fma2(f32x2 x) {
  float a, b;
  f2split(x, a, b);
  const f32x2 xc = f2(fmaxf(a, -125.f), fmaxf(b, -125.f));
  const f32x2 t = fadd2(xc, f2(12582912.f, 12582912.f));  // low mantissa bits = rint(x)
  const f32x2 j = fadd2(t, f2(-12582912.f, -12582912.f));
  const f32x2 fr = ffma2(j, f2(-1.f, -1.f), xc);            // f = x - j in [-0.5, 0.5]
  f32x2 p = ffma2(fr, f2(0.05517083778977394f, 0.05517083778977394f),
                  f2(0.24260935187339783f, 0.24260935187339783f));
  p = ffma2(fr, p, f2(0.6932609677314758f, 0.6932609677314758f));
  p = ffma2(fr, p, f2(0.9999281764030457f, 0.9999281764030457f));
  float pa, pb, ta, tb;
  f2split(p, pa, pb);
  f2split(t, ta, tb);
  // bits(t) = 0x4B400000 + j, and 0x4B400000 << 23 vanishes mod 2^32: this adds j to the exponent
  return f2(__uint_as_float(__float_as_uint(pa) + (__float_as_uint(ta) << 23)),
            __uint_as_float(__float_as_uint(pb) + (__float_as_uint(tb) << 23)));
}

// SwiGLU on pairs of columns, one fixed instruction sequence shared by the fused GEMM
// epilogues and the standalone kernels (so the two paths stay bit-identical):
// sig(g) = rcp(1 + 2^(-g log2 e)) (MUFU ex2 / rcp), a = g sig(g) u,
// dg = d u sig (1 + g (1 - sig)), du = d g sig.
__device__ __forceinline__ f32x2 swiglu_sig2(f32x2 g) {
  float e0, e1;
  f2split(fmul2(g, f2(-1.4426950408889634f, -1.4426950408889634f)), e0, e1);
  asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(e0));
  asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(e1));
  float d0, d1;
  f2split(fadd2(f2(e0, e1), f2(1.f, 1.f)), d0, d1);
  asm("rcp.approx.ftz.f32 %0, %0;" : "+f"(d0));
  asm("rcp.approx.ftz.f32 %0, %0;" : "+f"(d1));
  return f2(d0, d1);
}
__device__ __forceinline__ f32x2 swiglu_fwd2(f32x2 g, f32x2 u) { return fmul2(fmul2(g, swiglu_sig2(g)), u); }
// d = dL/da; returns dL/dg, dL/du
__device__ __forceinline__ void swiglu_bwd2(f32x2 g, f32x2 u, f32x2 d, f32x2& dg, f32x2& du) {
  const f32x2 sg = swiglu_sig2(g), one = f2(1.f, 1.f);
  du = fmul2(fmul2(d, g), sg);
  const f32x2 inner = ffma2(g, ffma2(sg, f2(-1.f, -1.f), one), one);  // 1 + g (1 - sig)
  dg = fmul2(fmul2(fmul2(d, u), sg), inner);
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
