// Issue throughput of the instructions the attention softmax loops are made of, on this GPU:
// ex2.approx (MUFU), cvt.rn.bf16x2.f32 (the P / dS packing), fma.rn.f32x2 (FFMA2), add.f32x2,
// 3-input max, prmt, iadd.  Each thread runs 8 independent chains of the op; 32 warps per SM.
// Prints lane-operations per clock per SM (clock64 on every SM, so the number is clock-exact).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_pipe_rates tools/pipe_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(1024) rate_kernel(float* out, long long* clk) {
  float a[8];
  unsigned u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = 0.001f * (threadIdx.x + i);
    u[i] = threadIdx.x * 7 + i;
  }
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if constexpr (OP == 1) {
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        u[i] ^= r;
      } else if constexpr (OP == 2) {
        unsigned long long v = (static_cast<unsigned long long>(__float_as_uint(a[i])) << 32) | __float_as_uint(a[i]);
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
        a[i] = __uint_as_float(static_cast<unsigned>(v));
      } else if constexpr (OP == 3) {
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      } else if constexpr (OP == 4) {
        asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      } else if constexpr (OP == 5) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      } else if constexpr (OP == 6) {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      } else if constexpr (OP == 7) {
        asm volatile("cvt.rn.bf16.f32 %0, %1;" : "=h"(*reinterpret_cast<unsigned short*>(&u[i])) : "f"(a[i]));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms) {
  float* out;
  long long* clk;
  cudaMalloc(&out, sizeof(float) * sms * 1024);
  cudaMalloc(&clk, sizeof(long long) * sms);
  rate_kernel<OP><<<sms, 1024>>>(out, clk);
  rate_kernel<OP><<<sms, 1024>>>(out, clk);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = 1024.0 * kIters * 8;  // lane-ops per SM
  printf("{\"op\": \"%s\", \"lane_ops_per_clk_per_sm\": %.2f}\n", name, ops / mx);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("ex2.approx.ftz.f32", sms);
  run<1>("cvt.rn.bf16x2.f32 (2 values)", sms);
  run<2>("fma.rn.f32x2 (2 values)", sms);
  run<3>("max.f32 3-input", sms);
  run<4>("prmt.b32", sms);
  run<5>("add.u32", sms);
  run<6>("fma.rn.f32", sms);
  run<7>("cvt.rn.bf16.f32", sms);
  return 0;
}
