// Fused LM head + cross-entropy (replaces logits = xn E_inv -> softmax_xent_loss_grad ->
// dlogits E_inv^T / xn^T dlogits of proj/src/model.cpp:250-253,322-342 and
// proj/src/kernels_serial.cpp:163-185 on the LLaMA bf16 path).
//
// No logits tensor is written and no pass over [M x V] runs outside the tensor-core GEMMs.
// With a per-row shift c_i the loss gradient factors as
//     dlogits[i, v] = grad_scale * (p_iv - [v == y_i]) = s_i * Q[i, v],
//     Q[i, v] = exp(l_iv - c_i)  (v != y_i),   Q[i, y_i] = expm1(l_iy - lse_i) * S_i,
//     S_i = sum_v exp(l_iv - c_i),   s_i = grad_scale / S_i,   lse_i = c_i + log S_i,
// so:
//   1. c_i = max of row i over the first 256 vocabulary columns (a 256-column GEMM + row max):
//      c_i <= max_v l_iv, hence S_i >= 1 (no underflow); the head GEMM's epilogue guards the
//      other side (a logit more than kXentGuard = 50 above c_i raises a device flag and a gated
//      rerun uses the row's true maximum -- no host round trip, always correct);
//   2. the head GEMM (epilogue kXentFwd, gemm_tc.cu) computes e = exp(l - c) from the fp32
//      accumulator, stores Q = bf16(e) (training only), the fp32 partial row sums per 128-column
//      half tile and the label's fp32 logit;
//   3. xent_combine: S_i in fixed order, lse, the row loss (fp64), s_i, the label entry of Q
//      (p - 1 through expm1, exact to fp32 before its bf16 rounding), and xs = bf16(s_i xn_i);
//   4. dxn = s_i (Q E_inv^T) (fp32-store epilogue with a per-row scale) and
//      gE_inv += xs^T Q -- the reference's two head backward GEMMs on Q.
// Numerics against the unfused path: every gradient entry is still one bf16 rounding of its
// fp32 value (Q is rounded where dlogits was), the probabilities come from fp32 logits instead
// of bf16-rounded ones, the loss from fp32 logits (tests/test_gpu_xent.py).
#include <algorithm>
#include <cmath>
#include <functional>

#include "common.cuh"
#include "gemm_tc.h"
#include "llama_kernels.h"
#include "sm100.cuh"

namespace ckf::llama {
namespace {

constexpr int kShiftCols = 256;
constexpr int kCombineRows = 128;

__device__ __forceinline__ int ord_of(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float f_of(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// c[i] = max_j l0[i, j] (j < ncols); vmax[i] = "none"; *flag = 0.  One warp per row.
__global__ void xent_shift_kernel(const float* __restrict__ l0, int M, int ncols, float* __restrict__ c,
                                  int* __restrict__ vmax, int* __restrict__ flag) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 0;
  if (warp >= M) return;
  const float* row = l0 + static_cast<size_t>(warp) * ncols;
  float m = -INFINITY;
  for (int j = lane; j < ncols; j += 32) m = fmaxf(m, row[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) {
    c[warp] = m;
    vmax[warp] = ord_of(-INFINITY);
  }
}

// Per row: S (fixed order over the partials), lse, row loss; training: s = grad_scale / S, the
// label entry of Q, and xs = bf16(s * xn) for the weight-gradient GEMM.
__global__ void __launch_bounds__(kCombineRows) xent_combine_kernel(
    const float* __restrict__ psum, int P, int M, const float* __restrict__ c, const int* __restrict__ vmax,
    const float* __restrict__ ly, const int* __restrict__ labels, float grad_scale, int train,
    double* __restrict__ row_loss, float* __restrict__ s_out, bf16* __restrict__ Q, int V,
    const bf16* __restrict__ xn, const float* __restrict__ h32, const float* __restrict__ rstd,
    const float* __restrict__ gain, bf16* __restrict__ xs, int d) {
  __shared__ float s_sm[kCombineRows];
  const int r0 = blockIdx.x * kCombineRows;
  const int i = r0 + threadIdx.x;
  if (i < M) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // four chains, folded in a fixed order
    int k = 0;
    for (; k + 4 <= P; k += 4) {
      a0 += psum[static_cast<size_t>(k) * M + i];
      a1 += psum[static_cast<size_t>(k + 1) * M + i];
      a2 += psum[static_cast<size_t>(k + 2) * M + i];
      a3 += psum[static_cast<size_t>(k + 3) * M + i];
    }
    for (; k < P; ++k) a0 += psum[static_cast<size_t>(k) * M + i];
    const float S = (a0 + a1) + (a2 + a3);
    const double cr = static_cast<double>(fmaxf(c[i], f_of(vmax[i])));
    const double lse = cr + log(static_cast<double>(S));
    const double lyd = static_cast<double>(ly[i]);
    row_loss[i] = lse - lyd;
    if (train) {
      const float s = grad_scale / S;
      s_sm[threadIdx.x] = s;
      s_out[i] = s;
      Q[static_cast<size_t>(i) * V + labels[i]] = __float2bfloat16_rn(static_cast<float>(expm1(lyd - lse)) * S);
    }
  }
  if (!train) return;
  __syncthreads();
  // xs rows of this block: 8 columns per thread, consecutive threads on consecutive chunks
  const int rows = min(kCombineRows, M - r0);
  const int cpr = d / 8;  // chunks per row
  if (h32) {  // one rounding of s * h * rstd * g (what xn rounded once)
    if (threadIdx.x < rows) s_sm[threadIdx.x] *= rstd[r0 + threadIdx.x];
    __syncthreads();
    for (int t = threadIdx.x; t < rows * cpr; t += kCombineRows) {
      const int rr = t / cpr, cc = t - rr * cpr;
      const size_t off = static_cast<size_t>(r0 + rr) * d + static_cast<size_t>(cc) * 8;
      const float4 a = *reinterpret_cast<const float4*>(h32 + off), b = *reinterpret_cast<const float4*>(h32 + off + 4);
      const float4 ga = *reinterpret_cast<const float4*>(gain + cc * 8), gb = *reinterpret_cast<const float4*>(gain + cc * 8 + 4);
      const float s = s_sm[rr];
      *reinterpret_cast<uint4*>(xs + off) =
          make_uint4(sm100::pack_bf16(a.x * s * ga.x, a.y * s * ga.y), sm100::pack_bf16(a.z * s * ga.z, a.w * s * ga.w),
                     sm100::pack_bf16(b.x * s * gb.x, b.y * s * gb.y), sm100::pack_bf16(b.z * s * gb.z, b.w * s * gb.w));
    }
    return;
  }
  for (int t = threadIdx.x; t < rows * cpr; t += kCombineRows) {
    const int rr = t / cpr, cc = t - rr * cpr;
    const size_t off = static_cast<size_t>(r0 + rr) * d + static_cast<size_t>(cc) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(xn + off);
    const float s = s_sm[rr];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      o[e] = sm100::pack_bf16(__uint_as_float(w[e] << 16) * s, __uint_as_float(w[e] & 0xffff0000u) * s);
    *reinterpret_cast<uint4*>(xs + off) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace

size_t head_xent_workspace(size_t M, size_t d, size_t V) {
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t P = static_cast<size_t>(tc::xent_partials(static_cast<int>(V)));
  return al(M * V * 2) + al(std::max<size_t>(P, kShiftCols) * M * 4) + 4 * al(M * 4) + al(4) + al(M * d * 2);
}

void head_xent(const HeadXent& h, const std::function<void(const tc::GemmDesc&)>& gemm,
               const std::function<void(const std::function<void()>&)>& loss_kernels, cudaStream_t st) {
  if (h.M <= 0) return;
  if (h.V % 8 || h.d % 8) raise(1, "head_xent: vocabulary and model width must be multiples of 8");
  if (h.h && (!h.rstd || !h.gain)) raise(1, "head_xent: h needs rstd and gain");
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const int M = h.M, d = h.d, V = h.V, P = tc::xent_partials(V);
  char* p = static_cast<char*>(h.ws);
  auto take = [&](size_t b) {
    char* r = p;
    p += al(b);
    return r;
  };
  bf16* Q = reinterpret_cast<bf16*>(take(static_cast<size_t>(M) * V * 2));
  float* psum = reinterpret_cast<float*>(take(static_cast<size_t>(std::max(P, kShiftCols)) * M * 4));
  float* c = reinterpret_cast<float*>(take(static_cast<size_t>(M) * 4));
  int* vmax = reinterpret_cast<int*>(take(static_cast<size_t>(M) * 4));
  float* ly = reinterpret_cast<float*>(take(static_cast<size_t>(M) * 4));
  float* s = reinterpret_cast<float*>(take(static_cast<size_t>(M) * 4));
  int* flag = reinterpret_cast<int*>(take(4));
  bf16* xs = reinterpret_cast<bf16*>(take(static_cast<size_t>(M) * d * 2));

  // 1. shift: the first 256 logit columns of every row (fp32, in the partial-sum buffer)
  const int n0 = std::min(V, kShiftCols);
  tc::GemmDesc g0;
  g0.M = M;
  g0.N = n0;
  g0.K = d;
  g0.A = h.xn;
  g0.lda = d;
  g0.B = h.Einv;
  g0.ldb = V;
  g0.b_mn = true;
  g0.C = psum;
  g0.ldc = n0;
  g0.epi = tc::kStoreF32;
  gemm(g0);
  loss_kernels([&] {
    xent_shift_kernel<<<static_cast<unsigned>((M + 7) / 8), 256, 0, st>>>(psum, M, n0, c, vmax, flag);
    CKF_LAUNCH_CHECK();
  });
  // 2. head GEMM with the cross-entropy epilogue, and its gated rerun
  tc::GemmDesc g;
  g.M = M;
  g.N = V;
  g.K = d;
  g.A = h.xn;
  g.lda = d;
  g.B = h.Einv;
  g.ldb = V;
  g.b_mn = true;
  g.C = Q;
  g.ldc = V;
  g.epi = tc::kXentFwd;
  g.xent.labels = h.labels;
  g.xent.c = c;
  g.xent.vmax = vmax;
  g.xent.psum = psum;
  g.xent.ly = ly;
  g.xent.flag = flag;
  g.xent.store = h.train ? 1 : 0;
  gemm(g);
  g.gate = flag;
  gemm(g);
  // 3. row statistics, loss, gradient scale, label entries, scaled xn
  loss_kernels([&] {
    xent_combine_kernel<<<static_cast<unsigned>((M + kCombineRows - 1) / kCombineRows), kCombineRows, 0, st>>>(
        psum, P, M, c, vmax, ly, h.labels, h.grad_scale, h.train ? 1 : 0, h.row_loss, s, Q, V, h.xn, h.h, h.rstd,
        h.gain, xs, d);
    CKF_LAUNCH_CHECK();
  });
  if (!h.train) return;
  // 4. head backward on Q: gE_inv += xs^T Q ; dxn = s * (Q E_inv^T)
  tc::GemmDesc gw;
  gw.M = d;
  gw.N = V;
  gw.K = M;
  gw.A = xs;
  gw.lda = d;
  gw.a_mn = true;
  gw.B = Q;
  gw.ldb = V;
  gw.b_mn = true;
  gw.C = h.gEinv;
  gw.ldc = V;
  gw.epi = tc::kAccF32;
  gemm(gw);
  tc::GemmDesc gd;
  gd.M = M;
  gd.N = d;
  gd.K = V;
  gd.A = Q;
  gd.lda = V;
  gd.B = h.Einv;
  gd.ldb = V;
  gd.C = h.dxn;
  gd.ldc = d;
  gd.epi = tc::kStoreF32;
  gd.row_scale = s;
  gemm(gd);
}

}  // namespace ckf::llama
