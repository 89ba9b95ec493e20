// Bandwidth kernels of the LLaMA-style stage block (llama_kernels.cu) and the
// flash attention kernels (attention.cu).  Activations are bf16, the residual
// stream and every reduction fp32; all reductions are deterministic.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>

#include "gemm_tc.h"

namespace ckf::llama {

using bf16 = __nv_bfloat16;
constexpr float kNormEps = 1e-5f;
constexpr float kRopeTheta = 10000.0f;

// h[t,:] = E[tok[t],:]  (fp32 master embedding rows)
void embed_fwd(const int* tok, size_t ntok, const float* E, size_t d, float* h, cudaStream_t s);
// gE[v,:] += sum over t with tok[t]==v of dh[t,:], summed in token order (stable sort) -> deterministic.
// scratch: >= embed_bwd_scratch(ntok) bytes
size_t embed_bwd_scratch(size_t ntok);
void embed_bwd(const int* tok, size_t ntok, const float* dh, size_t d, float* gE, void* scratch, cudaStream_t s);

// y = x * rsqrt(mean(x^2) + eps) * g  -> bf16; rstd[t]; xcopy (optional) = x
void rmsnorm_fwd(const float* x, const float* g, size_t rows, size_t d, bf16* y, float* rstd, float* xcopy,
                 cudaStream_t s);
// dh += d/dx rmsnorm(x) . dy ; dh_bf (optional) = bf16(dh after update);
// gain partials: gpart[blk, :] for blk < rmsnorm_bwd_blocks(rows) (fold with gain_fold)
int rmsnorm_bwd_blocks(size_t rows);
void rmsnorm_bwd(const float* dy, const float* x, const float* g, const float* rstd, size_t rows, size_t d, float* dh,
                 bf16* dh_bf, float* gpart, cudaStream_t s);
// gg[:] += sum_blk gpart[blk, :]  (fixed order)
void gain_fold(const float* gpart, int nblk, size_t d, float* gg, cudaStream_t s);

// rotary embedding on the q and k column blocks of qkv [ntok x 3d] in place;
// position = t % T; inverse = 1 applies the transpose (backward)
void rope(bf16* qkv, size_t ntok, size_t T, size_t d, size_t heads, int inverse, cudaStream_t s);
// device cos/sin table [T][hd/2] (float2), built on first use (the QKV GEMM epilogue reads it)
const float2* rope_table(size_t T, size_t hd, cudaStream_t s);
// the same values laid out [hd/2][T] (the GEMM epilogue's fused RoPE reads it)
const float2* rope_table_pair_major(size_t T, size_t hd, cudaStream_t s);

// a = silu(gate) * up ; gu = [gate | up] (ntok x 2f)
void swiglu_fwd(const bf16* gu, size_t ntok, size_t f, bf16* a, cudaStream_t s);
// dgu = [da * up * silu'(gate) | da * silu(gate)]
void swiglu_bwd(const bf16* gu, const bf16* da, size_t ntok, size_t f, bf16* dgu, cudaStream_t s);

// cross-entropy over bf16 logits rows: row_loss[r] = lse - logit[label]; logits are
// overwritten (in place) with (softmax - onehot) * grad_scale when grad != 0
void xent_bf16(bf16* logits, const int* labels, size_t rows, size_t V, float grad_scale, int grad, double* row_loss,
               cudaStream_t s);
// fused LM head + cross-entropy (head_xent.cu): row_loss[i] = lse_i - l_i,label (fp64), and when
// train: dxn = dlogits E_inv^T (fp32 store), gEinv += xn^T dlogits, dlogits = grad_scale (softmax -
// onehot) -- without a logits tensor.  xn [M x d] bf16, Einv [d x V] bf16 (row pitch V); ws >=
// head_xent_workspace(M, d, V) bytes.  gemm runs each GEMM (the caller's timing wrapper around
// tc::gemm_bf16); loss_kernels wraps the two small kernels likewise.
struct HeadXent {
  const bf16* xn = nullptr;
  const bf16* Einv = nullptr;
  const int* labels = nullptr;
  int M = 0, d = 0, V = 0;
  float grad_scale = 1.f;
  bool train = true;
  double* row_loss = nullptr;
  float* dxn = nullptr;
  float* gEinv = nullptr;
  void* ws = nullptr;
  // optional: the fp32 rows xn was normalised from (xn = bf16(h rstd g)); then the scaled copy for
  // the weight gradient is ONE rounding of s h rstd g instead of a second rounding of xn
  const float* h = nullptr;
  const float* rstd = nullptr;
  const float* gain = nullptr;
};
size_t head_xent_workspace(size_t M, size_t d, size_t V);
void head_xent(const HeadXent& h, const std::function<void(const tc::GemmDesc&)>& gemm,
               const std::function<void(const std::function<void()>&)>& loss_kernels, cudaStream_t s);
// *out = scale * sum(row_loss[0..rows)) in fixed order
void fold_mean(const double* row_loss, size_t rows, double scale, double* out, cudaStream_t s);

// labels of the token batch: lab[r*T + j] = x[r*(T+1) + j + 1]; inputs tok[r*T + j] = x[r*(T+1) + j]
void split_tokens(const int* x, size_t rows, size_t T, int* tok, int* lab, cudaStream_t s);

void f32_to_bf16(const float* x, bf16* y, size_t n, cudaStream_t s);

// ------------------------------------------------------------------ attention (attention.cu)
// q, k, v: bf16 column blocks of qkv [B*T x 3*H*hd] (row pitch ld = 3*H*hd); o [B*T x H*hd];
// lse [B*H*T] fp32 (natural log).  Causal, softmax scale 1/sqrt(hd).  hd in {64, 128}.
void attn_fwd(const bf16* qkv, size_t B, size_t T, size_t H, size_t hd, bf16* o, float* lse, cudaStream_t s);
// tcgen05/TMEM/TMA forward (attention_tc.cu) for head_dim 64, seq_len % 128 == 0
bool attn_fwd_tc_supported(size_t T, size_t hd);
long long* attn_fwd_debug_buffer();  // non-null only with CKF_ATTN_DEBUG=1
void attn_fwd_tc(const bf16* qkv, size_t B, size_t T, size_t H, size_t hd, bf16* o, float* lse, cudaStream_t s);
// rope_inverse: dq / dk leave with the RoPE backward applied (fused into the dK and dQ epilogues)
// d_ready: Dsum already holds D = rowsum(dout . o) (the O-projection dgrad's epilogue formed it)
void attn_bwd_tc(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
                 size_t hd, bf16* dqkv, float* Dsum, cudaStream_t s, bool rope_inverse = false, bool d_ready = false);
// dqkv [B*T x 3*H*hd]; Dsum scratch [B*H*T] fp32.  Deterministic (no atomics).
void attn_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, size_t B, size_t T, size_t H,
              size_t hd, bf16* dqkv, float* Dsum, cudaStream_t s);

}  // namespace ckf::llama
