/*
 * ckf.h -- the C-ABI boundary of the B200 CheckFree / CheckFree+ engine.
 *
 * Plain C: opaque handles, plain pointers and sizes, int status codes; no
 * C++ or torch types cross this line.  Host C++ (the drop-in `ckfree::` API
 * under include/ckfree/, and the reference itself via INTEGRATION.md) calls
 * CUDA only through these entry points.  Each group cites the reference
 * interface it replaces (paths relative to /root/reference/proj).
 *
 * Error convention: every entry point returns CKF_OK (0) or a CKF_E_* code
 * mirroring the reference's exception types (include/ckfree/errors.hpp:10-45);
 * the message is in ckf_last_error() (thread-local).  Nothing here throws.
 */
#ifndef CKF_H_
#define CKF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
enum ckf_status {
  CKF_OK = 0,
  CKF_E_CONFIG = 1,               /* ConfigError                (errors.hpp:10-13) */
  CKF_E_DIVERGENCE = 2,           /* NumericDivergenceError     (errors.hpp:15-26) */
  CKF_E_USAGE = 3,                /* UsageError                 (errors.hpp:28-32) */
  CKF_E_PARSE = 4,                /* ParseError                 (errors.hpp:34-38) */
  CKF_E_UNSUPPORTED_RECOVERY = 5, /* UnsupportedRecoveryError   (errors.hpp:40-45) */
  CKF_E_CUDA = 6,
  CKF_E_NCCL = 7
};

const char* ckf_last_error(void);
/* iteration carried by the last CKF_E_DIVERGENCE, -1 outside a training loop */
long ckf_last_error_iteration(void);
int ckf_version(void);
int ckf_device_count(int* out);

/* enumerations shared with the reference */
enum ckf_activation { CKF_ACT_TANH = 0, CKF_ACT_RELU = 1, CKF_ACT_IDENTITY = 2 }; /* kernels.hpp:19 */
enum ckf_task { CKF_TASK_REGRESSION = 0, CKF_TASK_CLASSIFICATION = 1 };           /* model.hpp:16 */
enum ckf_dtype { CKF_FP64 = 0, CKF_FP32 = 1, CKF_BF16 = 2 };

/* =====================================================================
 * (0) Host control logic (no GPU needed), bit-exact with the reference:
 *     failure traces (src/failures.cpp:57-196), even partition
 *     (src/model.cpp:63-73) and microbatch schedules (src/pipeline.cpp:11-56).
 * ===================================================================== */
/* generate_trace + serialize_trace ("checkfree-trace v1") into out */
int ckf_generate_trace(uint64_t seed, double p_hour, double iter_s, long n_iters, const int* stages, int n_stages,
                       char* out, size_t cap);
/* parse_trace (ParseError on malformed input) then canonical re-serialization */
int ckf_parse_trace(const char* text, char* out, size_t cap);
/* consecutive_conflicts: writes (iteration, stage) pairs, *n_out pairs */
int ckf_consecutive_conflicts(const char* text, long* out, int cap_pairs, int* n_out);
double ckf_hourly_to_per_iteration(double p_hour, double iter_s);
/* layers -> stages: writes 2*stages (first,last) 1-based */
int ckf_even_partition(size_t layers, size_t stages, size_t* out);
/* m execution orders of length s (standard, or swapped at even positions) */
int ckf_build_schedule(int m, int swapped_half, int s, int* out);

/* Multi-GPU pipeline plan: the global op sequence of one iteration for a
 * stage -> rank placement (stage_rank[s]), exactly as every rank of the engine
 * issues it.  6 ints per op: phase (0 fwd / 1 bwd), microbatch, kind
 * (0 embed fwd, 1 stage fwd, 2 transfer, 3 head = loss + head backward,
 * 4 stage bwd, 5 embed bwd), rank (transfer: source), arg (stage id, or the
 * transfer's destination rank), aux (transfer: 0 activations, 1 gradients).
 * schedule: 0 = forward+backward per microbatch (pipeline.cpp:66-81 order),
 * 1 = GPipe (all forwards, then all backwards in microbatch order). */
/* schedule 2 = 1F1B (host-simulated list schedule, see host_logic.cpp): stage_cost (s forward time
 * units, may be NULL = 1 each) and head_cost weigh the simulation; the engine uses its own costs
 * (ckf_engine_plan_cost).  ckf_pipeline_plan is ckf_pipeline_plan_cost with unit costs. */
int ckf_pipeline_plan_cost(int s, int m, const int* orders, const int* stage_rank, int schedule,
                           const double* stage_cost, double head_cost, int* out, int cap_ops, int* n_ops);
int ckf_pipeline_plan(int s, int m, const int* orders, const int* stage_rank, int schedule, int* out, int cap_ops,
                      int* n_ops);

/* =====================================================================
 * (1) L1 kernel seam.  Replaces the dispatching wrappers of
 *     ckfree::kernels (include/ckfree/kernels.hpp:26-69,
 *     src/kernels_dispatch.cpp:37-83) as a third Backend: identical
 *     signatures (HOST fp64 pointers), computed on the current CUDA device
 *     in fp64.  Staging through a device arena is internal.
 * ===================================================================== */
int ckf_k_gemm_nn(const double* a, const double* b, double* c, size_t m, size_t k, size_t n);
int ckf_k_gemm_nn_acc(const double* a, const double* b, double* c, size_t m, size_t k, size_t n);
int ckf_k_gemm_nt_acc(const double* a, const double* b, double* c, size_t m, size_t k, size_t n);
int ckf_k_gemm_tn_acc(const double* a, const double* b, double* c, size_t m, size_t k, size_t n);
int ckf_k_add_inplace(double* x, const double* y, size_t n);
int ckf_k_axpy(double alpha, const double* x, double* y, size_t n);
int ckf_k_scale(double alpha, double* x, size_t n);
int ckf_k_apply_activation(int act, const double* a, double* z, size_t n);
int ckf_k_activation_backward(int act, const double* z, const double* dz, double* da, size_t n);
int ckf_k_sum_squares(const double* x, size_t n, double* out);
int ckf_k_sum_squared_diff(const double* x, const double* y, size_t n, double* out);
int ckf_k_adam_update(double* w, double* m, double* v, const double* g, size_t n, double lr, double beta1,
                      double beta2, double eps, long step);
int ckf_k_mse_loss_grad(const double* pred, const double* target, size_t rows, size_t cols, double* dpred,
                        double* loss);
int ckf_k_softmax_xent_loss_grad(const double* logits, const int* labels, size_t rows, size_t cols,
                                 double* dlogits, double* loss);
/* recovery::recover_checkfree on flat host vectors (src/recovery.cpp:57-73) */
int ckf_k_recover_checkfree(const double* w_prev, const double* w_next, size_t n, double omega_prev,
                            double omega_next, double* out, int* degenerate);
/* n draws of CounterRng(key).uniform(lo, hi), counters 1..n (include/ckfree/rng.hpp:37-44), bit-exact */
int ckf_k_counter_uniform(uint64_t key, double lo, double hi, double* out, size_t n);

/* =====================================================================
 * (2) Device-pointer primitives (the hot kernels on their own, for
 *     benchmarks and for callers that keep state in HBM).  `stream` is a
 *     cudaStream_t (NULL = legacy default stream).
 * ===================================================================== */
/* out = (op*wp + on*wn)/(op+on) (recovery.cpp:57-73) in one streaming pass.
 * dtype CKF_FP64 is bit-exact with the reference (no FMA contraction); CKF_FP32
 * computes the coefficients in fp64 and one FMA per element.  wp/wn may be peer
 * (NVLink) pointers.  If old_out_sq is non-NULL the pass also reduces
 * ||out_before - out_after||^2 (reduction_error, recovery.cpp:120-126) into it
 * (device double*, deterministic order).  op+on == 0 -> uniform (degenerate). */
int ckf_recover_device(int dtype, const void* wp, const void* wn, void* out, size_t n, double op, double on,
                       double* old_out_sq, void* stream);
/* The engine's fused stage recovery on raw device pointers -- ONE streaming pass
 * (recovery.cpp:57-73 + trainer.cpp:230-276): w = (op*wp + on*wn)/(op+on) (degenerate
 * 0,0 -> uniform), moments Fresh (averaged = 0: m = v = 0) or omega-weighted from mp/mn,
 * vp/vn (averaged = 1, trainer.cpp:263-269), g = 0, bf16 shadow w_bf16 (may be NULL),
 * optional ||w_old - w_new||^2 into *old_sq (device double).  wp / wn / mp / mn / vp / vn
 * may be PEER pointers (another GPU's HBM mapped with CUDA IPC or peer access), which is
 * how a replacement GPU pulls its neighbours over NVLink inside the kernel. */
int ckf_recover_stage_device(int dtype, const void* wp, const void* wn, const void* mp, const void* mn,
                             const void* vp, const void* vn, void* w, void* m, void* v, void* g, void* w_bf16,
                             size_t n, double omega_prev, double omega_next, int averaged, double* old_sq,
                             void* stream);
/* fused Adam (kernels_serial.cpp:133-144) + omega = sum(g^2) (model.cpp:396):
 * g_eff = g_sum * grad_scale; w,m,v updated in place; if w_bf16 != NULL the bf16
 * shadow is rewritten; if zero_grad the accumulator is cleared for the next
 * iteration; omega (device double*) receives sum(g_eff^2).  bc1/bc2 are the
 * host-computed 1-beta^step (pow on the host). */
int ckf_adam_device(int dtype, void* w, void* m, void* v, void* g, void* w_bf16, size_t n, double lr,
                    double bc1, double bc2, double grad_scale, int zero_grad, double* omega, void* stream);

/* bf16 tensor-core GEMM (tcgen05 + TMA, fp32 accumulation in TMEM), the
 * stage-GEMM primitive that replaces gemm_nn / gemm_nn_acc / gemm_nt_acc /
 * gemm_tn_acc (kernels_serial.cpp:13-61) on the bf16 path:
 *   C[M,N] (epi) alpha * op(A) op(B)
 *   a_mn = 0: A stored [M][lda] (K contiguous), 1: A stored [K][lda] (M contiguous)
 *   b_mn = 0: B stored [N][ldb] (K contiguous), 1: B stored [K][ldb] (N contiguous)
 *   epi  = 0: C bf16 store, 1: C fp32 store, 2: C fp32 += (gradient accumulation)
 *   bn   = 0 (heuristic), 128 or 256: N tile.  Device pointers; lda/ldb % 8 == 0. */
int ckf_gemm_bf16(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
                  int ldc, int epi, float alpha, int bn, void* stream);
/* Same GEMM with the fused SwiGLU epilogues of the LLaMA MLP (gemm_tc.h):
 *   epi = 3 (forward, N = 2f, B MN-major): C = gu [M x 2f] bf16, aux = a [M x f] = silu(g) * u
 *   epi = 4 (dgrad da = dY Wd^T, N = f, B K-major): aux = gu (read), C = dgu [M x 2f] bf16 (ldc = 2f) */
// LLaMA head loss on DEVICE buffers (llama_kernels.cu xent_bf16): per-row loss lse - logit[label]
// into row_loss (fp64); with grad != 0 the bf16 logits are overwritten in place by
// grad_scale * (softmax - onehot).
int ckf_xent_bf16(void* logits, const int* labels, size_t rows, size_t V, float grad_scale, int grad, double* row_loss,
                  void* stream);
int ckf_gemm_bf16_aux(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
                      int ldc, int epi, float alpha, int bn, void* aux, int ldaux, void* stream);
// Fused LM head + cross-entropy on DEVICE buffers (head_xent.cu; replaces the logits GEMM ->
// softmax_xent_loss_grad -> head backward GEMMs of proj/src/model.cpp:250-253,322-342 and
// proj/src/kernels_serial.cpp:163-185 without a logits tensor): xn [M x d] bf16, Einv [d x V] bf16,
// labels [M]; row_loss[i] = logsumexp - logit[label] (fp64); train != 0: dxn [M x d] fp32 =
// dlogits Einv^T (stored), gEinv [d x V] fp32 += xn^T dlogits, dlogits = grad_scale (softmax -
// onehot).  Optional h [M x d] fp32, rstd [M], gain [d] (xn = bf16(h rstd gain), the final
// RMSNorm's input): the weight gradient's scaled rows are then rounded once from them (NULL: from
// xn).  ws: ckf_lm_head_xent_workspace(M, d, V) bytes of device memory.
size_t ckf_lm_head_xent_workspace(size_t M, size_t d, size_t V);
int ckf_lm_head_xent(const void* xn, const void* Einv, const int* labels, size_t M, size_t d, size_t V, float grad_scale,
                     int train, double* row_loss, float* dxn, float* gEinv, const float* h, const float* rstd,
                     const float* gain, void* ws, void* stream);

/* Causal attention of the LLaMA block on device bf16 buffers: qkv [B*T x 3*H*hd]
 * (q | k | v column blocks), o [B*T x H*hd], lse [B*H*T] fp32 (natural log).
 * impl: 0 = default for the shape, 1 = mma.sync flash kernel, 2 = tcgen05/TMEM
 * kernel (head_dim 64 or 128, T % 128 == 0).  Backward: dout [B*T x H*hd] ->
 * dqkv [B*T x 3*H*hd]; Dsum = [B*H*T] fp32 scratch.  Backward impl | CKF_ATTN_ROPE_BWD:
 * the dq / dk blocks leave with the RoPE backward (ckf_llama_rope inverse = 1) applied --
 * fused into the tcgen05 kernel's dK and dQ epilogues (one bf16 rounding instead of two). */
#define CKF_ATTN_ROPE_BWD 16
int ckf_attention_fwd(const void* qkv, size_t B, size_t T, size_t H, size_t hd, void* o, float* lse, int impl,
                      void* stream);
int ckf_attention_bwd(const void* qkv, const void* o, const float* lse, const void* dout, size_t B, size_t T,
                      size_t H, size_t hd, void* dqkv, float* Dsum, int impl, void* stream);

/* LLaMA block bandwidth kernels on DEVICE buffers (llama_kernels.cu), exported so each is
 * pinned on its own against fp32 torch at every width the workloads run:
 *   rmsnorm_fwd: y = bf16(x * rsqrt(mean(x^2) + 1e-5) * g), rstd[row], xcopy (optional) = x
 *   rmsnorm_bwd: dh += d rmsnorm(x)/dx . dy (fp32), dh_bf (optional) = bf16(dh), gg += gain grad
 *   rope: rotary embedding (theta 1e4, pairs (j, j+hd/2), position t % T) in place on the q and
 *         k column blocks of qkv [ntok x 3d]; inverse = 1 applies the transpose (backward)
 *   swiglu_fwd: a = silu(gate) * up, gu = [gate | up] [ntok x 2f];  swiglu_bwd: dgu from da
 *   embed_fwd: h = E[tok];  embed_bwd: gE[v] += sum of dh over tok == v (token order, deterministic)
 *   gemm_qkv_rope: C = bf16(A B) with RoPE fused into the epilogue on the first 2d columns
 *         (A [M x K] K-major, B [K x 3d] N-major; head_dim 64 or 128), as the QKV projection runs it */
int ckf_llama_rmsnorm_fwd(const float* x, const float* g, size_t rows, size_t d, void* y_bf16, float* rstd,
                          float* xcopy, void* stream);
int ckf_llama_rmsnorm_bwd(const float* dy, const float* x, const float* g, const float* rstd, size_t rows, size_t d,
                          float* dh, void* dh_bf16, float* gg, void* stream);
int ckf_llama_rope(void* qkv, size_t ntok, size_t T, size_t d, size_t heads, int inverse, void* stream);
int ckf_llama_swiglu_fwd(const void* gu, size_t ntok, size_t f, void* a, void* stream);
int ckf_llama_swiglu_bwd(const void* gu, const void* da, size_t ntok, size_t f, void* dgu, void* stream);
int ckf_llama_embed_fwd(const int* tok, size_t ntok, const float* E, size_t d, float* h, void* stream);
int ckf_llama_embed_bwd(const int* tok, size_t ntok, const float* dh, size_t d, float* gE, void* stream);
int ckf_gemm_qkv_rope(int M, int K, const void* A, const void* B, void* C, size_t T, size_t heads, void* stream);
/* O-projection dgrad with the attention backward's D in its epilogue, as the LLaMA block runs it:
 * dO = bf16(dH W^T) (dH [M x K] K-major, W [N x K] = Wo stored [K][N] read K-major, N = K = d)
 * into C [M x N], and D[(b * H + h) * T + q] = sum over the head's columns of bf16(dO) * O for
 * row = b * T + q, O [M x N] bf16, heads of hd = N / heads (64 or 128) columns. */
int ckf_gemm_o_dgrad_dsum(int M, int K, const void* A, const void* B, void* C, const void* O, float* D, size_t T,
                          size_t heads, void* stream);

/* LLaMA token stream (csrc/tokens.cu): rows x (T+1) int32 ids keyed
 * (data_seed, stream, index) like the reference's batches (dataset.cpp:15-20),
 * generated on the device, copied to host `out`. */
int ckf_llama_token_batch(uint64_t data_seed, uint64_t stream, uint64_t index, size_t rows, size_t T, size_t V,
                          int* out);

/* =====================================================================
 * (3) Device-resident engine: the throughput tier behind
 *     ckfree::pipeline::run_iteration (pipeline.hpp:44-47),
 *     ckfree::recovery (recovery.hpp:46-86) and harness::Trainer
 *     (src/trainer.cpp:63-289).
 * ===================================================================== */
typedef struct ckf_engine_s* ckf_engine_t;

enum ckf_block { CKF_BLOCK_MLP = 0, CKF_BLOCK_LLAMA = 1 };

typedef struct {
  int block;      /* ckf_block: residual MLP x + act(xW1)W2 (model.hpp:55-60) or LLaMA */
  int precision;  /* ckf_dtype of the arithmetic: FP64 / FP32 (parity) or BF16 (tcgen05) */
  int activation; /* MLP only */
  int task;       /* MLP only; LLaMA is next-token cross-entropy */
  size_t input_dim, hidden_dim, model_dim, output_dim; /* model.hpp:33-36; LLaMA: hidden = ffn width,
                                                          input = output = vocab */
  size_t num_layers, num_stages;
  size_t n_heads;                 /* LLaMA only (head_dim = model_dim / n_heads) */
  size_t seq_len;                 /* LLaMA only */
  const size_t* partition;        /* 2*num_stages 1-based (first,last); NULL = even_partition */
  size_t max_rows;                /* rows (MLP) or tokens (LLaMA) per microbatch */
  int device;                     /* CUDA ordinal */
} ckf_model_desc;

int ckf_engine_create(const ckf_model_desc* desc, ckf_engine_t* out);
int ckf_engine_destroy(ckf_engine_t e);
/* parameters of one stage (canonical flat layout, model.cpp:117-125) / of an edge (0 embed, 1 de-embed) */
int ckf_engine_param_counts(ckf_engine_t e, size_t* stage_params, size_t* embed_params, size_t* deembed_params);

/* init_model(spec, seed, lr) (model.cpp:174-197): counter-RNG Glorot streams, bit-exact in fp64 */
int ckf_engine_init(ckf_engine_t e, uint64_t seed, double lr);

/* multi-GPU placement: stage_rank[s-1] = rank owning stage s; the embedding is
 * co-located with stage 1, the de-embedding with stage s (cost_model.cpp:264-268).
 * uid is a ckf_nccl_unique_id blob shared by all ranks (e.g. via torch.distributed). */
int ckf_nccl_unique_id(void* uid_out, size_t cap);
int ckf_engine_attach_comm(ckf_engine_t e, const void* uid, int nranks, int rank, const int* stage_rank);
/* Placement only (no NCCL communicator): which rank owns which stage; the buffers of stages
 * this rank does not own are released.  attach_comm = placement + NCCL.  Used on its own when
 * only the peer-recovery path is exercised (ranks sharing one GPU through CUDA IPC). */
int ckf_engine_set_placement(ckf_engine_t e, int nranks, int rank, const int* stage_rank, int replicas);
/* Peer recovery over NVLink: CUDA IPC handles of this rank's stage buffers (w, m, v of every
 * owned stage) as an opaque blob; every rank imports the other ranks' blobs and maps the
 * stages it does not own, so recover_stage reads a failed stage's neighbours directly from
 * the peers' HBM inside the recovery kernel (no staging copy).  *len = bytes written. */
int ckf_engine_ipc_export(ckf_engine_t e, void* buf, size_t cap, size_t* len);
int ckf_engine_ipc_import(ckf_engine_t e, const void* buf, size_t len);
/* Collective over the attached communicator: all-gathers every rank's IPC blob and imports
 * them (ckf_engine_ipc_export / _import in one call). */
int ckf_engine_exchange_peers(ckf_engine_t e);
/* Peer-memory stage transport (no NCCL on the data path): allocates this rank's mailbox of
 * 2 x max_microbatches buffers (residual stream / gradient of one microbatch, fp32) and flags;
 * call on every rank BEFORE the IPC exchange (ckf_engine_exchange_peers, or ipc_export /
 * ipc_import).  1F1B transfers then copy straight into the receiver's mailbox over
 * NVLink (copy engine) and signal it through a flag in its HBM (release / acquire, system
 * scope) that its recv stream waits on. */
int ckf_engine_enable_peer_transport(ckf_engine_t e, int max_microbatches);
/* the per-stage forward costs and head cost the engine's 1F1B plan is simulated with */
int ckf_engine_plan_cost(ckf_engine_t e, double* stage_cost, double* head_cost);
/* pipeline x data parallel (config 4: 4 stages x DP2): nranks = replicas * P; rank r is
 * pipeline rank r % P of replica r / P; stage_rank[] names PIPELINE ranks (0..P-1).  Each
 * replica runs its own microbatches; owned gradients are summed over the replicas
 * (ncclAllReduce on an ncclCommSplit group) before Adam, which divides by m * replicas. */
int ckf_engine_attach_comm_dp(ckf_engine_t e, const void* uid, int nranks, int rank, const int* stage_rank,
                              int replicas);

/* One training iteration (pipeline.cpp:58-95).  orders: m*s stage ids, one
 * execution order per microbatch (ExecutionOrder, pipeline.hpp:12-24).
 * MLP: x = rows x input_dim, y = rows x output_dim (regression) or rows labels (as
 *      double, classification), fp64.
 * LLaMA: x = rows x (seq_len+1) int32 token ids (inputs are [:, :T], labels [:, 1:]).
 * on_device: 1 if x/y are device pointers.  loss: mean loss; omegas: s values
 * (only owned stages are meaningful under multi-GPU). */
int ckf_engine_run_iteration(ckf_engine_t e, const int* orders, int m, const void* x, const void* y,
                             size_t rows, int on_device, long iteration, double* loss, double* omegas);
/* loss of forward(model, order, x) against y (model.cpp:279-282,380-382), no update */
int ckf_engine_eval_loss(ckf_engine_t e, const int* order, const void* x, const void* y, size_t rows,
                         int on_device, double* loss);
/* one microbatch forward + backward along `order`, ACCUMULATING into the gradient
 * buffers without an optimizer step (Gradients::accumulate, model.cpp:299-305);
 * *loss = the microbatch loss.  With ckf_engine_zero_grad / ckf_engine_export_grad
 * this is the gradient-parity seam (tests/test_model.cpp:109-155 style checks). */
int ckf_engine_accumulate(ckf_engine_t e, const int* order, const void* x, const void* y, size_t rows, int on_device,
                          double* loss);
int ckf_engine_zero_grad(ckf_engine_t e);
/* which: 0 embedding, 1 de-embedding, 2 stage `stage`; canonical flat layout, fp64 */
int ckf_engine_export_grad(ckf_engine_t e, int which, int stage, double* g);
/* predictions of forward(model, order, x) into host fp64 (MLP only) */
int ckf_engine_predict(ckf_engine_t e, const int* order, const double* x, size_t rows, double* pred);

/* CheckFree+ edge replicas (recovery.cpp:80-88): copy E, E^-1 to the neighbours' buffers */
int ckf_engine_refresh_edge_replicas(ckf_engine_t e);
/* whole-stage loss: NaN-poisons the stage's weights and moments on its GPU */
int ckf_engine_kill_stage(ckf_engine_t e, int stage);

enum ckf_recovery_mode {
  CKF_REC_CHECKFREE = 0, /* omega-weighted neighbour average (recovery.cpp:57-73) */
  CKF_REC_UNIFORM = 1,   /* reinit_uniform_avg (recovery.cpp:105-110) */
  CKF_REC_COPY_PREV = 2, /* reinit_copy (recovery.cpp:103) */
  CKF_REC_RANDOM = 3,    /* reinit_random (recovery.cpp:112-118) */
  CKF_REC_EDGE = 4       /* CheckFree+ first/last stage: neighbour copy + replica (recovery.cpp:90-101) */
};
enum ckf_moments { CKF_MOM_FRESH = 0, CKF_MOM_AVERAGED = 1 }; /* recovery.hpp:31 */

typedef struct {
  int degenerate;          /* both neighbour omegas were zero -> uniform average */
  double reduction_error;  /* ||W_before - W_after||^2 (trainer.cpp:278-279), if requested */
  double latency_ms;       /* CUDA-event time from issue to the stage being ready */
} ckf_recovery_report;

/* Rebuilds `stage` per the trainer's semantics (trainer.cpp:199-276): weights,
 * moments (Fresh reset / Averaged), lr *= lr_bump, omega := 0, and for
 * CKF_REC_EDGE the edge layer from the fresh replica with its Adam state reset.
 * Neighbour weights are read peer-to-peer when they live on another GPU. */
int ckf_engine_recover_stage(ckf_engine_t e, int stage, int mode, int moments, double lr_bump,
                             uint64_t reinit_seed, int want_reduction_error, ckf_recovery_report* out);

/* state exchange in the canonical fp64 flat layout (model.cpp:117-157) */
int ckf_engine_export_stage(ckf_engine_t e, int stage, double* w, double* m, double* v);
int ckf_engine_import_stage(ckf_engine_t e, int stage, const double* w, const double* m, const double* v);
int ckf_engine_export_edge(ckf_engine_t e, int which, double* w, double* m, double* v);
int ckf_engine_import_edge(ckf_engine_t e, int which, const double* w, const double* m, const double* v);
int ckf_engine_get_scalars(ckf_engine_t e, int stage, double* omega, double* lr, long* step);
int ckf_engine_set_scalars(ckf_engine_t e, int stage, double omega, double lr, long step);
int ckf_engine_get_edge_scalars(ckf_engine_t e, double* lr, long* step_embed, long* step_deembed);
int ckf_engine_set_edge_scalars(ckf_engine_t e, double lr, long step_embed, long step_deembed);

/* iteration schedule: 0 = sequential (default on one GPU), 1 = GPipe (default once attached to >1 rank) */
int ckf_engine_set_schedule(ckf_engine_t e, int mode);
/* microbatch fusion when every stage is resident on this rank: microbatches sharing an
 * execution order run as one forward+backward of up to `cap` microbatches (same
 * arithmetic as pipeline.cpp:66-83; 0 = as many as HBM allows (default), 1 = off) */
int ckf_engine_set_group_cap(ckf_engine_t e, int cap);
/* device time of the last ckf_engine_run_iteration, CUDA events on the engine stream from its
 * first device operation (the input H2D copy when the batch is on the host) to the loss /
 * omega D2H copies -- host scheduling after the step is excluded */
int ckf_engine_last_step_ms(ckf_engine_t e, float* ms);
/* redundant-computation baseline (trainer.cpp:162-171), measured instead of modelled
 * (cost_model.cpp:242-279): per microbatch one extra forward of every stage's layers (the
 * downstream node's hot copy) and, after the optimizer step, a copy of every stage's master
 * weights to its replica.  LLaMA bf16 block. */
int ckf_engine_set_redundant(ckf_engine_t e, int on);
/* CheckFree+ per-step edge replica refresh inside the step (trainer.cpp:83-84): when on,
 * ckf_engine_run_iteration ends with the replica copy of E / E^-1 (to the GPUs of stages 2 and
 * s-1), inside the step's device bracket (ckf_engine_last_step_ms). */
int ckf_engine_set_edge_replicas(ckf_engine_t e, int on);
/* Hop log for a VIRTUAL placement (stage -> rank), used to check on one GPU that
 * the engine's stage transfers match ckf_pipeline_plan: when enabled, every
 * cross-rank transfer the placement implies is recorded as (src, dst, bytes). */
int ckf_engine_hop_log(ckf_engine_t e, int nranks, const int* stage_rank);
int ckf_engine_get_hop_log(ckf_engine_t e, long* out, int cap_triples, int* n_triples);

/* launches of the engine's own kernels since creation (evidence for gpu_launches) */
long ckf_engine_kernel_launches(ckf_engine_t e);
/* synchronises the engine's streams */
int ckf_engine_sync(ckf_engine_t e);
/* the cudaStream_t the engine launches its kernels on (for CUDA-event timing by the caller) */
int ckf_engine_stream(ckf_engine_t e, void** stream);

/* Per-class kernel timing (roofline evidence).  enable != 0 resets the stats
 * and brackets every tagged launch with CUDA events on the engine stream.
 * cls: 0 GEMM, 1 attention, 2 Adam+omega, 3 recovery, 4 norm/elementwise,
 * 5 loss, 6 stage transfer.  ms = summed device time; flops / bytes = the
 * launches' ALGORITHMIC work (2MNK per GEMM, compulsory bytes otherwise). */
int ckf_engine_kernel_timing(ckf_engine_t e, int enable);
int ckf_engine_kernel_stats(ckf_engine_t e, int cls, double* ms, long* launches, double* flops, double* bytes);

/* =====================================================================
 * (4) Trainer: harness::run_experiment (src/trainer.cpp:314-322) on the
 *     engine.  kv_config: "key=value;..." with the keys of
 *     ExperimentConfig::to_config_string (src/experiment.cpp:117-154) plus
 *     block/precision/heads/seq-len/vocab for LLaMA.  trace_text: a
 *     "checkfree-trace v1" file (failures.cpp:84-95); empty = generate from
 *     the config (experiment.cpp:102-115).  record: E/F/U lines
 *     ("E,iter,train,val", "F,iter,stage,action,reduction_error,loss_spike,recovery_ms",
 *     "U,reason").
 * ===================================================================== */
int ckf_run_experiment(const char* kv_config, const char* trace_text, uint64_t seed, char* record, size_t cap);
/* The same trainer as ONE rank of a multi-GPU run (one process per GPU): stages placed in
 * contiguous blocks over nranks / replicas pipeline ranks (edges with stages 1 and s),
 * `replicas` data-parallel copies (replica r trains on microbatches [r m/R, (r+1) m/R) of the
 * global batch), stage transfers 1F1B over NCCL, recovery reading the neighbours from the
 * peers' HBM.  Every rank calls it with the same arguments and the NCCL unique id of rank 0
 * (ckf_nccl_unique_id); every rank returns the same record. */
int ckf_run_experiment_rank(const char* kv_config, const char* trace_text, uint64_t seed, const void* nccl_uid,
                            int nranks, int rank, int replicas, char* record, size_t cap);
/* run_experiment_to_dir (src/experiment.cpp:202-213): the same run, writing
 * metrics.csv, events.csv, summary.json and config.resolved in the reference's
 * schema (format_version=1) into dir; wall_hours / recovery_s are measured. */
int ckf_run_experiment_to_dir(const char* kv_config, const char* trace_text, uint64_t seed, const char* dir);

#ifdef __cplusplus
}
#endif
#endif /* CKF_H_ */
