#include <type_traits>
// extern "C" entry points of include/ckf.h.  Nothing throws across this line:
// every call maps internal errors to CKF_E_* codes + ckf_last_error().
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ckf.h"
#include "engine.h"
#include "gemm_tc.h"
#include "host_logic.h"
#include "llama_kernels.h"

namespace ckf {
void llama_token_batch(uint64_t data_seed, uint64_t stream, uint64_t index, size_t rows, size_t T, size_t V, int* out,
                       cudaStream_t s);
int nccl_unique_id(void* out, size_t cap);
}  // namespace ckf

namespace {

thread_local std::string g_err;
thread_local long g_err_iter = -1;

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    g_err_iter = -1;
    return CKF_OK;
  } catch (const ckf::Error& e) {
    g_err = e.what();
    g_err_iter = e.iteration;
    return e.code;
  } catch (const ckf::host::HostError& e) {
    g_err = e.what();
    g_err_iter = -1;
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return CKF_E_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CKF_E_CONFIG;
  }
}

// ---------------------------------------------------------------- L1 seam context
// Host-pointer kernels stage through one device arena on a private stream.
struct Seam {
  std::mutex mu;
  cudaStream_t st = nullptr;
  void* arena = nullptr;
  size_t cap = 0;
  ckf::ReduceScratch red;
  double* scal = nullptr;
  int device = -1;

  void ensure() {
    int dev = 0;
    CKF_CUDA(cudaGetDevice(&dev));
    if (dev != device) {
      device = dev;
      CKF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      CKF_CUDA(cudaMalloc(&red.partials, ckf::ReduceScratch::kMaxReduceBlocks * sizeof(double)));
      CKF_CUDA(cudaMalloc(&scal, 64 * sizeof(double)));
      arena = nullptr;
      cap = 0;
    }
  }
  // returns n_bufs device pointers carved from the arena (each 256-B aligned)
  std::vector<double*> bufs(std::initializer_list<size_t> elems) {
    size_t total = 0;
    for (size_t e : elems) total += (e * sizeof(double) + 255) / 256 * 256;
    if (total > cap) {
      if (arena) CKF_CUDA(cudaFree(arena));
      CKF_CUDA(cudaMalloc(&arena, total));
      cap = total;
    }
    std::vector<double*> out;
    char* p = static_cast<char*>(arena);
    for (size_t e : elems) {
      out.push_back(reinterpret_cast<double*>(p));
      p += (e * sizeof(double) + 255) / 256 * 256;
    }
    return out;
  }
  void h2d(double* d, const double* h, size_t n) {
    if (n) CKF_CUDA(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  void d2h(double* h, const double* d, size_t n) {
    if (n) CKF_CUDA(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  void sync() { CKF_CUDA(cudaStreamSynchronize(st)); }
};
Seam& seam() {
  static Seam s;
  return s;
}

int seam_gemm(bool ta, bool tb, bool acc, const double* a, const double* b, double* c, size_t m, size_t k, size_t n) {
  return guard([&] {
    Seam& S = seam();
    std::lock_guard<std::mutex> lk(S.mu);
    S.ensure();
    auto d = S.bufs({m * k, k * n, m * n});
    S.h2d(d[0], a, m * k);
    S.h2d(d[1], b, k * n);
    if (acc) S.h2d(d[2], c, m * n);
    const size_t lda = ta ? m : k, ldb = tb ? k : n;
    ckf::k::gemm_simt<double>(ta, tb, m, n, k, d[0], lda, d[1], ldb, d[2], n, acc, S.st);
    S.d2h(c, d[2], m * n);
    S.sync();
  });
}

ckf::Engine* E(ckf_engine_t e) { return reinterpret_cast<ckf::Engine*>(e); }

}  // namespace

extern "C" {

const char* ckf_last_error(void) { return g_err.c_str(); }
long ckf_last_error_iteration(void) { return g_err_iter; }
int ckf_version(void) { return 1; }
int ckf_device_count(int* out) {
  return guard([&] { CKF_CUDA(cudaGetDeviceCount(out)); });
}

// ---------------------------------------------------------------- (0) host logic
int ckf_generate_trace(uint64_t seed, double p_hour, double iter_s, long n_iters, const int* stages, int n_stages,
                       char* out, size_t cap) {
  return guard([&] {
    auto t = ckf::host::generate_trace(seed, p_hour, iter_s, n_iters, std::vector<int>(stages, stages + n_stages));
    const std::string s = ckf::host::serialize_trace(t);
    if (s.size() + 1 > cap) ckf::raise(CKF_E_USAGE, "output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}
int ckf_parse_trace(const char* text, char* out, size_t cap) {
  return guard([&] {
    const std::string s = ckf::host::serialize_trace(ckf::host::parse_trace(text ? text : ""));
    if (s.size() + 1 > cap) ckf::raise(CKF_E_USAGE, "output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}
int ckf_pipeline_plan_cost(int s, int m, const int* orders, const int* stage_rank, int schedule,
                           const double* stage_cost, double head_cost, int* out, int cap_ops, int* n_ops) {
  return guard([&] {
    if (s < 1 || m < 1) ckf::raise(CKF_E_CONFIG, "pipeline plan needs s >= 1 and m >= 1");
    ckf::host::PlanCost cost;
    if (stage_cost) cost.stage.assign(stage_cost, stage_cost + s);
    cost.head = head_cost;
    const auto ops = ckf::host::pipeline_plan(
        s, m, std::vector<int>(orders, orders + static_cast<size_t>(s) * static_cast<size_t>(m)),
        std::vector<int>(stage_rank, stage_rank + s), schedule, &cost);
    if (static_cast<int>(ops.size()) > cap_ops) ckf::raise(CKF_E_USAGE, "output buffer too small");
    for (size_t i = 0; i < ops.size(); ++i) {
      int* o = out + 6 * i;
      o[0] = ops[i].phase;
      o[1] = ops[i].mb;
      o[2] = ops[i].kind;
      o[3] = ops[i].rank;
      o[4] = ops[i].arg;
      o[5] = ops[i].aux;
    }
    *n_ops = static_cast<int>(ops.size());
  });
}
int ckf_pipeline_plan(int s, int m, const int* orders, const int* stage_rank, int schedule, int* out, int cap_ops,
                      int* n_ops) {
  return ckf_pipeline_plan_cost(s, m, orders, stage_rank, schedule, nullptr, 1.0, out, cap_ops, n_ops);
}
int ckf_consecutive_conflicts(const char* text, long* out, int cap_pairs, int* n_out) {
  return guard([&] {
    auto c = ckf::host::consecutive_conflicts(ckf::host::parse_trace(text ? text : ""));
    if (static_cast<int>(c.size()) > cap_pairs) ckf::raise(CKF_E_USAGE, "output buffer too small");
    for (size_t i = 0; i < c.size(); ++i) {
      out[2 * i] = c[i].iteration;
      out[2 * i + 1] = c[i].stage;
    }
    *n_out = static_cast<int>(c.size());
  });
}
double ckf_hourly_to_per_iteration(double p_hour, double iter_s) {
  double r = NAN;
  guard([&] { r = ckf::host::hourly_to_per_iteration(p_hour, iter_s); });
  return r;
}
int ckf_even_partition(size_t layers, size_t stages, size_t* out) {
  return guard([&] {
    if (stages < 1 || stages > layers) ckf::raise(CKF_E_CONFIG, "num_stages must lie in [1, num_layers]");
    auto p = ckf::even_partition(layers, stages);
    for (size_t i = 0; i < p.size(); ++i) {
      out[2 * i] = p[i].first;
      out[2 * i + 1] = p[i].last;
    }
  });
}
int ckf_build_schedule(int m, int swapped_half, int s, int* out) {
  return guard([&] {
    auto o = ckf::host::build_schedule(m, swapped_half != 0, s);
    std::memcpy(out, o.data(), o.size() * sizeof(int));
  });
}

// ---------------------------------------------------------------- (1) L1 seam
int ckf_k_gemm_nn(const double* a, const double* b, double* c, size_t m, size_t k, size_t n) {
  return seam_gemm(false, false, false, a, b, c, m, k, n);
}
int ckf_k_gemm_nn_acc(const double* a, const double* b, double* c, size_t m, size_t k, size_t n) {
  return seam_gemm(false, false, true, a, b, c, m, k, n);
}
int ckf_k_gemm_nt_acc(const double* a, const double* b, double* c, size_t m, size_t k, size_t n) {
  return seam_gemm(false, true, true, a, b, c, m, k, n);
}
int ckf_k_gemm_tn_acc(const double* a, const double* b, double* c, size_t m, size_t k, size_t n) {
  return seam_gemm(true, false, true, a, b, c, m, k, n);
}

#define SEAM_BEGIN            \
  return guard([&] {          \
    Seam& S = seam();         \
    std::lock_guard<std::mutex> lk(S.mu); \
    S.ensure();
#define SEAM_END \
  S.sync();      \
  });

int ckf_k_add_inplace(double* x, const double* y, size_t n) {
  SEAM_BEGIN
  auto d = S.bufs({n, n});
  S.h2d(d[0], x, n);
  S.h2d(d[1], y, n);
  ckf::k::add_inplace(d[0], d[1], n, S.st);
  S.d2h(x, d[0], n);
  SEAM_END
}
int ckf_k_axpy(double alpha, const double* x, double* y, size_t n) {
  SEAM_BEGIN
  auto d = S.bufs({n, n});
  S.h2d(d[0], x, n);
  S.h2d(d[1], y, n);
  ckf::k::axpy(alpha, d[0], d[1], n, S.st);
  S.d2h(y, d[1], n);
  SEAM_END
}
int ckf_k_scale(double alpha, double* x, size_t n) {
  SEAM_BEGIN
  auto d = S.bufs({n});
  S.h2d(d[0], x, n);
  ckf::k::scale(alpha, d[0], n, S.st);
  S.d2h(x, d[0], n);
  SEAM_END
}
int ckf_k_apply_activation(int act, const double* a, double* z, size_t n) {
  SEAM_BEGIN
  auto d = S.bufs({n, n});
  S.h2d(d[0], a, n);
  ckf::k::act_fwd(act, d[0], d[1], n, S.st);
  S.d2h(z, d[1], n);
  SEAM_END
}
int ckf_k_activation_backward(int act, const double* z, const double* dz, double* da, size_t n) {
  SEAM_BEGIN
  auto d = S.bufs({n, n, n});
  S.h2d(d[0], z, n);
  S.h2d(d[1], dz, n);
  ckf::k::act_bwd(act, d[0], d[1], d[2], n, S.st);
  S.d2h(da, d[2], n);
  SEAM_END
}
int ckf_k_sum_squares(const double* x, size_t n, double* out) {
  SEAM_BEGIN
  auto d = S.bufs({n});
  S.h2d(d[0], x, n);
  ckf::k::sum_squares(d[0], n, S.scal, S.red, S.st);
  S.d2h(out, S.scal, 1);
  SEAM_END
}
int ckf_k_sum_squared_diff(const double* x, const double* y, size_t n, double* out) {
  SEAM_BEGIN
  auto d = S.bufs({n, n});
  S.h2d(d[0], x, n);
  S.h2d(d[1], y, n);
  ckf::k::sum_sq_diff(d[0], d[1], n, S.scal, S.red, S.st);
  S.d2h(out, S.scal, 1);
  SEAM_END
}
int ckf_k_adam_update(double* w, double* m, double* v, const double* g, size_t n, double lr, double beta1,
                      double beta2, double eps, long step) {
  if (beta1 != 0.9 || beta2 != 0.999 || eps != 1e-8) {
    g_err = "the fused Adam kernel is specialised for betas (0.9, 0.999), eps 1e-8 (model.hpp:72-74)";
    return CKF_E_CONFIG;
  }
  SEAM_BEGIN
  auto d = S.bufs({n, n, n, n});
  S.h2d(d[0], w, n);
  S.h2d(d[1], m, n);
  S.h2d(d[2], v, n);
  S.h2d(d[3], g, n);
  const double bc1 = 1.0 - std::pow(beta1, static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(beta2, static_cast<double>(step));
  ckf::k::adam<double>(d[0], d[1], d[2], d[3], nullptr, n, lr, bc1, bc2, 1.0, false, S.scal, S.red, S.st);
  S.d2h(w, d[0], n);
  S.d2h(m, d[1], n);
  S.d2h(v, d[2], n);
  SEAM_END
}
int ckf_k_mse_loss_grad(const double* pred, const double* target, size_t rows, size_t cols, double* dpred,
                        double* loss) {
  SEAM_BEGIN
  const size_t n = rows * cols;
  auto d = S.bufs({n, n, n});
  S.h2d(d[0], pred, n);
  S.h2d(d[1], target, n);
  ckf::k::mse_loss_grad(d[0], d[1], rows, cols, dpred ? d[2] : nullptr, S.scal, S.red, S.st);
  if (dpred) S.d2h(dpred, d[2], n);
  S.d2h(loss, S.scal, 1);
  SEAM_END
}
int ckf_k_softmax_xent_loss_grad(const double* logits, const int* labels, size_t rows, size_t cols, double* dlogits,
                                 double* loss) {
  SEAM_BEGIN
  const size_t n = rows * cols;
  auto d = S.bufs({n, n, (rows + 1) / 2});
  S.h2d(d[0], logits, n);
  CKF_CUDA(cudaMemcpyAsync(d[2], labels, rows * sizeof(int), cudaMemcpyHostToDevice, S.st));
  ckf::k::xent_loss_grad(d[0], reinterpret_cast<const int*>(d[2]), rows, cols, dlogits ? d[1] : nullptr, S.scal,
                         S.red, S.st);
  if (dlogits) S.d2h(dlogits, d[1], n);
  S.d2h(loss, S.scal, 1);
  SEAM_END
}
int ckf_k_recover_checkfree(const double* w_prev, const double* w_next, size_t n, double op, double on, double* out,
                            int* degenerate) {
  if (op < 0.0 || on < 0.0) {
    g_err = "gradient norms must be nonnegative";
    return CKF_E_CONFIG;
  }
  SEAM_BEGIN
  auto d = S.bufs({n, n, n});
  S.h2d(d[0], w_prev, n);
  S.h2d(d[1], w_next, n);
  ckf::k::recover<double>(d[0], d[1], d[2], n, op, on, nullptr, S.red, S.st);
  S.d2h(out, d[2], n);
  if (degenerate) *degenerate = op + on == 0.0 ? 1 : 0;
  SEAM_END
}
int ckf_k_counter_uniform(uint64_t key, double lo, double hi, double* out, size_t n) {
  SEAM_BEGIN
  auto d = S.bufs({n});
  ckf::k::uniform<double>(d[0], n, key, lo, hi, 0, S.st);
  S.d2h(out, d[0], n);
  SEAM_END
}

// ---------------------------------------------------------------- (2) device primitives
int ckf_recover_device(int dtype, const void* wp, const void* wn, void* out, size_t n, double op, double on,
                       double* old_out_sq, void* stream) {
  return guard([&] {
    if (op < 0.0 || on < 0.0) ckf::raise(CKF_E_CONFIG, "gradient norms must be nonnegative");
    static thread_local ckf::ReduceScratch red;
    if (!red.partials) CKF_CUDA(cudaMalloc(&red.partials, ckf::ReduceScratch::kMaxReduceBlocks * sizeof(double)));
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype == CKF_FP64)
      ckf::k::recover(static_cast<const double*>(wp), static_cast<const double*>(wn), static_cast<double*>(out), n, op,
                      on, old_out_sq, red, st);
    else if (dtype == CKF_FP32)
      ckf::k::recover(static_cast<const float*>(wp), static_cast<const float*>(wn), static_cast<float*>(out), n, op, on,
                      old_out_sq, red, st);
    else
      ckf::raise(CKF_E_CONFIG, "recover: dtype must be CKF_FP64 or CKF_FP32 (master weights)");
  });
}

int ckf_recover_stage_device(int dtype, const void* wp, const void* wn, const void* mp, const void* mn,
                             const void* vp, const void* vn, void* w, void* m, void* v, void* g, void* w_bf16,
                             size_t n, double omega_prev, double omega_next, int averaged, double* old_sq,
                             void* stream) {
  return guard([&] {
    if (omega_prev < 0.0 || omega_next < 0.0) ckf::raise(CKF_E_CONFIG, "gradient norms must be nonnegative");
    if (averaged && (!mp || !mn || !vp || !vn)) ckf::raise(CKF_E_CONFIG, "averaged moments need mp, mn, vp, vn");
    static thread_local ckf::ReduceScratch red;
    if (!red.partials) CKF_CUDA(cudaMalloc(&red.partials, ckf::ReduceScratch::kMaxReduceBlocks * sizeof(double)));
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      ckf::k::StageRecovery<T> r;
      r.wp = static_cast<const T*>(wp);
      r.wn = static_cast<const T*>(wn);
      r.mp = static_cast<const T*>(mp);
      r.mn = static_cast<const T*>(mn);
      r.vp = static_cast<const T*>(vp);
      r.vn = static_cast<const T*>(vn);
      r.w = static_cast<T*>(w);
      r.m = static_cast<T*>(m);
      r.v = static_cast<T*>(v);
      r.g = static_cast<T*>(g);
      r.wlp = static_cast<__nv_bfloat16*>(w_bf16);
      r.n = n;
      r.op = omega_prev;
      r.on = omega_next;
      r.averaged = averaged != 0;
      r.mop = omega_prev;
      r.mon = omega_next;
      r.old_sq = old_sq;
      ckf::k::recover_stage(r, red, static_cast<cudaStream_t>(stream));
    };
    if (dtype == CKF_FP64) {
      if (w_bf16) ckf::raise(CKF_E_CONFIG, "the fp64 parity precision keeps no bf16 shadow");
      run(static_cast<double*>(nullptr));
    } else if (dtype == CKF_FP32) {
      run(static_cast<float*>(nullptr));
    } else {
      ckf::raise(CKF_E_CONFIG, "recover_stage: dtype must be CKF_FP64 or CKF_FP32 (master weights)");
    }
  });
}

int ckf_adam_device(int dtype, void* w, void* m, void* v, void* g, void* w_bf16, size_t n, double lr, double bc1,
                    double bc2, double grad_scale, int zero_grad, double* omega, void* stream) {
  return guard([&] {
    static thread_local ckf::ReduceScratch red;
    if (!red.partials) CKF_CUDA(cudaMalloc(&red.partials, ckf::ReduceScratch::kMaxReduceBlocks * sizeof(double)));
    auto st = static_cast<cudaStream_t>(stream);
    auto lp = static_cast<__nv_bfloat16*>(w_bf16);
    if (dtype == CKF_FP64)
      ckf::k::adam(static_cast<double*>(w), static_cast<double*>(m), static_cast<double*>(v), static_cast<double*>(g),
                   lp, n, lr, bc1, bc2, grad_scale, zero_grad != 0, omega, red, st);
    else if (dtype == CKF_FP32)
      ckf::k::adam(static_cast<float*>(w), static_cast<float*>(m), static_cast<float*>(v), static_cast<float*>(g), lp,
                   n, lr, bc1, bc2, grad_scale, zero_grad != 0, omega, red, st);
    else
      ckf::raise(CKF_E_CONFIG, "adam: dtype must be CKF_FP64 or CKF_FP32 (master weights)");
  });
}

int ckf_gemm_bf16(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
                  int ldc, int epi, float alpha, int bn, void* stream) {
  if (epi > 2) return guard([&] { ckf::raise(CKF_E_CONFIG, "gemm_bf16: epi must be 0, 1 or 2 (3/4: ckf_gemm_bf16_aux)"); });
  return ckf_gemm_bf16_aux(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc, epi, alpha, bn, nullptr, 0, stream);
}

int ckf_xent_bf16(void* logits, const int* labels, size_t rows, size_t V, float grad_scale, int grad, double* row_loss,
                  void* stream) {
  return guard([&] {
    ckf::llama::xent_bf16(static_cast<__nv_bfloat16*>(logits), labels, rows, V, grad_scale, grad, row_loss,
                          static_cast<cudaStream_t>(stream));
  });
}

size_t ckf_lm_head_xent_workspace(size_t M, size_t d, size_t V) { return ckf::llama::head_xent_workspace(M, d, V); }

int ckf_lm_head_xent(const void* xn, const void* Einv, const int* labels, size_t M, size_t d, size_t V, float grad_scale,
                     int train, double* row_loss, float* dxn, float* gEinv, const float* h, const float* rstd,
                     const float* gain, void* ws, void* stream) {
  const float* hrows = h;
  return guard([&] {
    ckf::llama::HeadXent h;
    h.xn = static_cast<const __nv_bfloat16*>(xn);
    h.Einv = static_cast<const __nv_bfloat16*>(Einv);
    h.labels = labels;
    h.M = static_cast<int>(M);
    h.d = static_cast<int>(d);
    h.V = static_cast<int>(V);
    h.grad_scale = grad_scale;
    h.train = train != 0;
    h.row_loss = row_loss;
    h.dxn = dxn;
    h.gEinv = gEinv;
    h.ws = ws;
    h.h = hrows;
    h.rstd = rstd;
    h.gain = gain;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    ckf::llama::head_xent(h, [&](const ckf::tc::GemmDesc& g) { ckf::tc::gemm_bf16(g, st); },
                          [](const std::function<void()>& f) { f(); }, st);
  });
}

int ckf_gemm_bf16_aux(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
                      int ldc, int epi, float alpha, int bn, void* aux, int ldaux, void* stream) {
  return guard([&] {
    if (epi < 0 || epi > 4) ckf::raise(CKF_E_CONFIG, "gemm_bf16: epi must be 0..4");
    if ((epi == 3 && (a_mn || !b_mn)) || (epi == 4 && (a_mn || b_mn)))
      ckf::raise(CKF_E_CONFIG, "gemm_bf16: SwiGLU epilogues take A K-major and B MN-major (3) / K-major (4)");
    if (bn != 0 && bn != 128 && bn != 256) ckf::raise(CKF_E_CONFIG, "gemm_bf16: bn must be 0, 128 or 256");
    ckf::tc::GemmDesc g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = static_cast<const __nv_bfloat16*>(A);
    g.lda = lda;
    g.a_mn = a_mn != 0;
    g.B = static_cast<const __nv_bfloat16*>(B);
    g.ldb = ldb;
    g.b_mn = b_mn != 0;
    g.C = C;
    g.ldc = ldc;
    g.epi = epi;
    g.alpha = alpha;
    g.bn = bn;
    g.aux = aux;
    g.ldaux = ldaux;
    ckf::tc::gemm_bf16(g, static_cast<cudaStream_t>(stream));
  });
}

int ckf_attention_fwd(const void* qkv, size_t B, size_t T, size_t H, size_t hd, void* o, float* lse, int impl,
                      void* stream) {
  return guard([&] {
    auto st = static_cast<cudaStream_t>(stream);
    const auto* q = static_cast<const __nv_bfloat16*>(qkv);
    auto* out = static_cast<__nv_bfloat16*>(o);
    const bool tc = impl == 2 || (impl == 0 && ckf::llama::attn_fwd_tc_supported(T, hd));
    if (tc)
      ckf::llama::attn_fwd_tc(q, B, T, H, hd, out, lse, st);
    else
      ckf::llama::attn_fwd(q, B, T, H, hd, out, lse, st);
  });
}
int ckf_attention_bwd(const void* qkv, const void* o, const float* lse, const void* dout, size_t B, size_t T,
                      size_t H, size_t hd, void* dqkv, float* Dsum, int impl, void* stream) {
  return guard([&] {
    const bool rope = (impl & CKF_ATTN_ROPE_BWD) != 0;
    impl &= ~CKF_ATTN_ROPE_BWD;
    const bool tc = impl == 2 || (impl == 0 && ckf::llama::attn_fwd_tc_supported(T, hd));
    if (tc) {
      ckf::llama::attn_bwd_tc(static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(o), lse,
                              static_cast<const __nv_bfloat16*>(dout), B, T, H, hd, static_cast<__nv_bfloat16*>(dqkv),
                              Dsum, static_cast<cudaStream_t>(stream), rope);
      return;
    }
    ckf::llama::attn_bwd(static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(o), lse,
                         static_cast<const __nv_bfloat16*>(dout), B, T, H, hd, static_cast<__nv_bfloat16*>(dqkv), Dsum,
                         static_cast<cudaStream_t>(stream));
    if (rope) ckf::llama::rope(static_cast<__nv_bfloat16*>(dqkv), B * T, T, H * hd, H, 1, static_cast<cudaStream_t>(stream));
  });
}
// debug (not part of the ABI contract): per-CTA forward-attention timings, 8 longs per CTA
int ckf_debug_gemm_timings(long long* out, int n_ctas) {
  return guard([&] {
    long long* b = ckf::tc::gemm_debug_buffer();
    if (!b) ckf::raise(CKF_E_USAGE, "set CKF_GEMM_DEBUG=1");
    CKF_CUDA(cudaMemcpy(out, b, 8 * sizeof(long long) * static_cast<size_t>(n_ctas), cudaMemcpyDeviceToHost));
  });
}
int ckf_debug_attn_fwd_timings(long long* out, int n_ctas) {
  return guard([&] {
    long long* b = ckf::llama::attn_fwd_debug_buffer();
    if (!b) ckf::raise(CKF_E_USAGE, "set CKF_ATTN_DEBUG=1");
    CKF_CUDA(cudaMemcpy(out, b, 8 * sizeof(long long) * static_cast<size_t>(n_ctas), cudaMemcpyDeviceToHost));
  });
}
int ckf_llama_token_batch(uint64_t data_seed, uint64_t stream, uint64_t index, size_t rows, size_t T, size_t V,
                          int* out) {
  return guard([&] {
    if (V < 2 || V > (1ull << 31)) ckf::raise(CKF_E_CONFIG, "vocabulary size out of range");
    int* d = nullptr;
    const size_t n = rows * (T + 1);
    CKF_CUDA(cudaMalloc(&d, std::max<size_t>(n, 1) * sizeof(int)));
    ckf::llama_token_batch(data_seed, stream, index, rows, T, V, d, nullptr);
    const cudaError_t e = cudaMemcpy(out, d, n * sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d);
    CKF_CUDA(e);
  });
}

// ---------------------------------------------------------------- (3) engine
int ckf_engine_create(const ckf_model_desc* desc, ckf_engine_t* out) {
  return guard([&] {
    if (!desc || !out) ckf::raise(CKF_E_USAGE, "null argument");
    *out = reinterpret_cast<ckf_engine_t>(new ckf::Engine(*desc));
  });
}
int ckf_engine_destroy(ckf_engine_t e) {
  return guard([&] { delete E(e); });
}
int ckf_engine_param_counts(ckf_engine_t e, size_t* sp, size_t* ep, size_t* dp) {
  return guard([&] {
    if (sp) *sp = E(e)->stage(1).n;
    if (ep) *ep = E(e)->embed().n;
    if (dp) *dp = E(e)->deembed().n;
  });
}
int ckf_engine_init(ckf_engine_t e, uint64_t seed, double lr) {
  return guard([&] { E(e)->init(seed, lr); });
}
int ckf_nccl_unique_id(void* uid_out, size_t cap) {
  return guard([&] { ckf::nccl_unique_id(uid_out, cap); });
}
int ckf_engine_attach_comm(ckf_engine_t e, const void* uid, int nranks, int rank, const int* stage_rank) {
  return guard([&] { E(e)->attach_comm(uid, nranks, rank, stage_rank, 1); });
}
int ckf_engine_set_placement(ckf_engine_t e, int nranks, int rank, const int* stage_rank, int replicas) {
  return guard([&] { E(e)->set_placement(nranks, rank, stage_rank, replicas); });
}
int ckf_engine_ipc_export(ckf_engine_t e, void* buf, size_t cap, size_t* len) {
  return guard([&] { *len = E(e)->ipc_export(buf, cap); });
}
int ckf_engine_ipc_import(ckf_engine_t e, const void* buf, size_t len) {
  return guard([&] { E(e)->ipc_import(buf, len); });
}
int ckf_engine_exchange_peers(ckf_engine_t e) {
  return guard([&] { E(e)->exchange_peers(); });
}
int ckf_engine_enable_peer_transport(ckf_engine_t e, int max_microbatches) {
  return guard([&] { E(e)->enable_peer_transport(max_microbatches); });
}
int ckf_engine_plan_cost(ckf_engine_t e, double* stage_cost, double* head_cost) {
  return guard([&] {
    const auto c = E(e)->plan_cost();
    std::copy(c.stage.begin(), c.stage.end(), stage_cost);
    *head_cost = c.head;
  });
}
int ckf_engine_attach_comm_dp(ckf_engine_t e, const void* uid, int nranks, int rank, const int* stage_rank,
                              int replicas) {
  return guard([&] { E(e)->attach_comm(uid, nranks, rank, stage_rank, replicas); });
}
int ckf_engine_run_iteration(ckf_engine_t e, const int* orders, int m, const void* x, const void* y, size_t rows,
                             int on_device, long iteration, double* loss, double* omegas) {
  return guard([&] { E(e)->run_iteration(orders, m, x, y, rows, on_device != 0, iteration, loss, omegas); });
}
int ckf_engine_eval_loss(ckf_engine_t e, const int* order, const void* x, const void* y, size_t rows, int on_device,
                         double* loss) {
  return guard([&] { *loss = E(e)->eval_loss(order, x, y, rows, on_device != 0); });
}
int ckf_engine_accumulate(ckf_engine_t e, const int* order, const void* x, const void* y, size_t rows, int on_device,
                          double* loss) {
  return guard([&] {
    const double l = E(e)->accumulate(order, x, y, rows, on_device != 0);
    if (loss) *loss = l;
  });
}
int ckf_engine_zero_grad(ckf_engine_t e) {
  return guard([&] { E(e)->zero_grad(); });
}
int ckf_engine_export_grad(ckf_engine_t e, int which, int stage, double* g) {
  return guard([&] {
    ckf::Engine* en = E(e);
    if (which == 0)
      en->export_grad(en->embed(), g);
    else if (which == 1)
      en->export_grad(en->deembed(), g);
    else if (which == 2) {
      if (stage < 1 || static_cast<size_t>(stage) > en->desc().s) ckf::raise(CKF_E_CONFIG, "stage id out of range");
      en->export_grad(en->stage(stage), g);
    } else
      ckf::raise(CKF_E_CONFIG, "which must be 0 (embed), 1 (de-embed) or 2 (stage)");
  });
}
int ckf_engine_predict(ckf_engine_t e, const int* order, const double* x, size_t rows, double* pred) {
  return guard([&] { E(e)->predict(order, x, rows, pred); });
}
int ckf_engine_refresh_edge_replicas(ckf_engine_t e) {
  return guard([&] { E(e)->refresh_edge_replicas(); });
}
int ckf_engine_kill_stage(ckf_engine_t e, int stage) {
  return guard([&] { E(e)->kill_stage(stage); });
}
int ckf_engine_recover_stage(ckf_engine_t e, int stage, int mode, int moments, double lr_bump, uint64_t reinit_seed,
                             int want_reduction_error, ckf_recovery_report* out) {
  return guard([&] {
    ckf_recovery_report r = E(e)->recover_stage(stage, mode, moments, lr_bump, reinit_seed, want_reduction_error != 0);
    if (out) *out = r;
  });
}
int ckf_engine_export_stage(ckf_engine_t e, int stage, double* w, double* m, double* v) {
  return guard([&] { E(e)->export_group(E(e)->stage(stage), w, m, v); });
}
int ckf_engine_import_stage(ckf_engine_t e, int stage, const double* w, const double* m, const double* v) {
  return guard([&] { E(e)->import_group(E(e)->stage(stage), w, m, v); });
}
int ckf_engine_export_edge(ckf_engine_t e, int which, double* w, double* m, double* v) {
  return guard([&] { E(e)->export_group(which == 0 ? E(e)->embed() : E(e)->deembed(), w, m, v); });
}
int ckf_engine_import_edge(ckf_engine_t e, int which, const double* w, const double* m, const double* v) {
  return guard([&] { E(e)->import_group(which == 0 ? E(e)->embed() : E(e)->deembed(), w, m, v); });
}
int ckf_engine_get_scalars(ckf_engine_t e, int stage, double* omega, double* lr, long* step) {
  return guard([&] {
    auto& g = E(e)->stage(stage);
    if (omega) *omega = g.omega;
    if (lr) *lr = g.lr;
    if (step) *step = g.step;
  });
}
int ckf_engine_set_scalars(ckf_engine_t e, int stage, double omega, double lr, long step) {
  return guard([&] {
    auto& g = E(e)->stage(stage);
    g.omega = omega;
    g.lr = lr;
    g.step = step;
  });
}
int ckf_engine_get_edge_scalars(ckf_engine_t e, double* lr, long* se, long* sd) {
  return guard([&] {
    if (lr) *lr = E(e)->edge_lr;
    if (se) *se = E(e)->embed().step;
    if (sd) *sd = E(e)->deembed().step;
  });
}
int ckf_engine_set_edge_scalars(ckf_engine_t e, double lr, long se, long sd) {
  return guard([&] {
    E(e)->edge_lr = lr;
    E(e)->embed().step = se;
    E(e)->deembed().step = sd;
  });
}
int ckf_engine_set_schedule(ckf_engine_t e, int mode) {
  return guard([&] { E(e)->set_schedule(mode); });
}

int ckf_engine_set_redundant(ckf_engine_t e, int on) {
  return guard([&] { E(e)->set_redundant(on != 0); });
}

int ckf_engine_last_step_ms(ckf_engine_t e, float* ms) {
  return guard([&] { *ms = E(e)->last_step_ms(); });
}

int ckf_engine_set_edge_replicas(ckf_engine_t e, int on) {
  return guard([&] { E(e)->set_edge_replicas(on != 0); });
}

int ckf_engine_set_group_cap(ckf_engine_t e, int cap) {
  return guard([&] { E(e)->set_group_cap(cap); });
}
int ckf_engine_hop_log(ckf_engine_t e, int nranks, const int* stage_rank) {
  return guard([&] { E(e)->hop_log_enable(nranks, stage_rank); });
}
int ckf_engine_get_hop_log(ckf_engine_t e, long* out, int cap_triples, int* n_triples) {
  return guard([&] {
    const auto& l = E(e)->hop_log();
    const int n = static_cast<int>(l.size() / 3);
    if (n > cap_triples) ckf::raise(CKF_E_USAGE, "output buffer too small");
    std::copy(l.begin(), l.end(), out);
    *n_triples = n;
  });
}
long ckf_engine_kernel_launches(ckf_engine_t) { return ckf::launch_counter(); }
int ckf_engine_sync(ckf_engine_t e) {
  return guard([&] { CKF_CUDA(cudaStreamSynchronize(E(e)->stream())); });
}

int ckf_engine_stream(ckf_engine_t e, void** stream) {
  return guard([&] { *stream = static_cast<void*>(E(e)->stream()); });
}
int ckf_engine_kernel_timing(ckf_engine_t e, int enable) {
  return guard([&] { E(e)->kt_enable(enable != 0); });
}
int ckf_engine_kernel_stats(ckf_engine_t e, int cls, double* ms, long* launches, double* flops, double* bytes) {
  return guard([&] {
    if (cls < 0 || cls >= ckf::KC_N) ckf::raise(CKF_E_CONFIG, "kernel class out of range");
    const ckf::KStat& k = E(e)->kt_stat(cls);
    if (ms) *ms = k.ms;
    if (launches) *launches = k.launches;
    if (flops) *flops = k.flops;
    if (bytes) *bytes = k.bytes;
  });
}

// ---------------------------------------------------------------- (4) trainer
int ckf_run_experiment(const char* kv, const char* trace_text, uint64_t seed, char* record, size_t cap) {
  return guard([&] {
    const std::string r = ckf::run_experiment(kv ? kv : "", trace_text ? trace_text : "", seed, "");
    if (r.size() + 1 > cap) ckf::raise(CKF_E_USAGE, "record buffer too small");
    std::memcpy(record, r.c_str(), r.size() + 1);
  });
}

int ckf_run_experiment_rank(const char* kv, const char* trace_text, uint64_t seed, const void* nccl_uid, int nranks,
                            int rank, int replicas, char* record, size_t cap) {
  return guard([&] {
    if (!nccl_uid || nranks < 1 || rank < 0 || rank >= nranks || replicas < 1 || nranks % replicas)
      ckf::raise(CKF_E_CONFIG, "invalid world / rank / replicas");
    ckf::TrainerComm cm;
    cm.uid = nccl_uid;
    cm.nranks = nranks;
    cm.rank = rank;
    cm.replicas = replicas;
    const std::string r = ckf::run_experiment(kv ? kv : "", trace_text ? trace_text : "", seed, "", &cm);
    if (r.size() + 1 > cap) ckf::raise(CKF_E_USAGE, "record buffer too small");
    std::memcpy(record, r.c_str(), r.size() + 1);
  });
}

int ckf_run_experiment_to_dir(const char* kv, const char* trace_text, uint64_t seed, const char* dir) {
  return guard([&] {
    if (!dir || !*dir) ckf::raise(CKF_E_CONFIG, "output directory required");
    ckf::run_experiment(kv ? kv : "", trace_text ? trace_text : "", seed, dir);
  });
}

}  // extern "C"

// ------------------------------------------------------------------ LLaMA bandwidth kernels (standalone)
namespace {
void* scratch_ws(size_t bytes) {  // per-thread growable device scratch for the standalone entries
  static thread_local void* p = nullptr;
  static thread_local size_t have = 0;
  if (bytes > have) {
    if (p) CKF_CUDA(cudaFree(p));
    CKF_CUDA(cudaMalloc(&p, bytes));
    have = bytes;
  }
  return p;
}
}  // namespace

int ckf_llama_rmsnorm_fwd(const float* x, const float* g, size_t rows, size_t d, void* y_bf16, float* rstd,
                          float* xcopy, void* stream) {
  return guard([&] {
    ckf::llama::rmsnorm_fwd(x, g, rows, d, static_cast<__nv_bfloat16*>(y_bf16), rstd, xcopy,
                            static_cast<cudaStream_t>(stream));
  });
}
int ckf_llama_rmsnorm_bwd(const float* dy, const float* x, const float* g, const float* rstd, size_t rows, size_t d,
                          float* dh, void* dh_bf16, float* gg, void* stream) {
  return guard([&] {
    auto st = static_cast<cudaStream_t>(stream);
    const int nblk = ckf::llama::rmsnorm_bwd_blocks(rows);
    float* gpart = static_cast<float*>(scratch_ws(static_cast<size_t>(nblk) * d * sizeof(float)));
    ckf::llama::rmsnorm_bwd(dy, x, g, rstd, rows, d, dh, static_cast<__nv_bfloat16*>(dh_bf16), gpart, st);
    ckf::llama::gain_fold(gpart, nblk, d, gg, st);
    CKF_CUDA(cudaStreamSynchronize(st));
  });
}
int ckf_llama_rope(void* qkv, size_t ntok, size_t T, size_t d, size_t heads, int inverse, void* stream) {
  return guard([&] {
    ckf::llama::rope(static_cast<__nv_bfloat16*>(qkv), ntok, T, d, heads, inverse, static_cast<cudaStream_t>(stream));
  });
}
int ckf_llama_swiglu_fwd(const void* gu, size_t ntok, size_t f, void* a, void* stream) {
  return guard([&] {
    ckf::llama::swiglu_fwd(static_cast<const __nv_bfloat16*>(gu), ntok, f, static_cast<__nv_bfloat16*>(a),
                           static_cast<cudaStream_t>(stream));
  });
}
int ckf_llama_swiglu_bwd(const void* gu, const void* da, size_t ntok, size_t f, void* dgu, void* stream) {
  return guard([&] {
    ckf::llama::swiglu_bwd(static_cast<const __nv_bfloat16*>(gu), static_cast<const __nv_bfloat16*>(da), ntok, f,
                           static_cast<__nv_bfloat16*>(dgu), static_cast<cudaStream_t>(stream));
  });
}
int ckf_llama_embed_fwd(const int* tok, size_t ntok, const float* E, size_t d, float* h, void* stream) {
  return guard([&] { ckf::llama::embed_fwd(tok, ntok, E, d, h, static_cast<cudaStream_t>(stream)); });
}
int ckf_llama_embed_bwd(const int* tok, size_t ntok, const float* dh, size_t d, float* gE, void* stream) {
  return guard([&] {
    auto st = static_cast<cudaStream_t>(stream);
    ckf::llama::embed_bwd(tok, ntok, dh, d, gE, scratch_ws(ckf::llama::embed_bwd_scratch(ntok)), st);
    CKF_CUDA(cudaStreamSynchronize(st));
  });
}
int ckf_gemm_o_dgrad_dsum(int M, int K, const void* A, const void* B, void* C, const void* O, float* D, size_t T,
                          size_t heads, void* stream) {
  return guard([&] {
    const int hd = heads ? K / static_cast<int>(heads) : 0;
    if (K <= 0 || heads == 0 || K % static_cast<int>(heads) || (hd != 64 && hd != 128) || T == 0 || M % T)
      ckf::raise(CKF_E_CONFIG, "gemm_o_dgrad_dsum: head_dim 64 or 128, M a multiple of T");
    ckf::tc::GemmDesc g;
    g.M = M;
    g.N = K;
    g.K = K;
    g.A = static_cast<const __nv_bfloat16*>(A);
    g.lda = K;
    g.B = static_cast<const __nv_bfloat16*>(B);
    g.ldb = K;
    g.C = C;
    g.ldc = K;
    g.epi = ckf::tc::kStoreBF16;
    g.dsum_o = static_cast<const __nv_bfloat16*>(O);
    g.dsum_out = D;
    g.dsum_T = static_cast<int>(T);
    g.dsum_hd = hd;
    ckf::tc::gemm_bf16(g, static_cast<cudaStream_t>(stream));
  });
}
int ckf_gemm_qkv_rope(int M, int K, const void* A, const void* B, void* C, size_t T, size_t heads, void* stream) {
  return guard([&] {
    const int hd = heads ? K / static_cast<int>(heads) : 0;
    if (K <= 0 || heads == 0 || K % static_cast<int>(heads) || (hd != 64 && hd != 128))
      ckf::raise(CKF_E_CONFIG, "gemm_qkv_rope: the fused RoPE epilogue serves head_dim 64 or 128 (K = d = hd * heads)");
    auto st = static_cast<cudaStream_t>(stream);
    ckf::tc::GemmDesc g;
    g.M = M;
    g.N = 3 * K;
    g.K = K;
    g.A = static_cast<const __nv_bfloat16*>(A);
    g.lda = K;
    g.a_mn = false;
    g.B = static_cast<const __nv_bfloat16*>(B);
    g.ldb = 3 * K;
    g.b_mn = true;
    g.C = C;
    g.ldc = 3 * K;
    g.epi = ckf::tc::kStoreBF16;
    g.rope_tab = ckf::llama::rope_table_pair_major(T, hd, st);
    g.rope_T = static_cast<int>(T);
    g.rope_cols = 2 * K;
    g.rope_hd = hd;
    ckf::tc::gemm_bf16(g, st);
  });
}
