// ctypes shim over the UNMODIFIED reference library (test infrastructure only).
//
// Built by oracle/Makefile from the reference sources where they lie under
// /root/reference/proj/src (never copied into this repo) into oracle/_ref/.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs load it -- as the checker and the CPU baseline, never as product code.
//
// Every entry point forwards to the reference function named in its comment.

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "ckfree/dataset.hpp"
#include "ckfree/errors.hpp"
#include "ckfree/experiment.hpp"
#include "ckfree/failures.hpp"
#include "ckfree/kernels.hpp"
#include "ckfree/model.hpp"
#include "ckfree/pipeline.hpp"
#include "ckfree/recovery.hpp"
#include "ckfree/rng.hpp"

using namespace ckfree;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const NumericDivergenceError*>(&e)) return 2;
  if (dynamic_cast<const UsageError*>(&e)) return 3;
  if (dynamic_cast<const ParseError*>(&e)) return 4;
  if (dynamic_cast<const UnsupportedRecoveryError*>(&e)) return 5;
  return 9;
}

int copy_out(const std::string& s, char* out, std::size_t cap) {
  if (s.size() + 1 > cap) {
    g_err = "output buffer too small";
    return 8;
  }
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

// "key=value;key=value" -> map (keys as in ExperimentConfig::to_config_string).
std::map<std::string, std::string> parse_kv(const char* text) {
  std::map<std::string, std::string> kv;
  std::stringstream ss(text ? text : "");
  std::string item;
  while (std::getline(ss, item, ';')) {
    if (item.empty()) continue;
    auto eq = item.find('=');
    if (eq == std::string::npos) throw ConfigError("malformed kv item '" + item + "'");
    kv[item.substr(0, eq)] = item.substr(eq + 1);
  }
  return kv;
}

harness::ExperimentConfig config_from_kv(const char* text) {
  auto kv = parse_kv(text);
  harness::ExperimentConfig c;
  auto get = [&](const char* k) -> const std::string* {
    auto it = kv.find(k);
    return it == kv.end() ? nullptr : &it->second;
  };
  if (auto v = get("input-dim")) c.model.input_dim = std::stoul(*v);
  if (auto v = get("hidden-dim")) c.model.hidden_dim = std::stoul(*v);
  if (auto v = get("model-dim")) c.model.model_dim = std::stoul(*v);
  if (auto v = get("output-dim")) c.model.output_dim = std::stoul(*v);
  if (auto v = get("layers")) c.model.num_layers = std::stoul(*v);
  if (auto v = get("stages")) c.model.num_stages = std::stoul(*v);
  if (auto v = get("activation")) c.model.activation = parse_activation(*v);
  if (auto v = get("task")) c.model.task = parse_task(*v);
  if (auto v = get("strategy")) c.strategy.kind = recovery::parse_strategy(*v);
  if (auto v = get("checkpoint-interval")) c.strategy.checkpoint_interval = std::stol(*v);
  if (auto v = get("lr-bump")) c.strategy.lr_bump = std::stod(*v);
  if (auto v = get("recovered-moments"))
    c.strategy.recovered_moments =
        *v == "averaged" ? recovery::MomentRecovery::Averaged : recovery::MomentRecovery::Fresh;
  if (auto v = get("p-hour")) c.p_hour = std::stod(*v);
  if (auto v = get("p-iter")) c.p_iter = std::stod(*v);
  if (auto v = get("iter-seconds")) c.iteration_seconds = std::stod(*v);
  if (auto v = get("eligible")) c.eligible = *v;
  if (auto v = get("iters")) c.total_iterations = std::stol(*v);
  if (auto v = get("batch")) c.batch_size = std::stoul(*v);
  if (auto v = get("microbatches")) c.num_microbatches = std::stoi(*v);
  if (auto v = get("lr")) c.lr = std::stod(*v);
  if (auto v = get("eval-interval")) c.eval_interval = std::stol(*v);
  if (auto v = get("val-size")) c.val_size = std::stoul(*v);
  if (auto v = get("seed")) c.seed = std::stoull(*v);
  if (auto v = get("schedule")) c.schedule_mode = *v;
  if (auto v = get("swap-from")) c.swap_from_iteration = std::stol(*v);
  return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// rng.hpp:10-48
uint64_t ref_mix64(uint64_t x) { return rng::mix64(x); }
uint64_t ref_derive_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return rng::derive_key(seed, a, b, c);
}
double ref_unit_at(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { return rng::unit_at(seed, a, b, c); }
void ref_counter_uniform(uint64_t key, double lo, double hi, double* out, std::size_t n) {
  rng::CounterRng g(key);
  for (std::size_t i = 0; i < n; ++i) out[i] = g.uniform(lo, hi);
}

// failures.cpp:57-61
double ref_hourly_to_per_iteration(double p_hour, double iter_s) {
  return failures::hourly_to_per_iteration(p_hour, iter_s);
}

// failures.cpp:63-95: generate + serialize ("checkfree-trace v1")
int ref_generate_trace(uint64_t seed, double p_hour, double iter_s, long n_iters, const int* stages,
                       int n_stages, char* out, std::size_t cap) {
  try {
    failures::FailureRateSpec spec;
    spec.p_hour = p_hour;
    spec.seed = seed;
    spec.eligible_stages.assign(stages, stages + n_stages);
    return copy_out(failures::serialize_trace(failures::generate_trace(spec, n_iters, iter_s)), out, cap);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// failures.cpp:97-155 then 84-95 (parse -> canonical re-serialization)
int ref_parse_trace(const char* text, char* out, std::size_t cap) {
  try {
    return copy_out(failures::serialize_trace(failures::parse_trace(text)), out, cap);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// failures.cpp:171-184; writes (iteration, stage) pairs
int ref_consecutive_conflicts(const char* text, long* out, int cap, int* n_out) {
  try {
    auto c = failures::consecutive_conflicts(failures::parse_trace(text));
    if (static_cast<int>(c.size()) > cap) throw ConfigError("cap");
    for (std::size_t i = 0; i < c.size(); ++i) {
      out[2 * i] = c[i].iteration;
      out[2 * i + 1] = c[i].stage_id;
    }
    *n_out = static_cast<int>(c.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// model.cpp:63-73; writes first,last pairs
void ref_even_partition(std::size_t layers, std::size_t stages, std::size_t* out) {
  auto p = ModelSpec::even_partition(layers, stages);
  for (std::size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = p[i].first;
    out[2 * i + 1] = p[i].last;
  }
}

// pipeline.cpp:41-56; writes m*s stage ids
int ref_build_schedule(int m, int swapped_half, int s, int* out) {
  try {
    auto sch = pipeline::build_schedule(m, swapped_half ? pipeline::ScheduleMode::SwappedHalf
                                                        : pipeline::ScheduleMode::Standard, s);
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < s; ++j) out[k * s + j] = sch.orders[static_cast<std::size_t>(k)].sequence[static_cast<std::size_t>(j)];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// recovery.cpp:57-73
int ref_recover_checkfree(const double* wp, const double* wn, std::size_t n, double op, double on, double* out,
                          int* degenerate) {
  try {
    ParameterVector a(std::vector<double>(wp, wp + n), {n});
    ParameterVector b(std::vector<double>(wn, wn + n), {n});
    bool deg = false;
    ParameterVector r = recovery::recover_checkfree(a, b, op, on, &deg);
    std::memcpy(out, r.ptr(), n * sizeof(double));
    *degenerate = deg ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// recovery.cpp:120-126
int ref_reduction_error(const double* wp, const double* wf, const double* wn, std::size_t n, double op, double on,
                        double* out) {
  try {
    ParameterVector a(std::vector<double>(wp, wp + n), {n});
    ParameterVector f(std::vector<double>(wf, wf + n), {n});
    ParameterVector b(std::vector<double>(wn, wn + n), {n});
    *out = recovery::reduction_error(a, f, b, op, on);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_bump_lr(double lr, double f) { return recovery::bump_lr(lr, f); }

// Serial recover_checkfree timing, as shipped (allocation included): seconds per call.
double ref_time_recover_checkfree(std::size_t n, int reps) {
  std::vector<double> a(n), b(n);
  rng::CounterRng g(rng::derive_key(7, 1));
  for (std::size_t i = 0; i < n; ++i) {
    a[i] = g.uniform(-1, 1);
    b[i] = g.uniform(-1, 1);
  }
  ParameterVector pa(std::move(a), {n}), pb(std::move(b), {n});
  double sink = 0.0;
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    ParameterVector o = recovery::recover_checkfree(pa, pb, 4.0, 1.0);
    sink += o[static_cast<std::size_t>(r) % n];
  }
  auto t1 = std::chrono::steady_clock::now();
  if (sink == 12345.678) std::printf(" ");
  return std::chrono::duration<double>(t1 - t0).count() / reps;
}

// kernels_serial.cpp:104-115 / :133-144 (dispatching wrappers)
double ref_sum_squares(const double* x, std::size_t n) { return kernels::sum_squares(x, n); }
double ref_sum_squared_diff(const double* x, const double* y, std::size_t n) {
  return kernels::sum_squared_diff(x, y, n);
}
void ref_adam_update(double* w, double* m, double* v, const double* g, std::size_t n, double lr, long step) {
  kernels::adam_update(w, m, v, g, n, lr, kAdamBeta1, kAdamBeta2, kAdamEps, step);
}
void ref_gemm(int kind, const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) {
  switch (kind) {
    case 0: kernels::gemm_nn(a, b, c, m, k, n); break;
    case 1: kernels::gemm_nn_acc(a, b, c, m, k, n); break;
    case 2: kernels::gemm_nt_acc(a, b, c, m, k, n); break;
    default: kernels::gemm_tn_acc(a, b, c, m, k, n); break;
  }
}

// model.cpp:174-197: ModelState::all_weights_flat of init_model(spec, seed)
int ref_init_model_flat(const char* kv, uint64_t seed, double* out, std::size_t cap, std::size_t* n_out) {
  try {
    auto cfg = config_from_kv(kv);
    cfg.model.finalize();
    ModelState m = init_model(cfg.model, seed, cfg.lr);
    auto flat = m.all_weights_flat();
    if (flat.size() > cap) throw ConfigError("cap");
    std::memcpy(out, flat.data(), flat.size() * sizeof(double));
    *n_out = flat.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// dataset.cpp:15-57: x and regression targets of a training batch (index =
// model iteration) or of the validation set (index < 0).
int ref_batch(const char* kv, uint64_t run_seed, long index, std::size_t rows, double* x, double* y) {
  try {
    auto cfg = config_from_kv(kv);
    cfg.model.finalize();
    data::TaskContext task = harness::task_for_seed(cfg.model, run_seed);
    data::Batch b = index < 0 ? data::validation_set(task, rows) : data::training_batch(task, index, rows);
    std::memcpy(x, b.x.ptr(), b.x.size() * sizeof(double));
    if (cfg.model.task == TaskKind::Regression) {
      std::memcpy(y, b.y.values.ptr(), b.y.values.size() * sizeof(double));
    } else {
      for (std::size_t i = 0; i < rows; ++i) y[i] = b.y.labels[i];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One pipeline::run_iteration (pipeline.cpp:58-95) from init_model(seed) on
// an explicit batch: returns train loss, omegas, and the post-step flat weights.
int ref_run_iteration(const char* kv, uint64_t seed, int swapped_half, const double* x, const double* y,
                      std::size_t rows, long iteration, double* loss, double* omegas, double* flat_out) {
  try {
    auto cfg = config_from_kv(kv);
    cfg.model.finalize();
    ModelState m = init_model(cfg.model, seed, cfg.lr);
    Matrix xm(rows, cfg.model.input_dim);
    std::memcpy(xm.ptr(), x, xm.size() * sizeof(double));
    Targets t;
    if (cfg.model.task == TaskKind::Regression) {
      t.values = Matrix(rows, cfg.model.output_dim);
      std::memcpy(t.values.ptr(), y, t.values.size() * sizeof(double));
    } else {
      t.labels.resize(rows);
      for (std::size_t i = 0; i < rows; ++i) t.labels[i] = static_cast<int>(y[i]);
    }
    auto sch = pipeline::build_schedule(cfg.num_microbatches,
                                        swapped_half ? pipeline::ScheduleMode::SwappedHalf
                                                     : pipeline::ScheduleMode::Standard,
                                        static_cast<int>(cfg.model.num_stages));
    auto r = pipeline::run_iteration(m, sch, xm, t, iteration);
    *loss = r.train_loss;
    for (std::size_t i = 0; i < r.omegas.size(); ++i) omegas[i] = r.omegas[i];
    auto flat = m.all_weights_flat();
    std::memcpy(flat_out, flat.data(), flat.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// trainer.cpp:314-322 + experiment.cpp:156-174: metrics.csv and events.csv of one run.
int ref_run_experiment(const char* kv, const char* trace_text, uint64_t seed, char* metrics, std::size_t cap_m,
                       char* events, std::size_t cap_e) {
  try {
    auto cfg = config_from_kv(kv);
    failures::FailureTrace trace;
    if (trace_text && *trace_text) {
      trace = failures::parse_trace(trace_text);
    } else {
      cfg.model.finalize();
      trace = cfg.resolve_trace(seed);
    }
    harness::RunRecord rec = harness::run_experiment(cfg, trace, seed);
    int rc = copy_out(harness::metrics_csv(rec), metrics, cap_m);
    if (rc) return rc;
    return copy_out(harness::events_csv(rec), events, cap_e);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Same run, full-precision record: "E,iter,train,val" and
// "F,iter,stage,action,reduction_error,loss_spike" lines (%.17g), plus
// "U,<reason>" when the run stopped as unrecoverable.
int ref_run_experiment_full(const char* kv, const char* trace_text, uint64_t seed, char* out, std::size_t cap) {
  try {
    auto cfg = config_from_kv(kv);
    failures::FailureTrace trace = failures::parse_trace(trace_text);
    harness::RunRecord rec = harness::run_experiment(cfg, trace, seed);
    std::ostringstream o;
    char buf[256];
    for (const auto& e : rec.evals) {
      std::snprintf(buf, sizeof(buf), "E,%ld,%.17g,%.17g\n", e.iter, e.train_loss, e.val_loss);
      o << buf;
    }
    for (const auto& e : rec.events) {
      std::snprintf(buf, sizeof(buf), "F,%ld,%d,%s,%.17g,%.17g\n", e.iter, e.stage, e.action.c_str(),
                    e.reduction_error, e.loss_spike);
      o << buf;
    }
    if (rec.unrecoverable) o << "U," << rec.unrecoverable_reason << "\n";
    return copy_out(o.str(), out, cap);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU-baseline timing of the reference training loop body (trainer.cpp:75-84:
// training_batch + run_iteration), `iters` timed iterations after one warm-up.
// Returns seconds per iteration.
double ref_time_train_iterations(const char* kv, uint64_t seed, int iters) {
  try {
    auto cfg = config_from_kv(kv);
    cfg.model.finalize();
    data::TaskContext task = harness::task_for_seed(cfg.model, seed);
    ModelState m = init_model(cfg.model, rng::derive_key(seed, 11), cfg.lr);
    auto sch = pipeline::build_schedule(cfg.num_microbatches, cfg.resolved_schedule(),
                                        static_cast<int>(cfg.model.num_stages));
    {
      data::Batch b = data::training_batch(task, 1, cfg.batch_size);
      pipeline::run_iteration(m, sch, b.x, b.y, 1);
    }
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) {
      data::Batch b = data::training_batch(task, i + 2, cfg.batch_size);
      pipeline::run_iteration(m, sch, b.x, b.y, i + 2);
    }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count() / iters;
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

int ref_parallel_threads() { return kernels::parallel_threads(); }

}  // extern "C"
