// libckfree_b200: the reference's C++ stage / pipeline / recovery / failure API
// (/root/reference/proj/include/ckfree) re-implemented over the C-ABI of the
// B200 engine (include/ckf.h -> paper_2506_15461_b200/libckf.so).
//
// Host C++ keeps the reference's value semantics and error behaviour; every
// floating-point operation is a GPU kernel reached through the C-ABI:
//   * ckfree::kernels::*          -> ckf_k_* (device fp64 kernels)
//   * forward / backward          -> a cached device engine (ckf_engine_*), fp64
//   * init streams                -> ckf_k_counter_uniform (device counter RNG)
//   * recovery arithmetic         -> ckf_k_recover_checkfree / ckf_k_sum_squared_diff
//   * traces, schedules           -> ckf_generate_trace / ckf_parse_trace / ckf_build_schedule
// A C-ABI status is rethrown as the matching ckfree exception (errors.hpp).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../include/ckf.h"
#include "ckfree/errors.hpp"
#include "ckfree/failures.hpp"
#include "ckfree/kernels.hpp"
#include "ckfree/model.hpp"
#include "ckfree/pipeline.hpp"
#include "ckfree/recovery.hpp"
#include "ckfree/rng.hpp"

namespace {

// ------------------------------------------------------------------ C-ABI status -> exception
void ck(int rc) {
  if (rc == CKF_OK) return;
  const std::string msg = ckf_last_error();
  switch (rc) {
    case CKF_E_CONFIG: throw ckfree::ConfigError(msg);
    case CKF_E_DIVERGENCE: throw ckfree::NumericDivergenceError(msg, ckf_last_error_iteration());
    case CKF_E_USAGE: throw ckfree::UsageError(msg);
    case CKF_E_PARSE: throw ckfree::ParseError(msg);
    case CKF_E_UNSUPPORTED_RECOVERY: throw ckfree::UnsupportedRecoveryError(msg);
    default: throw std::runtime_error("B200 engine: " + msg);
  }
}

// ------------------------------------------------------------------ device engines for forward/backward
// One fp64 engine per model shape, created on first use and reused; the
// host ModelState is the source of truth and is uploaded per call.
struct DeviceModel {
  ckf_engine_t h = nullptr;
  ~DeviceModel() {
    if (h) ckf_engine_destroy(h);
  }
};

std::string shape_key(const ckfree::ModelSpec& s) {
  std::ostringstream k;
  k << s.input_dim << ',' << s.hidden_dim << ',' << s.model_dim << ',' << s.output_dim << ',' << s.num_layers << ','
    << s.num_stages << ',' << static_cast<int>(s.activation) << ',' << static_cast<int>(s.task);
  for (const auto& r : s.partition) k << ';' << r.first << '-' << r.last;
  return k.str();
}

ckf_engine_t engine_for(const ckfree::ModelSpec& spec) {
  static std::mutex mu;
  static std::map<std::string, std::unique_ptr<DeviceModel>> cache;
  std::lock_guard<std::mutex> lock(mu);
  const std::string key = shape_key(spec);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second->h;
  if (cache.size() >= 8) cache.clear();  // bound device memory held by idle shapes
  std::vector<size_t> part;
  for (const auto& r : spec.partition) {
    part.push_back(r.first);
    part.push_back(r.last);
  }
  ckf_model_desc d{};
  d.block = CKF_BLOCK_MLP;
  d.precision = CKF_FP64;
  d.activation = static_cast<int>(spec.activation);
  d.task = spec.task == ckfree::TaskKind::Regression ? CKF_TASK_REGRESSION : CKF_TASK_CLASSIFICATION;
  d.input_dim = spec.input_dim;
  d.hidden_dim = spec.hidden_dim;
  d.model_dim = spec.model_dim;
  d.output_dim = spec.output_dim;
  d.num_layers = spec.num_layers;
  d.num_stages = spec.num_stages;
  d.partition = part.data();
  d.max_rows = 256;
  d.device = 0;
  auto dm = std::make_unique<DeviceModel>();
  ck(ckf_engine_create(&d, &dm->h));
  ckf_engine_t h = dm->h;
  cache.emplace(key, std::move(dm));
  return h;
}

// Stage weights as uploaded: W2 of masked-out layers zeroed, which turns a
// block into the identity exactly (h + act(h W1) * 0 = h).
void upload(ckf_engine_t e, const ckfree::ModelState& m, const std::vector<int>* mask) {
  for (const auto& st : m.stages) {
    ckfree::ParameterVector flat = st.flat_weights();
    if (mask && !mask->empty()) {
      const ckfree::LayerRange& r = m.spec.stage_range(st.stage_id);
      size_t off = 0;
      for (size_t bi = 0; bi < st.blocks.size(); ++bi) {
        const size_t n1 = st.blocks[bi].w1.size(), n2 = st.blocks[bi].w2.size();
        if ((*mask)[r.first + bi - 1] == 0) std::fill(flat.ptr() + off + n1, flat.ptr() + off + n1 + n2, 0.0);
        off += n1 + n2;
      }
    }
    ck(ckf_engine_import_stage(e, st.stage_id, flat.ptr(), nullptr, nullptr));
  }
  ck(ckf_engine_import_edge(e, 0, m.edges.layers.embed.ptr(), nullptr, nullptr));
  ck(ckf_engine_import_edge(e, 1, m.edges.layers.deembed.ptr(), nullptr, nullptr));
}

void check_order(const ckfree::ModelSpec& spec, const std::vector<int>& order) {
  if (order.size() != spec.num_stages) throw ckfree::ConfigError("stage order length must equal num_stages");
  std::vector<char> seen(spec.num_stages, 0);
  for (int sid : order) {
    if (sid < 1 || static_cast<size_t>(sid) > spec.num_stages || seen[static_cast<size_t>(sid) - 1])
      throw ckfree::ConfigError("stage order must be a permutation of [1..num_stages]");
    seen[static_cast<size_t>(sid) - 1] = 1;
  }
}

// targets -> the engine's y layout (regression rows x out; classification labels as fp64)
std::vector<double> target_rows(const ckfree::ModelSpec& spec, const ckfree::Targets& t, size_t rows) {
  if (spec.task == ckfree::TaskKind::Regression) {
    if (t.values.rows != rows || t.values.cols != spec.output_dim)
      throw ckfree::ConfigError("target matrix shape does not match predictions");
    return t.values.data;
  }
  if (t.labels.size() != rows) throw ckfree::ConfigError("label count does not match batch size");
  std::vector<double> y(rows);
  for (size_t i = 0; i < rows; ++i) {
    if (t.labels[i] < 0 || static_cast<size_t>(t.labels[i]) >= spec.output_dim)
      throw ckfree::ConfigError("label out of range for output_dim");
    y[i] = t.labels[i];
  }
  return y;
}

ckfree::ParameterVector device_uniform(std::vector<size_t> shape, size_t fan_in, size_t fan_out, uint64_t key) {
  // sample_uniform semantics: U[-a, a], a = sqrt(6 / (fan_in + fan_out)), counters 1..n of key
  ckfree::ParameterVector p = ckfree::ParameterVector::zeros(std::move(shape));
  const double a = std::sqrt(6.0 / static_cast<double>(fan_in + fan_out));
  if (p.size()) ck(ckf_k_counter_uniform(key, -a, a, p.ptr(), p.size()));
  return p;
}

}  // namespace

// ====================================================================== kernels
namespace ckfree::kernels {

namespace {
Backend g_backend = Backend::Parallel;
}
Backend active_backend() { return g_backend; }
void set_backend(Backend b) { g_backend = b; }
bool parallel_available() { return true; }
int parallel_threads() {
  int n = 0;
  return ckf_device_count(&n) == CKF_OK && n > 0 ? 148 : 1;  // B200 SMs
}

#define CKF_DROPIN_IMPL                                                                                        \
  void gemm_nn(const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) {     \
    if (m && n) ck(ckf_k_gemm_nn(a, b, c, m, k, n));                                                           \
  }                                                                                                            \
  void gemm_nn_acc(const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) { \
    if (m && n && k) ck(ckf_k_gemm_nn_acc(a, b, c, m, k, n));                                                  \
  }                                                                                                            \
  void gemm_nt_acc(const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) { \
    if (m && n && k) ck(ckf_k_gemm_nt_acc(a, b, c, m, k, n));                                                  \
  }                                                                                                            \
  void gemm_tn_acc(const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) { \
    if (m && n && k) ck(ckf_k_gemm_tn_acc(a, b, c, m, k, n));                                                  \
  }                                                                                                            \
  void add_inplace(double* x, const double* y, std::size_t n) {                                               \
    if (n) ck(ckf_k_add_inplace(x, y, n));                                                                     \
  }                                                                                                            \
  void axpy(double alpha, const double* x, double* y, std::size_t n) {                                        \
    if (n) ck(ckf_k_axpy(alpha, x, y, n));                                                                     \
  }                                                                                                            \
  void scale(double alpha, double* x, std::size_t n) {                                                         \
    if (n) ck(ckf_k_scale(alpha, x, n));                                                                       \
  }                                                                                                            \
  void apply_activation(Activation act, const double* a, double* z, std::size_t n) {                          \
    if (n) ck(ckf_k_apply_activation(static_cast<int>(act), a, z, n));                                        \
  }                                                                                                            \
  void activation_backward(Activation act, const double* z, const double* dz, double* da, std::size_t n) {    \
    if (n) ck(ckf_k_activation_backward(static_cast<int>(act), z, dz, da, n));                                 \
  }                                                                                                            \
  double sum_squares(const double* x, std::size_t n) {                                                         \
    double out = 0.0;                                                                                          \
    if (n) ck(ckf_k_sum_squares(x, n, &out));                                                                  \
    return out;                                                                                                \
  }                                                                                                            \
  double sum_squared_diff(const double* x, const double* y, std::size_t n) {                                  \
    double out = 0.0;                                                                                          \
    if (n) ck(ckf_k_sum_squared_diff(x, y, n, &out));                                                          \
    return out;                                                                                                \
  }                                                                                                            \
  void adam_update(double* w, double* m, double* v, const double* g, std::size_t n, double lr, double b1,       \
                   double b2, double eps, long step) {                                                         \
    if (n) ck(ckf_k_adam_update(w, m, v, g, n, lr, b1, b2, eps, step));                                        \
  }                                                                                                            \
  double mse_loss_grad(const double* pred, const double* target, std::size_t rows, std::size_t cols,          \
                       double* dpred) {                                                                        \
    double loss = 0.0;                                                                                         \
    if (rows && cols) ck(ckf_k_mse_loss_grad(pred, target, rows, cols, dpred, &loss));                         \
    return loss;                                                                                               \
  }                                                                                                            \
  double softmax_xent_loss_grad(const double* logits, const int* labels, std::size_t rows, std::size_t cols,  \
                                double* dlogits) {                                                             \
    double loss = 0.0;                                                                                         \
    if (rows && cols) ck(ckf_k_softmax_xent_loss_grad(logits, labels, rows, cols, dlogits, &loss));            \
    return loss;                                                                                               \
  }

namespace serial {
CKF_DROPIN_IMPL
}
namespace par {
CKF_DROPIN_IMPL
}
CKF_DROPIN_IMPL
#undef CKF_DROPIN_IMPL

}  // namespace ckfree::kernels

// ====================================================================== model
namespace ckfree {

Activation parse_activation(const std::string& name) {
  static const std::map<std::string, Activation> m{
      {"tanh", Activation::Tanh}, {"relu", Activation::Relu}, {"identity", Activation::Identity}};
  auto it = m.find(name);
  if (it == m.end()) throw ConfigError("unknown activation '" + name + "' (expected tanh|relu|identity)");
  return it->second;
}
TaskKind parse_task(const std::string& name) {
  if (name == "regression") return TaskKind::Regression;
  if (name == "classification") return TaskKind::Classification;
  throw ConfigError("unknown task '" + name + "' (expected regression|classification)");
}
const char* to_string(Activation act) {
  return act == Activation::Tanh ? "tanh" : act == Activation::Relu ? "relu" : "identity";
}
const char* to_string(TaskKind task) { return task == TaskKind::Classification ? "classification" : "regression"; }

std::vector<LayerRange> ModelSpec::even_partition(std::size_t layers, std::size_t stages) {
  std::vector<size_t> pairs(2 * stages);
  ck(ckf_even_partition(layers, stages, pairs.data()));
  std::vector<LayerRange> out(stages);
  for (size_t i = 0; i < stages; ++i) out[i] = {pairs[2 * i], pairs[2 * i + 1]};
  return out;
}

void ModelSpec::finalize() {
  if (partition.empty()) partition = even_partition(num_layers, num_stages);
  validate();
}

void ModelSpec::validate() const {
  if (!input_dim || !hidden_dim || !model_dim || !output_dim || !num_layers)
    throw ConfigError("model dimensions and layer count must be positive");
  if (num_stages < 1 || num_stages > num_layers) throw ConfigError("num_stages must lie in [1, num_layers]");
  if (partition.size() != num_stages) throw ConfigError("partition must contain exactly num_stages ranges");
  size_t next = 1;
  for (const LayerRange& r : partition) {
    const bool ok = r.first == next && r.last >= r.first && r.last <= num_layers;
    if (!ok) throw ConfigError("partition ranges must be contiguous, ordered and cover [1, num_layers]");
    next = r.last + 1;
  }
  if (next != num_layers + 1) throw ConfigError("partition does not cover all layers");
  if (task == TaskKind::Classification && output_dim < 2)
    throw ConfigError("classification requires output_dim >= 2");
}

bool ModelSpec::uniform_partition() const {
  return std::all_of(partition.begin(), partition.end(),
                     [&](const LayerRange& r) { return r.count() == partition.front().count(); });
}

int ModelSpec::stage_of_layer(std::size_t layer) const {
  for (size_t i = 0; i < partition.size(); ++i)
    if (partition[i].first <= layer && layer <= partition[i].last) return static_cast<int>(i) + 1;
  throw ConfigError("layer index out of range");
}

std::size_t StageState::param_count() const {
  size_t n = 0;
  for (const ResidualBlock& b : blocks) n += b.param_count();
  return n;
}

ParameterVector StageState::flat_weights() const {
  std::vector<double> v;
  v.reserve(param_count());
  for (const ResidualBlock& b : blocks)
    for (const ParameterVector* p : {&b.w1, &b.w2}) v.insert(v.end(), p->values().begin(), p->values().end());
  const size_t n = v.size();
  return ParameterVector(std::move(v), {n});
}

void StageState::set_flat_weights(const ParameterVector& flat) {
  if (flat.size() != param_count()) throw ConfigError("flat weight size does not match stage parameter count");
  const double* src = flat.ptr();
  for (ResidualBlock& b : blocks)
    for (ParameterVector* p : {&b.w1, &b.w2}) {
      std::copy(src, src + p->size(), p->ptr());
      src += p->size();
    }
}

std::size_t ModelState::param_count() const {
  size_t n = edges.layers.embed.size() + edges.layers.deembed.size();
  for (const StageState& s : stages) n += s.param_count();
  return n;
}

std::vector<double> ModelState::all_weights_flat() const {
  std::vector<double> v(edges.layers.embed.values());
  v.insert(v.end(), edges.layers.deembed.values().begin(), edges.layers.deembed.values().end());
  for (const StageState& s : stages) {
    const ParameterVector f = s.flat_weights();
    v.insert(v.end(), f.values().begin(), f.values().end());
  }
  return v;
}

std::vector<ResidualBlock> init_stage_blocks(const ModelSpec& spec, int stage_id, std::uint64_t seed) {
  const LayerRange& r = spec.stage_range(stage_id);
  std::vector<ResidualBlock> out;
  for (size_t l = r.first; l <= r.last; ++l) {
    ResidualBlock b;  // tensor tags 2l / 2l+1 keep every tensor's stream partition-independent
    b.w1 = device_uniform({spec.model_dim, spec.hidden_dim}, spec.model_dim, spec.hidden_dim,
                          rng::derive_key(seed, 2 * l));
    b.w2 = device_uniform({spec.hidden_dim, spec.model_dim}, spec.hidden_dim, spec.model_dim,
                          rng::derive_key(seed, 2 * l + 1));
    out.push_back(std::move(b));
  }
  return out;
}

ModelState init_model(const ModelSpec& spec, std::uint64_t seed, double base_lr) {
  spec.validate();
  ModelState m;
  m.spec = spec;
  m.edges.layers.embed =
      device_uniform({spec.input_dim, spec.model_dim}, spec.input_dim, spec.model_dim, rng::derive_key(seed, 0));
  m.edges.layers.deembed =
      device_uniform({spec.model_dim, spec.output_dim}, spec.model_dim, spec.output_dim, rng::derive_key(seed, 1));
  m.edges.opt_embed.reset(m.edges.layers.embed.size());
  m.edges.opt_deembed.reset(m.edges.layers.deembed.size());
  m.edges.lr = base_lr;
  for (size_t i = 0; i < spec.num_stages; ++i) {
    StageState s;
    s.stage_id = static_cast<int>(i) + 1;
    s.blocks = init_stage_blocks(spec, s.stage_id, seed);
    s.opt.reset(s.param_count());
    s.lr = base_lr;
    m.stages.push_back(std::move(s));
  }
  return m;
}

namespace {
ForwardCache forward_on_device(const ModelState& model, const std::vector<int>& order, const Matrix& batch,
                               const std::vector<int>* mask, long iteration) {
  const ModelSpec& spec = model.spec;
  check_order(spec, order);
  if (batch.cols != spec.input_dim)
    throw ConfigError("batch column count " + std::to_string(batch.cols) + " does not match input_dim " +
                      std::to_string(spec.input_dim));
  if (mask && mask->size() != spec.num_layers) throw ConfigError("layer mask length must equal num_layers");
  ForwardCache c;
  c.stage_order = order;
  c.input = batch;
  c.iteration = iteration;
  if (mask) c.layer_mask = *mask;
  c.predictions = Matrix(batch.rows, spec.output_dim);
  if (batch.rows) {
    ckf_engine_t e = engine_for(spec);
    upload(e, model, mask);
    ck(ckf_engine_predict(e, order.data(), batch.ptr(), batch.rows, c.predictions.ptr()));
  }
  for (double v : c.predictions.data)
    if (!std::isfinite(v)) throw NumericDivergenceError("forward: non-finite activation", iteration);
  c.valid = true;
  return c;
}
}  // namespace

ForwardCache forward(const ModelState& model, const std::vector<int>& stage_order, const Matrix& batch,
                     long iteration) {
  return forward_on_device(model, stage_order, batch, nullptr, iteration);
}

ForwardCache forward_masked(const ModelState& model, const std::vector<int>& stage_order, const Matrix& batch,
                            const std::vector<int>& layer_mask, long iteration) {
  return forward_on_device(model, stage_order, batch, &layer_mask, iteration);
}

Gradients Gradients::zeros_like(const ModelState& model) {
  Gradients g;
  for (const StageState& s : model.stages) g.stage.emplace_back(s.param_count(), 0.0);
  g.embed.assign(model.edges.layers.embed.size(), 0.0);
  g.deembed.assign(model.edges.layers.deembed.size(), 0.0);
  return g;
}

void Gradients::accumulate(const Gradients& other) {
  for (size_t i = 0; i < stage.size(); ++i) kernels::add_inplace(stage[i].data(), other.stage[i].data(), stage[i].size());
  kernels::add_inplace(embed.data(), other.embed.data(), embed.size());
  kernels::add_inplace(deembed.data(), other.deembed.data(), deembed.size());
  loss += other.loss;
}

void Gradients::scale_all(double a) {
  for (auto& s : stage) kernels::scale(a, s.data(), s.size());
  kernels::scale(a, embed.data(), embed.size());
  kernels::scale(a, deembed.data(), deembed.size());
  loss *= a;
}

Gradients backward(const ModelState& model, const ForwardCache& cache, const Targets& targets) {
  if (!cache.valid) throw UsageError("backward called without a matching forward cache");
  const ModelSpec& spec = model.spec;
  const size_t rows = cache.input.rows;
  const std::vector<double> y = target_rows(spec, targets, rows);
  Gradients g = Gradients::zeros_like(model);
  if (rows == 0) return g;
  ckf_engine_t e = engine_for(spec);
  upload(e, model, cache.layer_mask.empty() ? nullptr : &cache.layer_mask);
  ck(ckf_engine_zero_grad(e));
  // the device replays the microbatch (forward + backward) and accumulates into its gradient buffers
  ck(ckf_engine_accumulate(e, cache.stage_order.data(), cache.input.ptr(), y.data(), rows, 0, &g.loss));
  for (const StageState& s : model.stages) ck(ckf_engine_export_grad(e, 2, s.stage_id, g.stage[static_cast<size_t>(s.stage_id) - 1].data()));
  ck(ckf_engine_export_grad(e, 0, 0, g.embed.data()));
  ck(ckf_engine_export_grad(e, 1, 0, g.deembed.data()));
  if (!cache.layer_mask.empty()) {
    // a skipped block contributes no gradient (it was never applied)
    for (const StageState& s : model.stages) {
      const LayerRange& r = spec.stage_range(s.stage_id);
      size_t off = 0;
      for (size_t bi = 0; bi < s.blocks.size(); ++bi) {
        const size_t n = s.blocks[bi].param_count();
        if (cache.layer_mask[r.first + bi - 1] == 0)
          std::fill_n(g.stage[static_cast<size_t>(s.stage_id) - 1].begin() + static_cast<std::ptrdiff_t>(off), n, 0.0);
        off += n;
      }
    }
  }
  for (const auto& sg : g.stage)
    for (double v : sg)
      if (!std::isfinite(v)) throw NumericDivergenceError("backward: non-finite gradient", cache.iteration);
  return g;
}

double loss_value(const ModelState& model, const Matrix& predictions, const Targets& targets) {
  const ModelSpec& spec = model.spec;
  if (spec.task == TaskKind::Regression) {
    if (targets.values.rows != predictions.rows || targets.values.cols != predictions.cols)
      throw ConfigError("target matrix shape does not match predictions");
    return kernels::mse_loss_grad(predictions.ptr(), targets.values.ptr(), predictions.rows, predictions.cols,
                                  nullptr);
  }
  if (targets.labels.size() != predictions.rows) throw ConfigError("label count does not match batch size");
  for (int l : targets.labels)
    if (l < 0 || static_cast<size_t>(l) >= predictions.cols) throw ConfigError("label out of range for output_dim");
  return kernels::softmax_xent_loss_grad(predictions.ptr(), targets.labels.data(), predictions.rows,
                                         predictions.cols, nullptr);
}

void adam_step(StageState& stage, const std::vector<double>& grads, double lr) {
  if (grads.size() != stage.param_count()) throw ConfigError("gradient size does not match stage parameter count");
  if (!(lr > 0.0)) throw ConfigError("learning rate must be positive");
  if (!std::all_of(grads.begin(), grads.end(), [](double v) { return std::isfinite(v); }))
    throw NumericDivergenceError("adam_step: non-finite gradient");
  ParameterVector w = stage.flat_weights();
  stage.opt.step += 1;
  kernels::adam_update(w.ptr(), stage.opt.m.data(), stage.opt.v.data(), grads.data(), w.size(), lr, kAdamBeta1,
                       kAdamBeta2, kAdamEps, stage.opt.step);
  stage.set_flat_weights(w);
  stage.omega = grad_norm_sq(grads);
}

void adam_step_edges(EdgeState& edges, const std::vector<double>& g_embed, const std::vector<double>& g_deembed) {
  edges.opt_embed.step += 1;
  kernels::adam_update(edges.layers.embed.ptr(), edges.opt_embed.m.data(), edges.opt_embed.v.data(), g_embed.data(),
                       g_embed.size(), edges.lr, kAdamBeta1, kAdamBeta2, kAdamEps, edges.opt_embed.step);
  edges.opt_deembed.step += 1;
  kernels::adam_update(edges.layers.deembed.ptr(), edges.opt_deembed.m.data(), edges.opt_deembed.v.data(),
                       g_deembed.data(), g_deembed.size(), edges.lr, kAdamBeta1, kAdamBeta2, kAdamEps,
                       edges.opt_deembed.step);
}

double grad_norm_sq(const std::vector<double>& grads) { return kernels::sum_squares(grads.data(), grads.size()); }

double layer_omission_loss(const ModelState& model, const std::vector<int>& layer_mask, const Matrix& batch,
                           const Targets& targets) {
  std::vector<int> order(model.spec.num_stages);
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i) + 1;
  return loss_value(model, forward_masked(model, order, batch, layer_mask).predictions, targets);
}

}  // namespace ckfree

// ====================================================================== pipeline
namespace ckfree::pipeline {

ExecutionOrder ExecutionOrder::standard(int num_stages) {
  ExecutionOrder o;
  for (int i = 1; i <= num_stages; ++i) o.sequence.push_back(i);
  return o;
}

ExecutionOrder ExecutionOrder::swapped(int num_stages) {
  if (num_stages < 4)
    throw ConfigError("swapped order requires at least 4 stages (first and last pairs must be disjoint)");
  ExecutionOrder o = standard(num_stages);
  std::swap(o.sequence[0], o.sequence[1]);
  std::swap(o.sequence[static_cast<size_t>(num_stages) - 2], o.sequence[static_cast<size_t>(num_stages) - 1]);
  return o;
}

bool ExecutionOrder::is_standard() const {
  for (size_t i = 0; i < sequence.size(); ++i)
    if (sequence[i] != static_cast<int>(i) + 1) return false;
  return true;
}

int MicrobatchSchedule::swapped_count() const {
  return static_cast<int>(std::count_if(orders.begin(), orders.end(), [](const ExecutionOrder& o) {
    return !o.is_standard();
  }));
}

MicrobatchSchedule build_schedule(int num_microbatches, ScheduleMode mode, int num_stages) {
  if (num_microbatches < 1) throw ConfigError("microbatch count must be positive");
  const bool sw = mode == ScheduleMode::SwappedHalf;
  if (sw && num_microbatches % 2) throw ConfigError("swapped_half schedule requires an even microbatch count");
  if (sw && num_stages < 4)
    throw ConfigError("swapped order requires at least 4 stages (first and last pairs must be disjoint)");
  std::vector<int> flat(static_cast<size_t>(num_microbatches) * static_cast<size_t>(num_stages));
  ck(ckf_build_schedule(num_microbatches, sw ? 1 : 0, num_stages, flat.data()));  // host logic, bit-exact
  MicrobatchSchedule s;
  s.num_microbatches = num_microbatches;
  for (int k = 0; k < num_microbatches; ++k) {
    ExecutionOrder o;
    o.sequence.assign(flat.begin() + k * num_stages, flat.begin() + (k + 1) * num_stages);
    s.orders.push_back(std::move(o));
  }
  return s;
}

IterationResult run_iteration(ModelState& model, const MicrobatchSchedule& schedule, const Matrix& x,
                              const Targets& y, long iteration) {
  const int m = schedule.num_microbatches;
  if (static_cast<int>(schedule.orders.size()) != m)
    throw ConfigError("schedule order count does not match microbatch count");
  if (x.rows == 0 || x.rows % static_cast<size_t>(m))
    throw ConfigError("batch size must be divisible by the microbatch count");
  const size_t per = x.rows / static_cast<size_t>(m);
  Gradients sum = Gradients::zeros_like(model);
  for (int k = 0; k < m; ++k) {
    const size_t r0 = static_cast<size_t>(k) * per;
    Targets yk;
    if (model.spec.task == TaskKind::Regression)
      yk.values = y.values.row_slice(r0, per);
    else
      yk.labels.assign(y.labels.begin() + static_cast<std::ptrdiff_t>(r0),
                       y.labels.begin() + static_cast<std::ptrdiff_t>(r0 + per));
    const ForwardCache c = forward(model, schedule.orders[static_cast<size_t>(k)].sequence, x.row_slice(r0, per),
                                   iteration);
    sum.accumulate(backward(model, c, yk));
  }
  sum.scale_all(1.0 / static_cast<double>(m));  // mean gradient and mean loss
  for (StageState& st : model.stages) adam_step(st, sum.stage[static_cast<size_t>(st.stage_id) - 1], st.lr);
  adam_step_edges(model.edges, sum.embed, sum.deembed);
  IterationResult r;
  r.train_loss = sum.loss;
  r.iteration = iteration;
  for (const StageState& st : model.stages) r.omegas.push_back(st.omega);
  return r;
}

std::vector<std::size_t> effective_function(const ExecutionOrder& order, const ModelSpec& spec) {
  if (order.sequence.size() != spec.num_stages) throw ConfigError("execution order length must equal num_stages");
  std::vector<size_t> out;
  for (int sid : order.sequence)
    for (size_t l = spec.stage_range(sid).first; l <= spec.stage_range(sid).last; ++l) out.push_back(l);
  return out;
}

}  // namespace ckfree::pipeline

// ====================================================================== recovery
namespace ckfree::recovery {

namespace {
const std::pair<StrategyKind, const char*> kNames[] = {
    {StrategyKind::NoFailures, "no-failures"},     {StrategyKind::Checkpointing, "checkpointing"},
    {StrategyKind::RedundantComputation, "redundant"}, {StrategyKind::CheckFree, "checkfree"},
    {StrategyKind::CheckFreePlus, "checkfree-plus"}, {StrategyKind::ReinitRandom, "reinit-random"},
    {StrategyKind::ReinitCopy, "reinit-copy"},     {StrategyKind::ReinitUniformAvg, "reinit-uniform-avg"},
};

ParameterVector weighted(const ParameterVector& a, const ParameterVector& b, double wa, double wb, bool* deg) {
  if (!a.same_shape(b)) throw ConfigError("neighbor stage weights differ in shape");
  if (wa < 0.0 || wb < 0.0) throw ConfigError("gradient norms must be nonnegative");
  std::vector<double> out(a.size());
  int degenerate = 0;
  if (a.size()) ck(ckf_k_recover_checkfree(a.ptr(), b.ptr(), a.size(), wa, wb, out.data(), &degenerate));
  else degenerate = wa + wb == 0.0;
  if (deg) *deg = degenerate != 0;
  return ParameterVector(std::move(out), a.shape());
}
}  // namespace

const char* to_string(StrategyKind kind) {
  for (const auto& kv : kNames)
    if (kv.first == kind) return kv.second;
  return "?";
}

StrategyKind parse_strategy(const std::string& name) {
  for (const auto& kv : kNames)
    if (name == kv.second) return kv.first;
  throw ConfigError("unknown strategy '" + name + "'");
}

void StrategyConfig::validate() const {
  if (!(lr_bump > 0.0)) throw ConfigError("lr_bump must be positive");
  if (kind == StrategyKind::Checkpointing && checkpoint_interval < 1)
    throw ConfigError("checkpoint interval must be >= 1");
}

bool StrategyConfig::neighbor_based() const {
  return kind == StrategyKind::CheckFree || kind == StrategyKind::CheckFreePlus || kind == StrategyKind::ReinitCopy ||
         kind == StrategyKind::ReinitUniformAvg || kind == StrategyKind::ReinitRandom;
}

ParameterVector recover_checkfree(const ParameterVector& w_prev, const ParameterVector& w_next, double omega_prev,
                                  double omega_next, bool* degenerate) {
  bool deg = false;
  ParameterVector out = weighted(w_prev, w_next, omega_prev, omega_next, &deg);
  if (deg) std::fprintf(stderr, "warning: both neighbor gradient norms are zero; using the uniform average\n");
  if (degenerate) *degenerate = deg;
  return out;
}

double bump_lr(double lr, double factor) {
  if (!(factor > 0.0)) throw ConfigError("lr bump factor must be positive");
  return lr * factor;
}

void refresh_edge_replicas(const EdgeLayers& edges, EdgeReplica& replica) {
  replica.embed = edges.embed;
  replica.deembed = edges.deembed;
  replica.staleness = 0;
}

void age_edge_replicas(EdgeReplica& replica) {
  if (replica.staleness >= 0) ++replica.staleness;
}

std::pair<ParameterVector, ParameterVector> recover_edge_stage(EdgeSide side, const ParameterVector& neighbor_weights,
                                                               const EdgeReplica& replica, StrategyKind active) {
  if (active != StrategyKind::CheckFreePlus)
    throw UnsupportedRecoveryError(std::string("first/last stage failure cannot be recovered by ") +
                                   to_string(active) + " (only checkfree-plus keeps edge replicas)");
  if (!replica.fresh()) throw ConfigError("edge replica is stale; refresh must precede recovery");
  return {neighbor_weights, side == EdgeSide::First ? replica.embed : replica.deembed};
}

ParameterVector reinit_copy(const ParameterVector& w_prev) { return w_prev; }

ParameterVector reinit_uniform_avg(const ParameterVector& w_prev, const ParameterVector& w_next) {
  return weighted(w_prev, w_next, 1.0, 1.0, nullptr);
}

ParameterVector reinit_random(const ModelSpec& spec, int stage_id, std::uint64_t seed) {
  StageState s;
  s.blocks = init_stage_blocks(spec, stage_id, seed);
  return s.flat_weights();
}

double reduction_error(const ParameterVector& w_prev, const ParameterVector& w_failed, const ParameterVector& w_next,
                       double omega_prev, double omega_next) {
  const ParameterVector r = recover_checkfree(w_prev, w_next, omega_prev, omega_next);
  if (!r.same_shape(w_failed)) throw ConfigError("failed stage weights differ in shape");
  return kernels::sum_squared_diff(r.ptr(), w_failed.ptr(), r.size());
}

// ---- checkpointing baseline: value-semantics snapshot (checkpoint.cpp:70-83) and the
//      "ckfree-ckpt v1" byte container (checkpoint.cpp:85-179), little-endian host
CheckpointSnapshot checkpoint_save(const ModelState& model, long iteration, std::uint64_t data_cursor) {
  return CheckpointSnapshot{iteration, data_cursor, model};
}

void checkpoint_restore(const CheckpointSnapshot& snapshot, ModelState& model, long& iteration,
                        std::uint64_t& data_cursor) {
  model = snapshot.model;
  iteration = snapshot.iteration;
  data_cursor = snapshot.data_cursor;
}

namespace {
const std::string kCkptHeader = "ckfree-ckpt v1\n";

class CkptWriter {
 public:
  void word(std::uint64_t v) {
    for (int i = 0; i < 8; ++i) bytes.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
  }
  void doubles(const double* p, std::size_t n) {  // length prefix, then the raw f64 bits
    word(n);
    for (std::size_t i = 0; i < n; ++i) {
      std::uint64_t b;
      std::memcpy(&b, p + i, 8);
      word(b);
    }
  }
  void doubles(const std::vector<double>& v) { doubles(v.data(), v.size()); }
  std::vector<std::uint8_t> bytes;
};

class CkptReader {
 public:
  explicit CkptReader(const std::vector<std::uint8_t>& b) : b_(b) {}
  std::uint64_t word() {
    if (at_ + 8 > b_.size()) throw ParseError("checkpoint: truncated integer");
    std::uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b_[at_ + static_cast<std::size_t>(i)];
    at_ += 8;
    return v;
  }
  std::vector<double> doubles(std::size_t expect) {
    const std::uint64_t n = word();
    if (n != expect)
      throw ParseError("checkpoint: array length " + std::to_string(n) + ", expected " + std::to_string(expect));
    std::vector<double> v(n);
    for (auto& x : v) {
      const std::uint64_t bits = word();
      std::memcpy(&x, &bits, 8);
    }
    return v;
  }
  bool done() const { return at_ == b_.size(); }
  std::size_t at_ = 0;

 private:
  const std::vector<std::uint8_t>& b_;
};
}  // namespace

std::vector<std::uint8_t> serialize_checkpoint(const CheckpointSnapshot& snapshot) {
  const ModelState& m = snapshot.model;
  CkptWriter w;
  w.bytes.assign(kCkptHeader.begin(), kCkptHeader.end());
  w.word(static_cast<std::uint64_t>(snapshot.iteration));
  const EdgeState& e = m.edges;
  w.doubles(e.layers.embed.values());
  w.doubles(e.opt_embed.m);
  w.doubles(e.opt_embed.v);
  w.doubles(e.layers.deembed.values());
  w.doubles(e.opt_deembed.m);
  w.doubles(e.opt_deembed.v);
  w.doubles(std::vector<double>{static_cast<double>(e.opt_embed.step), static_cast<double>(e.opt_deembed.step), e.lr});
  for (const StageState& st : m.stages) w.doubles(st.flat_weights().values());
  for (const StageState& st : m.stages) {
    w.doubles(st.opt.m);
    w.doubles(st.opt.v);
    w.doubles(std::vector<double>{static_cast<double>(st.opt.step), st.omega, st.lr});
  }
  w.word(snapshot.data_cursor);
  return std::move(w.bytes);
}

CheckpointSnapshot deserialize_checkpoint(const std::vector<std::uint8_t>& bytes, const ModelSpec& spec) {
  if (bytes.size() < kCkptHeader.size() || !std::equal(kCkptHeader.begin(), kCkptHeader.end(), bytes.begin()))
    throw ParseError("checkpoint: missing 'ckfree-ckpt v1' header");
  CkptReader r(bytes);
  r.at_ = kCkptHeader.size();
  CheckpointSnapshot snap;
  snap.iteration = static_cast<long>(r.word());
  ModelState& m = snap.model;
  m.spec = spec;
  EdgeState& e = m.edges;
  const std::size_t ne = spec.input_dim * spec.model_dim, nd = spec.model_dim * spec.output_dim;
  e.layers.embed = ParameterVector(r.doubles(ne), {spec.input_dim, spec.model_dim});
  e.opt_embed.m = r.doubles(ne);
  e.opt_embed.v = r.doubles(ne);
  e.layers.deembed = ParameterVector(r.doubles(nd), {spec.model_dim, spec.output_dim});
  e.opt_deembed.m = r.doubles(nd);
  e.opt_deembed.v = r.doubles(nd);
  const std::vector<double> es = r.doubles(3);
  e.opt_embed.step = static_cast<long>(es[0]);
  e.opt_deembed.step = static_cast<long>(es[1]);
  e.lr = es[2];
  m.stages.resize(spec.num_stages);
  for (std::size_t i = 0; i < spec.num_stages; ++i) {
    StageState& st = m.stages[i];
    st.stage_id = static_cast<int>(i + 1);
    st.blocks.resize(spec.stage_range(st.stage_id).count());
    for (ResidualBlock& b : st.blocks) {
      b.w1 = ParameterVector::zeros({spec.model_dim, spec.hidden_dim});
      b.w2 = ParameterVector::zeros({spec.hidden_dim, spec.model_dim});
    }
    const std::size_t n = st.param_count();
    st.set_flat_weights(ParameterVector(r.doubles(n), {n}));
  }
  for (StageState& st : m.stages) {
    st.opt.m = r.doubles(st.param_count());
    st.opt.v = r.doubles(st.param_count());
    const std::vector<double> sc = r.doubles(3);
    st.opt.step = static_cast<long>(sc[0]);
    st.omega = sc[1];
    st.lr = sc[2];
  }
  snap.data_cursor = r.word();
  if (!r.done()) throw ParseError("checkpoint: trailing bytes after data cursor");
  return snap;
}

void save_checkpoint_file(const CheckpointSnapshot& snapshot, const std::string& path) {
  const std::vector<std::uint8_t> b = serialize_checkpoint(snapshot);
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw ConfigError("cannot open '" + path + "' for writing");
  const std::size_t wrote = std::fwrite(b.data(), 1, b.size(), f);
  std::fclose(f);
  if (wrote != b.size()) throw ConfigError("short write to '" + path + "'");
}

CheckpointSnapshot load_checkpoint_file(const std::string& path, const ModelSpec& spec) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw ConfigError("cannot open checkpoint file '" + path + "'");
  std::vector<std::uint8_t> b;
  std::uint8_t buf[1 << 16];
  std::size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + got);
  std::fclose(f);
  return deserialize_checkpoint(b, spec);
}

}  // namespace ckfree::recovery

// ====================================================================== failures
namespace ckfree::failures {

namespace {
FailureTrace from_canonical(const std::string& text) {
  // "checkfree-trace v1 seed=S p_hour=P iter_s=I stages=a,b,..\n" then "iter,stage" lines
  FailureTrace t;
  std::istringstream in(text);
  std::string header;
  std::getline(in, header);
  std::istringstream h(header);
  std::string tok;
  while (h >> tok) {
    const auto eq = tok.find('=');
    if (eq == std::string::npos) continue;
    const std::string k = tok.substr(0, eq), v = tok.substr(eq + 1);
    if (k == "seed") t.spec.seed = std::stoull(v);
    else if (k == "p_hour") t.spec.p_hour = std::stod(v);
    else if (k == "iter_s") t.iteration_seconds = std::stod(v);
    else if (k == "stages") {
      std::istringstream sv(v);
      std::string s;
      while (std::getline(sv, s, ','))
        if (!s.empty()) t.spec.eligible_stages.push_back(std::stoi(s));
    }
  }
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    const auto c = line.find(',');
    t.events.push_back({std::stol(line.substr(0, c)), std::stoi(line.substr(c + 1))});
  }
  return t;
}
}  // namespace

void FailureRateSpec::validate() const {
  if (p_hour < 0.0 || p_hour >= 1.0) throw ConfigError("p_hour must lie in [0, 1)");
  for (int s : eligible_stages)
    if (s < 1) throw ConfigError("stage ids are 1-based");
}

void FailureTrace::validate() const {
  spec.validate();
  if (!(iteration_seconds > 0.0)) throw ConfigError("iteration_seconds must be positive");
  long last = 0;
  std::vector<std::pair<long, int>> seen;
  for (const FailureEvent& e : events) {
    if (e.iteration < 1) throw ConfigError("trace iterations are 1-based");
    if (e.iteration < last) throw ConfigError("trace events must be sorted by iteration");
    if (e.stage_id < 1) throw ConfigError("stage ids are 1-based");
    if (std::find(spec.eligible_stages.begin(), spec.eligible_stages.end(), e.stage_id) == spec.eligible_stages.end())
      throw ConfigError("trace event targets stage " + std::to_string(e.stage_id) + " outside the eligible set");
    const std::pair<long, int> key{e.iteration, e.stage_id};
    if (std::find(seen.begin(), seen.end(), key) != seen.end())
      throw ConfigError("duplicate event for stage " + std::to_string(e.stage_id) + " at iteration " +
                        std::to_string(e.iteration));
    seen.push_back(key);
    last = e.iteration;
  }
}

double hourly_to_per_iteration(double p_hour, double iteration_seconds) {
  return ckf_hourly_to_per_iteration(p_hour, iteration_seconds);
}

FailureTrace generate_trace(const FailureRateSpec& spec, long num_iterations, double iteration_seconds) {
  spec.validate();
  if (num_iterations < 0) throw ConfigError("iteration count must be non-negative");
  if (!(iteration_seconds > 0.0)) throw ConfigError("iteration_seconds must be positive");
  std::vector<char> buf(1 << 16);
  for (;;) {
    const int rc = ckf_generate_trace(spec.seed, spec.p_hour, iteration_seconds, num_iterations,
                                      spec.eligible_stages.data(), static_cast<int>(spec.eligible_stages.size()),
                                      buf.data(), buf.size());
    if (rc == CKF_E_USAGE && buf.size() < (1u << 30)) {
      buf.resize(buf.size() * 8);
      continue;
    }
    ck(rc);
    break;
  }
  FailureTrace t = from_canonical(buf.data());
  t.spec = spec;  // keep the caller's stage list verbatim
  t.iteration_seconds = iteration_seconds;
  return t;
}

std::string serialize_trace(const FailureTrace& trace) {
  std::ostringstream o;
  char num[64];
  o << "checkfree-trace v1 seed=" << trace.spec.seed;
  std::snprintf(num, sizeof num, "%.17g", trace.spec.p_hour);
  o << " p_hour=" << num;
  std::snprintf(num, sizeof num, "%.17g", trace.iteration_seconds);
  o << " iter_s=" << num << " stages=";
  for (size_t i = 0; i < trace.spec.eligible_stages.size(); ++i) o << (i ? "," : "") << trace.spec.eligible_stages[i];
  o << '\n';
  for (const FailureEvent& e : trace.events) o << e.iteration << ',' << e.stage_id << '\n';
  return o.str();
}

FailureTrace parse_trace(const std::string& text, const std::string& context_name) {
  std::vector<char> buf(text.size() * 2 + 4096);
  const int rc = ckf_parse_trace(text.c_str(), buf.data(), buf.size());
  if (rc == CKF_E_PARSE) throw ParseError(context_name + ": " + ckf_last_error());
  ck(rc);
  return from_canonical(buf.data());
}

void save_trace(const FailureTrace& trace, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw ConfigError("cannot write trace file '" + path + "'");
  f << serialize_trace(trace);
}

FailureTrace load_trace(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ConfigError("cannot read trace file '" + path + "'");
  const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return parse_trace(text, path);
}

std::vector<FailureEvent> consecutive_conflicts(const FailureTrace& trace) {
  std::vector<long> pairs(2 * trace.events.size() + 2);
  int n = 0;
  ck(ckf_consecutive_conflicts(serialize_trace(trace).c_str(), pairs.data(), static_cast<int>(pairs.size() / 2), &n));
  std::vector<FailureEvent> out;
  for (int i = 0; i < n; ++i) out.push_back({pairs[2 * i], static_cast<int>(pairs[2 * i + 1])});
  return out;
}

std::vector<int> intermediate_stages(int num_stages) {
  std::vector<int> v;
  for (int s = 2; s < num_stages; ++s) v.push_back(s);
  return v;
}

std::vector<int> all_stages(int num_stages) {
  std::vector<int> v;
  for (int s = 1; s <= num_stages; ++s) v.push_back(s);
  return v;
}

}  // namespace ckfree::failures
