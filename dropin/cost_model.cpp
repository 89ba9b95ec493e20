// Cost model of the drop-in (include/ckfree/cost_model.hpp).  Restates the reference's
// accounting (src/cost_model.cpp) -- the floating-point evaluation order is kept so that
// iteration/recovery/train times match the reference bit-for-bit (tests/test_cost_model.py)
// -- and adds the B200 profile / parameter constructors.
#include "ckfree/cost_model.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>

#include "ckfree/errors.hpp"

namespace ckfree::cost {

using recovery::StrategyConfig;
using recovery::StrategyKind;

namespace {

std::size_t site_of(const NetworkProfile& p, int stage) {
  return static_cast<std::size_t>(p.assignment[static_cast<std::size_t>(stage - 1)]);
}

// one message of `bytes` from stage a's site to stage b's site
double hop(const NetworkProfile& p, int a, int b, double bytes) { return p.link_latency(a, b) + bytes / p.link_bandwidth(a, b); }

template <class F>
void for_each_offdiag(const NetworkProfile& p, F&& f) {
  const std::size_t n = p.locations.size();
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j)
      if (i != j) f(i, j);
}

std::string g17(double v) {
  char b[48];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

void put_matrix(std::ostringstream& os, const Matrix& m) {
  for (std::size_t i = 0; i < m.rows; ++i) {
    for (std::size_t j = 0; j < m.cols; ++j) os << (j == 0 ? "" : " ") << g17(m.at(i, j));
    os << '\n';
  }
}

}  // namespace

// ------------------------------------------------------------------ NetworkProfile
void NetworkProfile::validate() const {  // cost_model.cpp:17-33
  const std::size_t n = locations.size();
  if (n == 0) throw ConfigError("network profile needs at least one location");
  const bool square = latency_s.rows == n && latency_s.cols == n && bandwidth_bps.rows == n && bandwidth_bps.cols == n;
  if (!square) throw ConfigError("latency/bandwidth matrices must be square over the locations");
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      if (latency_s.at(i, j) < 0.0) throw ConfigError("latencies must be nonnegative");
      if (i != j && !(bandwidth_bps.at(i, j) > 0.0)) throw ConfigError("bandwidths must be positive");
    }
  if (assignment.empty()) throw ConfigError("stage assignment must be total");
  if (std::any_of(assignment.begin(), assignment.end(), [n](int a) { return a < 0 || static_cast<std::size_t>(a) >= n; }))
    throw ConfigError("stage assigned to unknown location");
}

double NetworkProfile::link_latency(int a, int b) const { return latency_s.at(site_of(*this, a), site_of(*this, b)); }

double NetworkProfile::link_bandwidth(int a, int b) const {  // cost_model.cpp:40-47
  const std::size_t sa = site_of(*this, a), sb = site_of(*this, b);
  const double bw = bandwidth_bps.at(sa, sb);
  if (sa == sb && !(bw > 0.0)) return 1e12;  // co-located stages, no diagonal entry given
  return bw;
}

double NetworkProfile::storage_latency() const {
  double worst = 0.0;
  for_each_offdiag(*this, [&](std::size_t i, std::size_t j) { worst = std::max(worst, latency_s.at(i, j)); });
  return worst;
}

double NetworkProfile::storage_bandwidth() const {
  double slowest = -1.0;
  for_each_offdiag(*this, [&](std::size_t i, std::size_t j) {
    const double bw = bandwidth_bps.at(i, j);
    slowest = slowest < 0.0 ? bw : std::min(slowest, bw);
  });
  return slowest < 0.0 ? 1e12 : slowest;  // single site: storage is local
}

NetworkProfile NetworkProfile::synthetic_default(int num_stages) {  // cost_model.cpp:71-99
  // the reference's fixed 5-site WAN: one-way latency (ms) and link rate (Mb/s)
  static constexpr int kSites = 5;
  static const char* const names[kSites] = {"us-east", "eu-west", "asia-se", "us-west", "eu-north"};
  static constexpr double ms[kSites][kSites] = {
      {0, 80, 150, 60, 90}, {80, 0, 120, 110, 50}, {150, 120, 0, 130, 140}, {60, 110, 130, 0, 100}, {90, 50, 140, 100, 0}};
  static constexpr double mbit[kSites][kSites] = {{10000, 300, 100, 400, 250},
                                                  {300, 10000, 150, 200, 500},
                                                  {100, 150, 10000, 120, 140},
                                                  {400, 200, 120, 10000, 220},
                                                  {250, 500, 140, 220, 10000}};
  NetworkProfile p;
  p.locations.assign(names, names + kSites);
  p.latency_s = Matrix(kSites, kSites);
  p.bandwidth_bps = Matrix(kSites, kSites);
  for (int i = 0; i < kSites; ++i)
    for (int j = 0; j < kSites; ++j) {
      p.latency_s.at(i, j) = ms[i][j] / 1000.0;
      p.bandwidth_bps.at(i, j) = mbit[i][j] * 1e6 / 8.0;
    }
  for (int s = 0; s < num_stages; ++s) p.assignment.push_back(s % kSites);
  p.validate();
  return p;
}

NetworkProfile NetworkProfile::b200_cluster(int num_stages, int gpus_per_node, int nodes, const B200Links& l) {
  if (num_stages < 1 || gpus_per_node < 1 || nodes < 1) throw ConfigError("b200 profile needs positive sizes");
  const int gpus = gpus_per_node * nodes;
  const std::size_t n = static_cast<std::size_t>(gpus) + 1;  // + storage
  NetworkProfile p;
  for (int g = 0; g < gpus; ++g)
    p.locations.push_back("node" + std::to_string(g / gpus_per_node) + "-gpu" + std::to_string(g % gpus_per_node));
  p.locations.push_back("storage");
  p.latency_s = Matrix(n, n);
  p.bandwidth_bps = Matrix(n, n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      double lat, bw;
      if (i == j) {
        lat = 0.0, bw = l.hbm_bps;
      } else if (i == n - 1 || j == n - 1) {
        lat = l.storage_latency_s, bw = l.storage_bps;
      } else if (static_cast<int>(i) / gpus_per_node == static_cast<int>(j) / gpus_per_node) {
        lat = l.nvlink_latency_s, bw = l.nvlink_bps;
      } else {
        lat = l.nic_latency_s, bw = l.nic_bps;
      }
      p.latency_s.at(i, j) = lat;
      p.bandwidth_bps.at(i, j) = bw;
    }
  for (int s = 0; s < num_stages; ++s) p.assignment.push_back(s % gpus);
  p.validate();
  return p;
}

// "ckfree-net v1": header, `sites ...`, `assignment ...`, `latency` + n rows, `bandwidth` + n rows
std::string serialize_profile(const NetworkProfile& profile) {
  std::ostringstream os;
  os << "ckfree-net v1\nsites";
  for (const auto& s : profile.locations) os << ' ' << s;
  os << "\nassignment";
  for (int a : profile.assignment) os << ' ' << a;
  os << "\nlatency\n";
  put_matrix(os, profile.latency_s);
  os << "bandwidth\n";
  put_matrix(os, profile.bandwidth_bps);
  return os.str();
}

NetworkProfile parse_profile(const std::string& text, const std::string& ctx) {  // cost_model.cpp:133-190
  std::istringstream in(text);
  std::string line;
  std::size_t no = 0;
  auto where = [&] { return ctx + ":" + std::to_string(no) + ": "; };
  auto next = [&](const std::string& what) {
    if (!std::getline(in, line)) throw ParseError(ctx + ": unexpected end of file, expected " + what);
    ++no;
  };
  auto keyword_line = [&](const std::string& kw) {  // "<kw> tok tok ..." -> stream positioned after kw
    next(kw == "sites" ? "site list" : kw);
    auto ls = std::make_unique<std::istringstream>(line);
    std::string head;
    *ls >> head;
    if (head != kw) throw ParseError(where() + "expected '" + kw + "'");
    return ls;
  };

  next("header");
  if (line != "ckfree-net v1") throw ParseError(ctx + ":1: expected header 'ckfree-net v1'");
  NetworkProfile p;
  {
    auto ls = keyword_line("sites");
    for (std::string s; *ls >> s;) p.locations.push_back(s);
  }
  {
    auto ls = keyword_line("assignment");
    for (int a; *ls >> a;) p.assignment.push_back(a);
  }
  const std::size_t n = p.locations.size();
  auto matrix = [&](const std::string& name) {
    next(name);
    if (line != name) throw ParseError(where() + "expected '" + name + "'");
    Matrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) {
      next("matrix row");
      std::istringstream ls(line);
      for (std::size_t j = 0; j < n; ++j)
        if (!(ls >> m.at(i, j))) throw ParseError(where() + "expected " + std::to_string(n) + " values");
    }
    return m;
  };
  p.latency_s = matrix("latency");
  p.bandwidth_bps = matrix("bandwidth");
  try {
    p.validate();
  } catch (const ConfigError& e) {
    throw ParseError(ctx + ": " + e.what());
  }
  return p;
}

void save_profile(const NetworkProfile& profile, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw ConfigError("cannot open '" + path + "' for writing");
  f << serialize_profile(profile);
}

NetworkProfile load_profile(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ConfigError("cannot open profile '" + path + "'");
  std::stringstream ss;
  ss << f.rdbuf();
  return parse_profile(ss.str(), path);
}

// ------------------------------------------------------------------ CostParams
void CostParams::validate() const {  // cost_model.cpp:198-208
  if (!(fwd_seconds > 0.0) || !(bwd_seconds > 0.0)) throw ConfigError("compute seconds must be positive");
  if (bwd_seconds < fwd_seconds) throw ConfigError("backward must cost at least as much as forward");
  if (!activation_bytes || !stage_weight_bytes || !edge_weight_bytes || !full_model_bytes)
    throw ConfigError("message sizes must be positive");
  if (num_microbatches < 1) throw ConfigError("microbatch count must be positive");
  if (edge_weight_bytes >= stage_weight_bytes)
    std::cerr << "warning: edge layers are not smaller than a stage (" << edge_weight_bytes << " >= "
              << stage_weight_bytes << " bytes); replica overhead will be significant\n";
}

CostParams CostParams::from_model(const ModelSpec& spec, std::size_t batch_size, int num_microbatches,
                                  double fwd_seconds, double bwd_seconds) {  // cost_model.cpp:210-232
  constexpr std::size_t f64 = sizeof(double);
  const std::size_t per_block = spec.model_dim * spec.hidden_dim * 2;  // w1 + w2
  std::size_t largest = 0, blocks_total = 0;
  for (std::size_t s = 0; s < spec.num_stages; ++s) {
    const std::size_t params = spec.partition[s].count() * per_block;
    largest = std::max(largest, params);
    blocks_total += params;
  }
  const std::size_t embed = spec.input_dim * spec.model_dim, deembed = spec.model_dim * spec.output_dim;
  CostParams p;
  p.fwd_seconds = fwd_seconds;
  p.bwd_seconds = bwd_seconds;
  p.num_microbatches = num_microbatches;
  p.activation_bytes = batch_size / static_cast<std::size_t>(num_microbatches) * spec.model_dim * f64;
  p.stage_weight_bytes = largest * f64;
  p.edge_weight_bytes = std::max(embed, deembed) * f64;
  p.full_model_bytes = (blocks_total + embed + deembed) * 3 * f64;  // weights + two Adam moments
  return p;
}

CostParams CostParams::from_b200(double fwd_seconds, double bwd_seconds, std::uint64_t tokens_per_microbatch,
                                 std::size_t model_dim, std::uint64_t stage_params, std::uint64_t edge_params,
                                 std::uint64_t total_params, int num_microbatches) {
  CostParams p;
  p.fwd_seconds = fwd_seconds;
  p.bwd_seconds = bwd_seconds;
  p.num_microbatches = num_microbatches;
  p.activation_bytes = tokens_per_microbatch * model_dim * 2;  // bf16 hidden state per boundary hop
  p.stage_weight_bytes = stage_params * 4;                     // fp32 masters
  p.edge_weight_bytes = edge_params * 4;
  p.full_model_bytes = total_params * 12;  // fp32 masters + Adam m + v
  p.validate();
  return p;
}

// ------------------------------------------------------------------ accounting
IterationCost iteration_cost(const StrategyConfig& strategy, const NetworkProfile& profile, const CostParams& params) {
  profile.validate();
  params.validate();
  strategy.validate();
  const int s = profile.num_stages();
  const StrategyKind k = strategy.kind;
  const bool rc = k == StrategyKind::RedundantComputation;

  // RC (cost_model.cpp:244-253): microbatches halved in size and doubled in count to make
  // room for the hosted copy; every stage also runs the copy's forward
  const int mb = params.num_microbatches * (rc ? 2 : 1);
  const double f = rc ? params.fwd_seconds / 2.0 : params.fwd_seconds;
  const double b = rc ? params.bwd_seconds / 2.0 : params.bwd_seconds;
  const double act = rc ? static_cast<double>(params.activation_bytes) / 2.0 : static_cast<double>(params.activation_bytes);
  const double stage_step = rc ? 2.0 * f + b : f + b;

  IterationCost c;
  c.compute = static_cast<double>(mb) * static_cast<double>(s) * stage_step;
  for (int i = 1; i < s; ++i) c.communication += static_cast<double>(mb) * hop(profile, i, i + 1, act);

  if (k == StrategyKind::CheckFreePlus && s >= 2) {  // embedding -> stage 2, de-embedding -> stage s-1
    const double e = static_cast<double>(params.edge_weight_bytes);
    c.communication += hop(profile, 1, 2, e);
    c.communication += hop(profile, s, s - 1, e);
  }
  if (rc) {  // each stage refreshes its copy on the ring predecessor (stage 1's on stage s)
    const double w = static_cast<double>(params.stage_weight_bytes);
    for (int i = 1; i <= s; ++i) c.communication += hop(profile, i, i == 1 ? s : i - 1, w);
  }
  if (k == StrategyKind::Checkpointing) {
    const double upload = static_cast<double>(params.full_model_bytes) / profile.storage_bandwidth();
    const double every = static_cast<double>(strategy.checkpoint_interval);
    c.checkpoint_overhead =
        (strategy.blocking_checkpoint_upload ? profile.storage_latency() + upload : upload) / every;
  }
  return c;
}

double iteration_time(const StrategyConfig& strategy, const NetworkProfile& profile, const CostParams& params) {
  return iteration_cost(strategy, profile, params).total();
}

double recovery_time(const StrategyConfig& strategy, const NetworkProfile& profile, const CostParams& params,
                     int failed_stage) {  // cost_model.cpp:290-340
  const int s = profile.num_stages();
  const int f = failed_stage;
  if (f < 1 || f > s) throw ConfigError("failed stage out of range");
  const double w = static_cast<double>(params.stage_weight_bytes);
  const bool edge = f == 1 || f == s;
  // both neighbours stream their stage to the replacement at once; the omegas ride along
  auto from_both = [&] { return std::max(hop(profile, f - 1, f, w), hop(profile, f + 1, f, w)); };

  switch (strategy.kind) {
    case StrategyKind::NoFailures:
      return 0.0;
    case StrategyKind::ReinitRandom:
      if (edge) throw UnsupportedRecoveryError("random reinitialization covers intermediate stages only");
      return 0.0;
    case StrategyKind::ReinitCopy:
      if (edge) throw UnsupportedRecoveryError("copy reinitialization covers intermediate stages only");
      return hop(profile, f - 1, f, w);
    case StrategyKind::ReinitUniformAvg:
    case StrategyKind::CheckFree:
      if (edge) throw UnsupportedRecoveryError("neighbor averaging cannot recover the first or last stage");
      return from_both();
    case StrategyKind::CheckFreePlus:
      if (!edge) return from_both();
      // the surviving neighbour sends its stage (the swapped-order copy) plus the edge-layer replica
      return hop(profile, f == 1 ? 2 : s - 1, f, w + static_cast<double>(params.edge_weight_bytes));
    case StrategyKind::RedundantComputation:
      return hop(profile, f == 1 ? s : f - 1, f, w);
    case StrategyKind::Checkpointing:
      return profile.storage_latency() + static_cast<double>(params.full_model_bytes) / profile.storage_bandwidth();
  }
  return 0.0;
}

TrainTime train_time(long iterations_to_target, const IterationCost& per_iteration,
                     const std::vector<failures::FailureEvent>& events, const StrategyConfig& strategy,
                     const NetworkProfile& profile, const CostParams& params) {  // cost_model.cpp:342-383
  if (iterations_to_target < 0) throw ConfigError("iterations_to_target must be nonnegative");
  TrainTime t;
  const double n = static_cast<double>(iterations_to_target);
  t.breakdown.compute = n * per_iteration.compute;
  t.breakdown.communication = n * per_iteration.communication;
  t.breakdown.checkpoint_overhead = n * per_iteration.checkpoint_overhead;
  for (const auto& e : events) t.breakdown.recovery += recovery_time(strategy, profile, params, e.stage_id);

  if (strategy.kind == StrategyKind::Checkpointing) {
    // replay the trainer: a snapshot every `interval` model iterations; each failing slot
    // (however many stages fail in it) rolls back to the last snapshot once
    const long every = strategy.checkpoint_interval;
    long model_iter = 0, last_slot = 0, lost = 0;
    for (std::size_t i = 0; i < events.size();) {
      const long slot = events[i].iteration;
      model_iter += slot - last_slot;
      last_slot = slot;
      const long snapshot = model_iter / every * every;
      lost += model_iter - snapshot;
      model_iter = snapshot;
      while (i < events.size() && events[i].iteration == slot) ++i;
    }
    t.breakdown.rollback_lost = static_cast<double>(lost) * per_iteration.total();
  }
  t.hours = t.breakdown.total() / 3600.0;
  return t;
}

}  // namespace ckfree::cost

// ------------------------------------------------------------------ C entry points
namespace {

thread_local std::string g_cost_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ckfree::ParseError& e) {
    g_cost_error = e.what();
    return 2;
  } catch (const ckfree::UnsupportedRecoveryError& e) {
    g_cost_error = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_cost_error = e.what();
    return 1;
  }
}

ckfree::cost::CostParams unpack(const double* v) {
  ckfree::cost::CostParams p;
  p.fwd_seconds = v[0];
  p.bwd_seconds = v[1];
  p.activation_bytes = static_cast<std::uint64_t>(v[2]);
  p.stage_weight_bytes = static_cast<std::uint64_t>(v[3]);
  p.edge_weight_bytes = static_cast<std::uint64_t>(v[4]);
  p.full_model_bytes = static_cast<std::uint64_t>(v[5]);
  p.num_microbatches = static_cast<int>(v[6]);
  return p;
}

ckfree::recovery::StrategyConfig strategy_of(const char* name, long interval, int blocking) {
  ckfree::recovery::StrategyConfig s;
  s.kind = ckfree::recovery::parse_strategy(name);
  s.checkpoint_interval = interval;
  s.blocking_checkpoint_upload = blocking != 0;
  return s;
}

void copy_out(const std::string& text, char* out, std::size_t cap) {
  if (text.size() + 1 > cap) throw ckfree::ConfigError("output buffer too small for the profile text");
  std::memcpy(out, text.c_str(), text.size() + 1);
}

}  // namespace

extern "C" {

const char* ckfree_cost_last_error() { return g_cost_error.c_str(); }

int ckfree_cost_profile_synthetic(int num_stages, char* out, std::size_t cap) {
  return guarded([&] { copy_out(serialize_profile(ckfree::cost::NetworkProfile::synthetic_default(num_stages)), out, cap); });
}

int ckfree_cost_profile_b200(int num_stages, int gpus_per_node, int nodes, const double* links, char* out,
                             std::size_t cap) {
  return guarded([&] {
    ckfree::cost::NetworkProfile::B200Links l;
    if (links) {
      l.nvlink_bps = links[0], l.nvlink_latency_s = links[1], l.nic_bps = links[2], l.nic_latency_s = links[3];
      l.hbm_bps = links[4], l.storage_bps = links[5], l.storage_latency_s = links[6];
    }
    copy_out(serialize_profile(ckfree::cost::NetworkProfile::b200_cluster(num_stages, gpus_per_node, nodes, l)), out,
             cap);
  });
}

int ckfree_cost_params_b200(double fwd_seconds, double bwd_seconds, std::uint64_t tokens_per_microbatch,
                            std::size_t model_dim, std::uint64_t stage_params, std::uint64_t edge_params,
                            std::uint64_t total_params, int num_microbatches, double* out7) {
  return guarded([&] {
    const auto p = ckfree::cost::CostParams::from_b200(fwd_seconds, bwd_seconds, tokens_per_microbatch, model_dim,
                                                       stage_params, edge_params, total_params, num_microbatches);
    out7[0] = p.fwd_seconds, out7[1] = p.bwd_seconds, out7[2] = static_cast<double>(p.activation_bytes);
    out7[3] = static_cast<double>(p.stage_weight_bytes), out7[4] = static_cast<double>(p.edge_weight_bytes);
    out7[5] = static_cast<double>(p.full_model_bytes), out7[6] = p.num_microbatches;
  });
}

int ckfree_cost_iteration(const char* strategy, long interval, int blocking, const char* profile_text,
                          const double* params, double* out3) {
  return guarded([&] {
    const auto c = ckfree::cost::iteration_cost(strategy_of(strategy, interval, blocking),
                                                ckfree::cost::parse_profile(profile_text), unpack(params));
    out3[0] = c.compute, out3[1] = c.communication, out3[2] = c.checkpoint_overhead;
  });
}

int ckfree_cost_recovery(const char* strategy, long interval, const char* profile_text, const double* params,
                         int failed_stage, double* out) {
  return guarded([&] {
    *out = ckfree::cost::recovery_time(strategy_of(strategy, interval, 0), ckfree::cost::parse_profile(profile_text),
                                       unpack(params), failed_stage);
  });
}

int ckfree_cost_train(const char* strategy, long interval, int blocking, const char* profile_text, const double* params,
                      long iterations_to_target, const long* event_iter, const int* event_stage, int n_events,
                      double* out6) {
  return guarded([&] {
    const auto sc = strategy_of(strategy, interval, blocking);
    const auto prof = ckfree::cost::parse_profile(profile_text);
    const auto par = unpack(params);
    std::vector<ckfree::failures::FailureEvent> ev(static_cast<std::size_t>(std::max(0, n_events)));
    for (std::size_t i = 0; i < ev.size(); ++i) ev[i] = {event_iter[i], event_stage[i]};
    const auto t = ckfree::cost::train_time(iterations_to_target, ckfree::cost::iteration_cost(sc, prof, par), ev, sc,
                                            prof, par);
    const auto& b = t.breakdown;
    out6[0] = b.compute, out6[1] = b.communication, out6[2] = b.checkpoint_overhead, out6[3] = b.recovery,
    out6[4] = b.rollback_lost, out6[5] = t.hours;
  });
}

}  // extern "C"
