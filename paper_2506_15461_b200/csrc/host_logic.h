// Host-side control logic shared by the engine's trainer and the C++ drop-in:
// failure traces, schedules, experiment configuration.  Pure C++ (no CUDA).
// Restates src/failures.cpp:57-196, src/pipeline.cpp:11-56 and
// src/experiment.cpp:34-115 bit-exactly (integer logic + host pow).
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace ckf::host {

struct HostError : std::runtime_error {
  int code;
  HostError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw HostError(code, m); }

inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t derive_key(uint64_t seed, uint64_t a = 0, uint64_t b = 0, uint64_t c = 0) {
  uint64_t h = mix64(seed ^ 0x6a09e667f3bcc909ULL);
  h = mix64(h ^ a);
  h = mix64(h ^ b);
  return mix64(h ^ c);
}
inline double to_unit(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
inline double unit_at(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
  return to_unit(derive_key(seed, a, b, c));
}

// ------------------------------------------------------------------ traces
struct Event {
  long iteration = 0;
  int stage = 0;
};
struct Trace {
  uint64_t seed = 0;
  double p_hour = 0.0;
  double iter_s = 3600.0;
  std::vector<int> stages;
  std::vector<Event> events;
};

double hourly_to_per_iteration(double p_hour, double iter_s);
Trace generate_trace(uint64_t seed, double p_hour, double iter_s, long n_iters, std::vector<int> stages);
std::string serialize_trace(const Trace& t);
Trace parse_trace(const std::string& text, const std::string& ctx = "<string>");
void validate_trace(const Trace& t);
std::vector<Event> consecutive_conflicts(const Trace& t);

// ------------------------------------------------------------------ schedules
std::vector<int> standard_order(int s);
std::vector<int> swapped_order(int s);
// m*s flattened orders; swapped at even positions (pipeline.cpp:41-56)
std::vector<int> build_schedule(int m, bool swapped_half, int s);

// ------------------------------------------------------------------ multi-GPU pipeline plan
// The global op sequence of one iteration for a stage -> rank placement, in
// the order every rank issues it (the engine's stage walk, engine.cu /
// *_block.cu): each microbatch enters at the embedding (owned with stage 1),
// visits the stages in its execution order, leaves through the de-embedding
// (owned with stage s), and the backward walks the applied stages in reverse.
// schedule 0 = forward+backward per microbatch, 1 = GPipe (all forwards, then
// all backwards in microbatch order).
struct PlanOp {
  enum Kind { kEmbedFwd = 0, kStageFwd = 1, kXfer = 2, kHead = 3, kStageBwd = 4, kEmbedBwd = 5 };
  int phase;  // 0 forward, 1 backward
  int mb;
  int kind;
  int rank;   // executing rank (kXfer: source)
  int arg;    // stage id (kStage*) or destination rank (kXfer)
  int aux;    // kXfer: 0 activations, 1 activation gradients
};
// schedule 2 = 1F1B: a list schedule simulated on the host (per rank: backward segments first,
// forward and backward segments each in microbatch order, at most `limit` microbatches in
// flight per rank) and flattened into ONE global order of ops and transfers that every rank
// issues its share of (see pipeline_plan in host_logic.cpp).  cost: forward time units per
// stage (index sid-1) and of the head (loss + head backward); the backward of a stage costs 2x.
struct PlanCost {
  std::vector<double> stage;
  double head = 1.0;
  double embed = 0.05;
};
std::vector<PlanOp> pipeline_plan(int s, int m, const std::vector<int>& orders, const std::vector<int>& stage_rank,
                                  int schedule, const PlanCost* cost = nullptr, int limit = 0);
// microbatches a rank can hold in flight under schedule 2 (activation cache slots): the number
// of pipeline ranks, at most m
int plan_inflight_limit(int m, const std::vector<int>& stage_rank);

// ------------------------------------------------------------------ config
struct Config {
  // model (model.hpp:32-42) + LLaMA extension
  std::string block = "mlp";
  std::string precision = "fp64";
  size_t input_dim = 16, hidden_dim = 64, model_dim = 32, output_dim = 16, layers = 8, stages = 4;
  size_t heads = 4, seq_len = 128;
  std::string activation = "tanh", task = "regression";
  // strategy (recovery.hpp:31-43)
  std::string strategy = "no-failures";
  long checkpoint_interval = 100;
  double lr_bump = 1.1;
  std::string recovered_moments = "fresh";
  // experiment (experiment.hpp:20-59)
  std::string trace_path;
  double p_hour = 0.0, p_iter = -1.0, iter_seconds = 120.0;
  std::string eligible = "auto";
  long iters = 2000;
  size_t batch = 256;
  int microbatches = 8;
  double lr = 3e-4;
  double target_loss = -1.0;
  long eval_interval = 25;
  size_t val_size = 1024;
  uint64_t seed = 1;
  std::string schedule = "auto";
  long swap_from = 0;
  int device = 0;

  static Config from_kv(const std::string& kv);
  void validate() const;
  bool swapped_schedule() const;
  bool neighbor_based() const;
  std::vector<int> resolved_eligible() const;
  Trace resolve_trace(uint64_t seed) const;
};

}  // namespace ckf::host
