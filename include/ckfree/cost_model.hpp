// Wall-clock cost model of the drop-in (reference include/ckfree/cost_model.hpp:13-113,
// src/cost_model.cpp).  Same types, entry points, text format ("ckfree-net v1") and
// arithmetic as the reference -- tests/test_cost_model.py checks the outputs byte-for-byte
// against the reference compiled from source -- plus the B200 re-parameterisation:
//
//   * NetworkProfile::b200_cluster   -- stages placed on B200 GPUs joined by NVLink 5 /
//                                       NVSwitch inside a node and by the scale-out NIC
//                                       between nodes, checkpoints going to host storage;
//   * CostParams::from_b200          -- per-stage per-microbatch forward/backward seconds
//                                       MEASURED on the B200 engine and message sizes of the
//                                       B200 data layout (bf16 boundary activations, fp32
//                                       master weights, fp32 Adam moments).
//
// The model is host arithmetic (no device work); it lives in libckfree_b200.so next to the
// rest of the reference-facing C++ API and is exported to Python through the extern "C"
// ckfree_cost_* entry points at the bottom of this header (paper_2506_15461_b200/cost.py).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "ckfree/failures.hpp"
#include "ckfree/matrix.hpp"
#include "ckfree/model.hpp"
#include "ckfree/recovery.hpp"

namespace ckfree::cost {

// Sites with a square latency (s) / bandwidth (B/s) matrix and the stage -> site map
// (cost_model.hpp:16-34).
struct NetworkProfile {
  std::vector<std::string> locations;
  Matrix latency_s;
  Matrix bandwidth_bps;
  std::vector<int> assignment;  // stage id - 1 -> location index

  int num_stages() const { return static_cast<int>(assignment.size()); }
  void validate() const;

  double link_latency(int stage_a, int stage_b) const;
  double link_bandwidth(int stage_a, int stage_b) const;
  // worst off-diagonal path: where checkpoint uploads and restores go
  double storage_latency() const;
  double storage_bandwidth() const;

  // the reference's 5-site WAN profile (50-150 ms, 100-500 Mb/s), stages round-robin
  static NetworkProfile synthetic_default(int num_stages);

  // B200 deployment: `nodes` nodes of `gpus_per_node` GPUs plus one "storage" site.
  // Stage s runs on GPU (s-1) % (nodes*gpus_per_node), filling node 0 first.  GPU<->GPU
  // inside a node: NVLink 5 through NVSwitch (every pair at full per-direction bandwidth);
  // across nodes: the scale-out NIC; GPU<->storage: the host path checkpoints take.
  // A GPU to itself (co-located stages) uses the HBM copy bandwidth.
  struct B200Links {
    double nvlink_bps = 900e9;        // per direction, NVLink 5 via NVSwitch (nominal)
    double nvlink_latency_s = 3e-6;   // one NCCL p2p send at small size
    double nic_bps = 50e9;            // 400 Gb/s per GPU scale-out (nominal)
    double nic_latency_s = 10e-6;
    double hbm_bps = 7.7e12;          // same-GPU copy (override with MEASURED_PEAKS.json)
    double storage_bps = 25e9;        // checkpoint path GPU -> host -> storage
    double storage_latency_s = 1e-3;
  };
  static NetworkProfile b200_cluster(int num_stages, int gpus_per_node, int nodes, const B200Links& links);
  static NetworkProfile b200_cluster(int num_stages, int gpus_per_node = 8, int nodes = 1) {
    return b200_cluster(num_stages, gpus_per_node, nodes, B200Links{});
  }
};

std::string serialize_profile(const NetworkProfile& profile);
NetworkProfile parse_profile(const std::string& text, const std::string& context_name = "<string>");
void save_profile(const NetworkProfile& profile, const std::string& path);
NetworkProfile load_profile(const std::string& path);

// Per-stage compute seconds and message sizes (cost_model.hpp:38-53).
struct CostParams {
  double fwd_seconds = 1.0;  // per stage per microbatch
  double bwd_seconds = 2.0;  // per stage per microbatch, >= fwd_seconds
  std::uint64_t activation_bytes = 1 << 16;
  std::uint64_t stage_weight_bytes = 1 << 20;
  std::uint64_t edge_weight_bytes = 1 << 14;
  std::uint64_t full_model_bytes = 1 << 22;
  int num_microbatches = 8;

  void validate() const;  // warns on stderr when the edge layers are not smaller than a stage
  // reference sizing for its fp64 residual-MLP stages
  static CostParams from_model(const ModelSpec& spec, std::size_t batch_size, int num_microbatches,
                               double fwd_seconds, double bwd_seconds);
  // B200 sizing: tokens_per_microbatch x model_dim bf16 activations cross each boundary;
  // recovery ships fp32 masters (stage_params x 4 B, edge_params x 4 B); a checkpoint holds
  // masters + both Adam moments (total_params x 12 B).  fwd/bwd seconds are the engine's
  // measured per-stage per-microbatch times.
  static CostParams from_b200(double fwd_seconds, double bwd_seconds, std::uint64_t tokens_per_microbatch,
                              std::size_t model_dim, std::uint64_t stage_params, std::uint64_t edge_params,
                              std::uint64_t total_params, int num_microbatches);
};

struct IterationCost {
  double compute = 0.0;
  double communication = 0.0;
  double checkpoint_overhead = 0.0;
  double total() const { return compute + communication + checkpoint_overhead; }
};

// cost_model.hpp:62-71: serialized compute chain + one activation hop per boundary per
// microbatch + strategy extras (CF+ edge-replica refresh, RC ring weight refresh,
// amortised checkpoint upload).
IterationCost iteration_cost(const recovery::StrategyConfig& strategy, const NetworkProfile& profile,
                             const CostParams& params);
double iteration_time(const recovery::StrategyConfig& strategy, const NetworkProfile& profile,
                      const CostParams& params);

// cost_model.hpp:73-75: seconds to provision a replacement for failed_stage
double recovery_time(const recovery::StrategyConfig& strategy, const NetworkProfile& profile,
                     const CostParams& params, int failed_stage);

struct TimeBreakdown {
  double compute = 0.0;
  double communication = 0.0;
  double checkpoint_overhead = 0.0;
  double recovery = 0.0;
  double rollback_lost = 0.0;
  double total() const { return compute + communication + checkpoint_overhead + recovery + rollback_lost; }
};

struct TrainTime {
  double hours = 0.0;
  TimeBreakdown breakdown;
};

// cost_model.hpp:91-98: productive iterations + per-event recovery + (checkpointing)
// iterations replayed after each rollback, one rollback per failing iteration
TrainTime train_time(long iterations_to_target, const IterationCost& per_iteration,
                     const std::vector<failures::FailureEvent>& events, const recovery::StrategyConfig& strategy,
                     const NetworkProfile& profile, const CostParams& params);

}  // namespace ckfree::cost

// ---- C entry points for the Python face (paper_2506_15461_b200/cost.py) --------------
// Every function returns 0 on success, else the CKF_E_* class of the C++ exception
// (1 config, 2 parse, 3 unsupported recovery) with the message in ckfree_cost_last_error().
// `params` is {fwd_s, bwd_s, activation_B, stage_weight_B, edge_weight_B, full_model_B,
// num_microbatches}; `strategy` is the reference's strategy name.
extern "C" {
const char* ckfree_cost_last_error();
int ckfree_cost_profile_synthetic(int num_stages, char* out, std::size_t cap);
// links = {nvlink_bps, nvlink_latency_s, nic_bps, nic_latency_s, hbm_bps, storage_bps, storage_latency_s}
int ckfree_cost_profile_b200(int num_stages, int gpus_per_node, int nodes, const double* links, char* out,
                             std::size_t cap);
// out7 = CostParams::from_b200(...) packed like `params`
int ckfree_cost_params_b200(double fwd_seconds, double bwd_seconds, std::uint64_t tokens_per_microbatch,
                            std::size_t model_dim, std::uint64_t stage_params, std::uint64_t edge_params,
                            std::uint64_t total_params, int num_microbatches, double* out7);
int ckfree_cost_iteration(const char* strategy, long checkpoint_interval, int blocking_upload,
                          const char* profile_text, const double* params, double* out3);
int ckfree_cost_recovery(const char* strategy, long checkpoint_interval, const char* profile_text,
                         const double* params, int failed_stage, double* out);
// out6 = {compute, communication, checkpoint_overhead, recovery, rollback_lost, hours}
int ckfree_cost_train(const char* strategy, long checkpoint_interval, int blocking_upload, const char* profile_text,
                      const double* params, long iterations_to_target, const long* event_iter,
                      const int* event_stage, int n_events, double* out6);
}
