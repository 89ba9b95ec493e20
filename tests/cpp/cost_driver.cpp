// Cost-model compatibility driver (test infrastructure).  Compiled twice from this one
// source: against the reference library (oracle/_ref/cost_driver_ref) and against the B200
// drop-in (dropin/_bin/cost_driver_dropin).  Both print every quantity of the reference's
// cost API (include/ckfree/cost_model.hpp) as exact hex floats over a grid of profiles,
// parameter sets, strategies, failed stages and failure-event lists; tests/test_cost_model.py
// requires the two outputs to be identical.
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "ckfree/cost_model.hpp"
#include "ckfree/errors.hpp"
#include "ckfree/failures.hpp"
#include "ckfree/model.hpp"
#include "ckfree/recovery.hpp"

using namespace ckfree;
using recovery::StrategyKind;

namespace {

const StrategyKind kKinds[] = {StrategyKind::NoFailures,   StrategyKind::Checkpointing,
                               StrategyKind::RedundantComputation, StrategyKind::CheckFree,
                               StrategyKind::CheckFreePlus, StrategyKind::ReinitRandom,
                               StrategyKind::ReinitCopy,   StrategyKind::ReinitUniformAvg};

unsigned long fnv(const std::string& s) {
  unsigned long h = 1469598103934665603ul;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ul;
  return h;
}

// a 3-site profile with two stages on one site and a zero diagonal bandwidth (the
// co-located 1e12 path of link_bandwidth)
cost::NetworkProfile colocated(int stages) {
  std::string t = "ckfree-net v1\nsites a b c\nassignment";
  for (int s = 0; s < stages; ++s) t += " " + std::to_string(s % 2 == 0 ? 0 : (s % 3 == 1 ? 1 : 2));
  t += "\nlatency\n0 0.002 0.03\n0.002 0.001 0.05\n0.03 0.05 0\n";
  t += "bandwidth\n0 2.5e9 1.25e8\n2.5e9 4e10 6e7\n1.25e8 6e7 0\n";
  return cost::parse_profile(t, "colocated");
}

void dump(const char* tag, const cost::NetworkProfile& prof, const cost::CostParams& par) {
  const int s = prof.num_stages();
  std::printf("== %s stages=%d profile=%016lx storage=%a/%a\n", tag, s, fnv(cost::serialize_profile(prof)),
              prof.storage_latency(), prof.storage_bandwidth());
  // deterministic failure lists: none, singles, a repeated slot, multi-stage slots
  std::vector<std::vector<failures::FailureEvent>> lists = {{}, {{5, 2}}, {{3, 2}, {3, 3}, {40, 2}, {41, s - 1}}};
  std::vector<failures::FailureEvent> many;
  for (long it = 7; it < 2000; it += 37 + it % 11) many.push_back({it, 2 + static_cast<int>(it % (s > 2 ? s - 2 : 1))});
  lists.push_back(many);
  std::vector<failures::FailureEvent> with_edges = {{2, 1}, {9, s}, {9, 2}, {150, 1}};
  lists.push_back(with_edges);

  for (StrategyKind k : kKinds)
    for (long interval : {1L, 10L, 100L})
      for (bool blocking : {false, true}) {
        if (k != StrategyKind::Checkpointing && (interval != 100 || blocking)) continue;
        recovery::StrategyConfig sc;
        sc.kind = k;
        sc.checkpoint_interval = interval;
        sc.blocking_checkpoint_upload = blocking;
        const cost::IterationCost c = cost::iteration_cost(sc, prof, par);
        std::printf("%s/%ld/%d iter %a %a %a total %a time %a\n", recovery::to_string(k), interval, blocking ? 1 : 0,
                    c.compute, c.communication, c.checkpoint_overhead, c.total(), cost::iteration_time(sc, prof, par));
        std::printf("  recovery");
        for (int f = 0; f <= s + 1; ++f) {
          try {
            std::printf(" %a", cost::recovery_time(sc, prof, par, f));
          } catch (const UnsupportedRecoveryError&) {
            std::printf(" unsupported");
          } catch (const ConfigError&) {
            std::printf(" config");
          }
        }
        std::printf("\n");
        for (std::size_t li = 0; li < lists.size(); ++li)
          for (long iters : {0L, 100L, 12345L}) {
            try {
              const cost::TrainTime t = cost::train_time(iters, c, lists[li], sc, prof, par);
              const auto& b = t.breakdown;
              std::printf("  train[%zu,%ld] %a | %a %a %a %a %a\n", li, iters, t.hours, b.compute, b.communication,
                          b.checkpoint_overhead, b.recovery, b.rollback_lost);
            } catch (const UnsupportedRecoveryError&) {
              std::printf("  train[%zu,%ld] unsupported\n", li, iters);
            }
          }
      }
}

}  // namespace

int main() {
  // CostParams::from_model over a reference-style spec, plus hand-set parameters
  ModelSpec spec;
  spec.input_dim = 40;
  spec.hidden_dim = 96;
  spec.model_dim = 48;
  spec.output_dim = 24;
  spec.num_layers = 12;
  spec.num_stages = 6;
  spec.partition = ModelSpec::even_partition(spec.num_layers, spec.num_stages);
  spec.finalize();
  const cost::CostParams fm = cost::CostParams::from_model(spec, 256, 8, 0.35, 0.8);
  std::printf("from_model fwd=%a bwd=%a act=%llu stage=%llu edge=%llu full=%llu mb=%d\n", fm.fwd_seconds,
              fm.bwd_seconds, (unsigned long long)fm.activation_bytes, (unsigned long long)fm.stage_weight_bytes,
              (unsigned long long)fm.edge_weight_bytes, (unsigned long long)fm.full_model_bytes, fm.num_microbatches);
  cost::CostParams big;
  big.fwd_seconds = 0.0123;
  big.bwd_seconds = 0.0311;
  big.activation_bytes = 3ull << 24;
  big.stage_weight_bytes = 7ull << 28;
  big.edge_weight_bytes = 5ull << 26;
  big.full_model_bytes = 9ull << 32;
  big.num_microbatches = 24;

  for (int s : {3, 4, 6, 8}) {
    const cost::NetworkProfile syn = cost::NetworkProfile::synthetic_default(s);
    // serialize -> parse -> serialize is a fixed point
    const std::string text = cost::serialize_profile(syn);
    std::printf("roundtrip %d %d\n", s, cost::serialize_profile(cost::parse_profile(text)) == text ? 1 : 0);
    dump("synthetic/from_model", syn, fm);
    dump("synthetic/big", syn, big);
    dump("colocated/big", colocated(s), big);
  }
  std::printf("synthetic6 %s", cost::serialize_profile(cost::NetworkProfile::synthetic_default(6)).c_str());

  // parse errors (error class only: messages are free text)
  const char* bad[] = {"",
                       "ckfree-net v2\n",
                       "ckfree-net v1\nsite a\n",
                       "ckfree-net v1\nsites a b\nassignment 0 1\nlatency\n0 1\n",
                       "ckfree-net v1\nsites a b\nassignment 0 1\nlatency\n0 1\n1 0\nbandwidth\n0 -1\n1 0\n",
                       "ckfree-net v1\nsites a b\nassignment 0 2\nlatency\n0 1\n1 0\nbandwidth\n0 1\n1 0\n",
                       "ckfree-net v1\nsites a b\nassignment\nlatency\n0 1\n1 0\nbandwidth\n0 1\n1 0\n"};
  for (const char* t : bad) {
    try {
      cost::parse_profile(t, "bad");
      std::printf("parse ok\n");
    } catch (const ParseError&) {
      std::printf("parse ParseError\n");
    } catch (const std::exception&) {
      std::printf("parse other\n");
    }
  }
  // invalid parameters
  cost::CostParams p = big;
  p.bwd_seconds = p.fwd_seconds / 2;
  recovery::StrategyConfig cf;
  cf.kind = StrategyKind::CheckFree;
  try {
    cost::iteration_cost(cf, cost::NetworkProfile::synthetic_default(4), p);
    std::printf("params ok\n");
  } catch (const ConfigError&) {
    std::printf("params ConfigError\n");
  }
  try {
    cost::train_time(-1, cost::IterationCost{}, {}, cf, cost::NetworkProfile::synthetic_default(4), big);
    std::printf("train ok\n");
  } catch (const ConfigError&) {
    std::printf("train ConfigError\n");
  }
  return 0;
}
