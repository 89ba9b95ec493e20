// Checkpoint container compatibility driver (test infrastructure).  Compiled twice from
// this one source: against the reference library (oracle/_ref/ckpt_roundtrip_ref) and
// against the B200 drop-in (dropin/_bin/ckpt_roundtrip_dropin).  Both print the byte
// size and an FNV-1a digest of serialize_checkpoint() for the same model state, and
// check that deserialize -> serialize reproduces the bytes (reference recovery.hpp:88-108).
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "ckfree/model.hpp"
#include "ckfree/recovery.hpp"

using namespace ckfree;

int main(int argc, char** argv) {
  ModelSpec spec;
  spec.input_dim = 16;
  spec.hidden_dim = 24;
  spec.model_dim = 12;
  spec.output_dim = 8;
  spec.num_layers = 6;
  spec.num_stages = 3;
  spec.partition = ModelSpec::even_partition(spec.num_layers, spec.num_stages);
  spec.finalize();
  ModelState m = init_model(spec, 7, 3e-4);
  // deterministic optimizer state and scalars
  auto fill = [](std::vector<double>& v, double a) {
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = a * static_cast<double>(i % 97) - 0.25;
  };
  m.edges.opt_embed.m.assign(m.edges.layers.embed.size(), 0.0);
  m.edges.opt_embed.v.assign(m.edges.layers.embed.size(), 0.0);
  m.edges.opt_deembed.m.assign(m.edges.layers.deembed.size(), 0.0);
  m.edges.opt_deembed.v.assign(m.edges.layers.deembed.size(), 0.0);
  fill(m.edges.opt_embed.m, 1e-3);
  fill(m.edges.opt_deembed.v, 2e-6);
  m.edges.opt_embed.step = 11;
  m.edges.opt_deembed.step = 12;
  m.edges.lr = 5e-4;
  for (StageState& s : m.stages) {
    s.opt.m.assign(s.param_count(), 0.0);
    s.opt.v.assign(s.param_count(), 0.0);
    fill(s.opt.m, 1e-4 * s.stage_id);
    fill(s.opt.v, 3e-7);
    s.opt.step = 40 + s.stage_id;
    s.omega = 0.125 * s.stage_id;
    s.lr = 3e-4 * (1.0 + 0.1 * s.stage_id);
  }
  const recovery::CheckpointSnapshot snap = recovery::checkpoint_save(m, 77, 1234567u);
  const std::vector<std::uint8_t> a = recovery::serialize_checkpoint(snap);
  const std::vector<std::uint8_t> b =
      recovery::serialize_checkpoint(recovery::deserialize_checkpoint(a, spec));
  std::uint64_t h = 1469598103934665603ull;
  for (std::uint8_t c : a) h = (h ^ c) * 1099511628211ull;
  if (argc > 1) recovery::save_checkpoint_file(snap, argv[1]);
  std::printf("%s size=%zu fnv=%016llx\n", a == b ? "OK" : "MISMATCH", a.size(), static_cast<unsigned long long>(h));
  return a == b ? 0 : 1;
}
