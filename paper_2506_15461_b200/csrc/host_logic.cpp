// Host control logic (see host_logic.h).  Bit-exact restatement of the
// reference's integer / host-double logic; checked against the reference's
// golden traces and schedules in tests/test_host_logic.py.
#include "host_logic.h"

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <set>

namespace ckf::host {

namespace {
std::string fmt17(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}
}  // namespace

double hourly_to_per_iteration(double p_hour, double iter_s) {
  // failures.cpp:57-61
  if (p_hour < 0.0 || p_hour >= 1.0) fail(1, "p_hour must lie in [0, 1)");
  if (iter_s <= 0.0) fail(1, "iteration_seconds must be positive");
  return 1.0 - std::pow(1.0 - p_hour, iter_s / 3600.0);
}

Trace generate_trace(uint64_t seed, double p_hour, double iter_s, long n_iters, std::vector<int> stages) {
  // failures.cpp:63-82: each (iteration, stage) fails iff unit_at(seed, iter, stage) < p_iter
  for (int s : stages)
    if (s < 1) fail(1, "stage ids are 1-based");
  if (n_iters <= 0) fail(1, "num_iterations must be positive");
  Trace t;
  t.seed = seed;
  t.p_hour = p_hour;
  t.iter_s = iter_s;
  t.stages = stages;
  const double p = hourly_to_per_iteration(p_hour, iter_s);
  std::sort(stages.begin(), stages.end());
  for (long it = 1; it <= n_iters; ++it)
    for (int st : stages)
      if (unit_at(seed, static_cast<uint64_t>(it), static_cast<uint64_t>(st)) < p) t.events.push_back({it, st});
  return t;
}

std::string serialize_trace(const Trace& t) {
  // failures.cpp:84-95
  std::ostringstream o;
  o << "checkfree-trace v1 seed=" << t.seed << " p_hour=" << fmt17(t.p_hour) << " iter_s=" << fmt17(t.iter_s)
    << " stages=";
  for (size_t i = 0; i < t.stages.size(); ++i) o << (i ? "," : "") << t.stages[i];
  o << '\n';
  for (const auto& e : t.events) o << e.iteration << ',' << e.stage << '\n';
  return o.str();
}

void validate_trace(const Trace& t) {
  // failures.cpp:30-54 (FailureRateSpec::validate + FailureTrace::validate)
  if (t.p_hour < 0.0 || t.p_hour >= 1.0) fail(1, "p_hour must lie in [0, 1)");
  for (int s : t.stages)
    if (s < 1) fail(1, "stage ids are 1-based");
  if (t.iter_s <= 0.0) fail(1, "iteration_seconds must be positive");
  std::set<int> eligible(t.stages.begin(), t.stages.end());
  std::set<std::pair<long, int>> seen;
  long prev = 0;
  for (const auto& e : t.events) {
    if (e.iteration < 1) fail(1, "trace iterations are 1-based");
    if (e.iteration < prev) fail(1, "trace events must be sorted by iteration");
    if (e.stage < 1) fail(1, "stage ids are 1-based");
    if (!eligible.count(e.stage)) fail(1, "trace event targets stage " + std::to_string(e.stage) + " outside the eligible set");
    if (!seen.insert({e.iteration, e.stage}).second)
      fail(1, "duplicate event for stage " + std::to_string(e.stage) + " at iteration " + std::to_string(e.iteration));
    prev = e.iteration;
  }
}

Trace parse_trace(const std::string& text, const std::string& ctx) {
  // failures.cpp:97-155; errors are ParseError (code 4)
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line)) fail(4, ctx + ":1: empty trace file");
  Trace t;
  {
    std::istringstream h(line);
    std::string magic, ver, kv;
    h >> magic >> ver;
    if (magic != "checkfree-trace" || ver != "v1") fail(4, ctx + ":1: expected header 'checkfree-trace v1'");
    while (h >> kv) {
      const auto eq = kv.find('=');
      if (eq == std::string::npos) fail(4, ctx + ":1: malformed header field '" + kv + "'");
      const std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
      try {
        if (k == "seed") {
          t.seed = std::stoull(v);
        } else if (k == "p_hour") {
          t.p_hour = std::stod(v);
        } else if (k == "iter_s") {
          t.iter_s = std::stod(v);
        } else if (k == "stages") {
          std::istringstream ls(v);
          std::string tok;
          while (std::getline(ls, tok, ','))
            if (!tok.empty()) t.stages.push_back(std::stoi(tok));
        } else {
          fail(4, ctx + ":1: unknown header field '" + k + "'");
        }
      } catch (const std::invalid_argument&) {
        fail(4, ctx + ":1: invalid value for '" + k + "'");
      } catch (const std::out_of_range&) {
        fail(4, ctx + ":1: value out of range for '" + k + "'");
      }
    }
  }
  size_t ln = 1;
  while (std::getline(in, line)) {
    ++ln;
    if (line.empty()) continue;
    long it = 0;
    int st = 0;
    if (std::sscanf(line.c_str(), "%ld,%d", &it, &st) != 2) fail(4, ctx + ":" + std::to_string(ln) + ": expected 'iteration,stage'");
    t.events.push_back({it, st});
  }
  try {
    validate_trace(t);
  } catch (const HostError& e) {
    fail(4, ctx + ": " + e.what());
  }
  return t;
}

std::vector<Event> consecutive_conflicts(const Trace& t) {
  // failures.cpp:171-184
  std::vector<Event> out;
  size_t i = 0;
  while (i < t.events.size()) {
    size_t j = i;
    while (j < t.events.size() && t.events[j].iteration == t.events[i].iteration) ++j;
    std::set<int> st;
    for (size_t q = i; q < j; ++q) st.insert(t.events[q].stage);
    for (int s : st)
      if (st.count(s + 1)) out.push_back({t.events[i].iteration, s});
    i = j;
  }
  return out;
}

std::vector<int> standard_order(int s) {
  std::vector<int> o(static_cast<size_t>(s));
  for (int i = 0; i < s; ++i) o[static_cast<size_t>(i)] = i + 1;
  return o;
}

std::vector<int> swapped_order(int s) {
  // pipeline.cpp:18-26
  if (s < 4) fail(1, "swapped order requires at least 4 stages (first and last pairs must be disjoint)");
  auto o = standard_order(s);
  std::swap(o[0], o[1]);
  std::swap(o[static_cast<size_t>(s - 2)], o[static_cast<size_t>(s - 1)]);
  return o;
}

std::vector<int> build_schedule(int m, bool swapped_half, int s) {
  if (m < 1) fail(1, "microbatch count must be positive");
  if (swapped_half && m % 2 != 0) fail(1, "swapped_half schedule requires an even microbatch count");
  std::vector<int> out;
  for (int k = 0; k < m; ++k) {
    auto o = swapped_half && k % 2 == 0 ? swapped_order(s) : standard_order(s);
    out.insert(out.end(), o.begin(), o.end());
  }
  return out;
}

// ------------------------------------------------------------------ config
Config Config::from_kv(const std::string& text) {
  Config c;
  std::stringstream ss(text);
  std::string item;
  std::map<std::string, std::string> kv;
  while (std::getline(ss, item, ';')) {
    // also accept newline-separated "key = value" (config.resolved format)
    std::stringstream ls(item);
    std::string line;
    while (std::getline(ls, line, '\n')) {
      if (line.empty() || line[0] == '#') continue;
      const auto eq = line.find('=');
      if (eq == std::string::npos) fail(1, "malformed config item '" + line + "'");
      auto trim = [](std::string s) {
        const auto a = s.find_first_not_of(" \t"), b = s.find_last_not_of(" \t\r");
        return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
      };
      kv[trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
    }
  }
  auto U = [&](const char* k, size_t& v) { if (kv.count(k)) v = std::stoul(kv[k]); };
  auto L_ = [&](const char* k, long& v) { if (kv.count(k)) v = std::stol(kv[k]); };
  auto D = [&](const char* k, double& v) { if (kv.count(k)) v = std::stod(kv[k]); };
  auto S = [&](const char* k, std::string& v) { if (kv.count(k)) v = kv[k]; };
  try {
    S("block", c.block);
    S("precision", c.precision);
    U("input-dim", c.input_dim);
    U("hidden-dim", c.hidden_dim);
    U("model-dim", c.model_dim);
    U("output-dim", c.output_dim);
    U("layers", c.layers);
    U("stages", c.stages);
    U("heads", c.heads);
    U("seq-len", c.seq_len);
    if (kv.count("vocab")) c.input_dim = c.output_dim = std::stoul(kv["vocab"]);
    if (kv.count("ffn")) c.hidden_dim = std::stoul(kv["ffn"]);
    S("activation", c.activation);
    S("task", c.task);
    S("strategy", c.strategy);
    L_("checkpoint-interval", c.checkpoint_interval);
    D("lr-bump", c.lr_bump);
    S("recovered-moments", c.recovered_moments);
    S("trace", c.trace_path);
    D("p-hour", c.p_hour);
    D("p-iter", c.p_iter);
    D("iter-seconds", c.iter_seconds);
    S("eligible", c.eligible);
    L_("iters", c.iters);
    U("batch", c.batch);
    if (kv.count("microbatches")) c.microbatches = std::stoi(kv["microbatches"]);
    D("lr", c.lr);
    D("target-loss", c.target_loss);
    L_("eval-interval", c.eval_interval);
    U("val-size", c.val_size);
    if (kv.count("seed")) c.seed = std::stoull(kv["seed"]);
    S("schedule", c.schedule);
    L_("swap-from", c.swap_from);
    if (kv.count("device")) c.device = std::stoi(kv["device"]);
  } catch (const std::logic_error& e) {
    fail(1, std::string("invalid config value: ") + e.what());
  }
  return c;
}

bool Config::swapped_schedule() const {
  if (schedule == "standard") return false;
  if (schedule == "swapped-half") return true;
  return strategy == "checkfree-plus";  // experiment.cpp:64-69
}

bool Config::neighbor_based() const {
  return strategy == "checkfree" || strategy == "checkfree-plus" || strategy == "reinit-random" ||
         strategy == "reinit-copy" || strategy == "reinit-uniform-avg";  // recovery.cpp:44-55
}

std::vector<int> Config::resolved_eligible() const {
  // experiment.cpp:71-85
  const int s = static_cast<int>(stages);
  std::vector<int> mid, all;
  for (int i = 2; i < s; ++i) mid.push_back(i);
  for (int i = 1; i <= s; ++i) all.push_back(i);
  if (eligible == "intermediate") return mid;
  if (eligible == "all") return all;
  if (strategy == "checkfree" || strategy == "reinit-random" || strategy == "reinit-copy" ||
      strategy == "reinit-uniform-avg")
    return mid;
  return all;
}

void Config::validate() const {
  // experiment.cpp:34-62 plus the model checks (model.cpp:80-97)
  static const std::set<std::string> kinds = {"no-failures", "checkpointing", "redundant", "checkfree",
                                              "checkfree-plus", "reinit-random", "reinit-copy", "reinit-uniform-avg"};
  if (!kinds.count(strategy)) fail(1, "unknown strategy '" + strategy + "'");
  if (block != "mlp" && block != "llama") fail(1, "block must be mlp|llama");
  if (precision != "fp64" && precision != "fp32" && precision != "bf16") fail(1, "precision must be fp64|fp32|bf16");
  if (activation != "tanh" && activation != "relu" && activation != "identity")
    fail(1, "unknown activation '" + activation + "' (expected tanh|relu|identity)");
  if (task != "regression" && task != "classification")
    fail(1, "unknown task '" + task + "' (expected regression|classification)");
  if (input_dim == 0 || hidden_dim == 0 || model_dim == 0 || output_dim == 0 || layers == 0)
    fail(1, "model dimensions and layer count must be positive");
  if (stages < 1 || stages > layers) fail(1, "num_stages must lie in [1, num_layers]");
  if (stages < 2) fail(1, "experiments need a pipeline of at least 2 stages");
  if (strategy == "checkpointing" && checkpoint_interval <= 0) fail(1, "checkpoint interval must be positive");
  if (lr_bump <= 0.0) fail(1, "lr_bump must be positive");
  if (iters <= 0) fail(1, "total_iterations must be positive");
  if (batch == 0 || microbatches <= 0 || batch % static_cast<size_t>(microbatches) != 0)
    fail(1, "batch size must be a positive multiple of the microbatch count");
  if (lr <= 0.0) fail(1, "learning rate must be positive");
  if (eval_interval <= 0) fail(1, "eval_interval must be positive");
  if (val_size == 0) fail(1, "validation set must be non-empty");
  if (p_iter >= 1.0) fail(1, "p_iter must lie in [0, 1)");
  if (p_hour < 0.0 || p_hour >= 1.0) fail(1, "p_hour must lie in [0, 1)");
  if (iter_seconds <= 0.0) fail(1, "iteration_seconds must be positive");
  if (schedule != "auto" && schedule != "standard" && schedule != "swapped-half")
    fail(1, "schedule_mode must be auto|standard|swapped-half");
  if (eligible != "auto" && eligible != "intermediate" && eligible != "all")
    fail(1, "eligible must be auto|intermediate|all");
  if (swapped_schedule()) {
    if (stages < 4) fail(1, "the swapped schedule requires at least 4 stages");
    if (microbatches % 2 != 0) fail(1, "the swapped schedule requires an even microbatch count");
  }
  if (neighbor_based() && layers % stages != 0)
    fail(1, "neighbor-based recovery requires a uniform stage partition");
  if (block == "llama") {
    if (model_dim % heads != 0) fail(1, "model_dim must be divisible by heads");
    if (precision == "fp64") fail(1, "the LLaMA block runs in fp32 (parity) or bf16");
  } else if (precision == "bf16") {
    fail(1, "the residual-MLP parity block runs in fp64 or fp32");
  }
}

Trace Config::resolve_trace(uint64_t s) const {
  // experiment.cpp:102-115
  if (!trace_path.empty()) {
    std::ifstream in(trace_path, std::ios::binary);
    if (!in) fail(1, "cannot open trace file '" + trace_path + "'");
    std::ostringstream b;
    b << in.rdbuf();
    return parse_trace(b.str(), trace_path);
  }
  if (p_iter >= 0.0) return generate_trace(s, p_iter, 3600.0, iters, resolved_eligible());
  return generate_trace(s, p_hour, iter_seconds, iters, resolved_eligible());
}

// ------------------------------------------------------------------ pipeline plan
int plan_inflight_limit(int m, const std::vector<int>& stage_rank) {
  std::vector<int> r(stage_rank);
  std::sort(r.begin(), r.end());
  const int P = static_cast<int>(std::unique(r.begin(), r.end()) - r.begin());
  return std::max(1, std::min(m, P));
}

namespace {
// 1F1B list schedule.  A microbatch's route (embedding, its stages in execution order, head) is
// cut into SEGMENTS: maximal runs of consecutive route positions on one rank.  The forward
// segments run in route order; the segment holding the head also runs the loss and the head
// backward; the backward segments walk the route back.  Each rank keeps two FIFO queues
// (forward segments and backward segments, both ordered by microbatch then route position) and,
// whenever it is idle, runs the head of its backward queue if that is ready, else the head of its
// forward queue if that is ready and fewer than `limit` microbatches are in flight on the rank.
// The earliest unfinished microbatch is always runnable (both queues are in microbatch order),
// so the simulation cannot stall.  The segments and their transfers are then sorted by simulated
// time (a transfer at its producer's finish time, before any segment starting at that time):
// the result is a topological order of the iteration in which every rank's ops, and every
// link's transfers, appear in the order that rank / link executes them.  Each rank issuing its
// share of this one order onto in-order streams can therefore never deadlock, whatever the
// real durations are.
struct Seg {
  int k, phase, rank, dep;
  std::vector<PlanOp> ops;
  double dur;
  double start = -1, fin = -1;
};
}  // namespace

std::vector<PlanOp> pipeline_plan(int s, int m, const std::vector<int>& orders, const std::vector<int>& stage_rank,
                                  int schedule, const PlanCost* cost, int limit) {
  if (s < 1 || m < 1) fail(1, "pipeline plan needs s >= 1 and m >= 1");
  if (orders.size() != static_cast<size_t>(s) * static_cast<size_t>(m)) fail(1, "orders must hold m*s stage ids");
  if (stage_rank.size() != static_cast<size_t>(s)) fail(1, "placement must name one rank per stage");
  if (schedule < 0 || schedule > 2) fail(1, "schedule must be 0 (sequential), 1 (gpipe) or 2 (1f1b)");
  auto owner = [&](int code) {  // 0 embedding, 1..s stages, s+1 de-embedding
    const int sid = code <= 0 ? 1 : code > s ? s : code;
    return stage_rank[static_cast<size_t>(sid - 1)];
  };
  std::vector<PlanOp> ops;
  auto xfer = [&](int phase, int mb, int from, int to, int aux) {
    if (owner(from) != owner(to)) ops.push_back({phase, mb, PlanOp::kXfer, owner(from), owner(to), aux});
  };
  auto fwd = [&](int k) {
    const int* o = orders.data() + static_cast<size_t>(k) * static_cast<size_t>(s);
    ops.push_back({0, k, PlanOp::kEmbedFwd, owner(0), 0, 0});
    int at = 0;
    for (int i = 0; i < s; ++i) {
      xfer(0, k, at, o[i], 0);
      ops.push_back({0, k, PlanOp::kStageFwd, owner(o[i]), o[i], 0});
      at = o[i];
    }
    xfer(0, k, at, s + 1, 0);
    ops.push_back({0, k, PlanOp::kHead, owner(s + 1), 0, 0});
  };
  auto bwd = [&](int k) {
    const int* o = orders.data() + static_cast<size_t>(k) * static_cast<size_t>(s);
    int at = s + 1;
    for (int i = s - 1; i >= 0; --i) {
      xfer(1, k, at, o[i], 1);
      ops.push_back({1, k, PlanOp::kStageBwd, owner(o[i]), o[i], 0});
      at = o[i];
    }
    xfer(1, k, at, 0, 1);
    ops.push_back({1, k, PlanOp::kEmbedBwd, owner(0), 0, 0});
  };
  if (schedule == 0) {
    for (int k = 0; k < m; ++k) {
      fwd(k);
      bwd(k);
    }
    return ops;
  }
  if (schedule == 1) {
    for (int k = 0; k < m; ++k) fwd(k);
    for (int k = 0; k < m; ++k) bwd(k);
    return ops;
  }

  // ---- schedule 2: 1F1B list schedule
  if (limit <= 0) limit = plan_inflight_limit(m, stage_rank);
  auto scost = [&](int sid) {
    return cost && cost->stage.size() == static_cast<size_t>(s) ? cost->stage[static_cast<size_t>(sid - 1)] : 1.0;
  };
  const double head_cost = cost ? cost->head : 1.0, embed_cost = cost ? cost->embed : 0.05;
  int nranks = 0;
  for (int r : stage_rank) nranks = std::max(nranks, r + 1);
  std::vector<Seg> segs;
  for (int k = 0; k < m; ++k) {
    const int* o = orders.data() + static_cast<size_t>(k) * static_cast<size_t>(s);
    // forward route: E, o[0..s-1], head
    std::vector<int> route{0};
    route.insert(route.end(), o, o + s);
    route.push_back(s + 1);
    int prev = -1;
    for (size_t i = 0; i < route.size();) {
      Seg g{k, 0, owner(route[i]), prev, {}, 0.0};
      while (i < route.size() && owner(route[i]) == g.rank) {
        const int c = route[i++];
        if (c == 0) {
          g.ops.push_back({0, k, PlanOp::kEmbedFwd, g.rank, 0, 0});
          g.dur += embed_cost;
        } else if (c == s + 1) {
          g.ops.push_back({0, k, PlanOp::kHead, g.rank, 0, 0});
          g.dur += 3.0 * head_cost;
        } else {
          g.ops.push_back({0, k, PlanOp::kStageFwd, g.rank, c, 0});
          g.dur += scost(c);
        }
      }
      segs.push_back(std::move(g));
      prev = static_cast<int>(segs.size()) - 1;
    }
    // backward route: o[s-1..0], E
    std::vector<int> broute(o, o + s);
    std::reverse(broute.begin(), broute.end());
    broute.push_back(0);
    for (size_t i = 0; i < broute.size();) {
      Seg g{k, 1, owner(broute[i]), prev, {}, 0.0};
      while (i < broute.size() && owner(broute[i]) == g.rank) {
        const int c = broute[i++];
        if (c == 0) {
          g.ops.push_back({1, k, PlanOp::kEmbedBwd, g.rank, 0, 0});
          g.dur += embed_cost;
        } else {
          g.ops.push_back({1, k, PlanOp::kStageBwd, g.rank, c, 0});
          g.dur += 2.0 * scost(c);
        }
      }
      segs.push_back(std::move(g));
      prev = static_cast<int>(segs.size()) - 1;
    }
  }
  // per-rank FIFO queues (segments were appended in microbatch, then route order)
  std::vector<std::vector<int>> qf(static_cast<size_t>(nranks)), qb(static_cast<size_t>(nranks));
  std::vector<std::vector<int>> bleft(static_cast<size_t>(nranks), std::vector<int>(static_cast<size_t>(m), 0));
  for (size_t i = 0; i < segs.size(); ++i) {
    (segs[i].phase ? qb : qf)[static_cast<size_t>(segs[i].rank)].push_back(static_cast<int>(i));
    if (segs[i].phase) ++bleft[static_cast<size_t>(segs[i].rank)][static_cast<size_t>(segs[i].k)];
  }
  std::vector<size_t> pf(static_cast<size_t>(nranks), 0), pb(static_cast<size_t>(nranks), 0);
  std::vector<double> free_at(static_cast<size_t>(nranks), 0.0);
  std::vector<std::vector<char>> started(static_cast<size_t>(nranks), std::vector<char>(static_cast<size_t>(m), 0));
  std::vector<int> inflight(static_cast<size_t>(nranks), 0);
  std::vector<int> busy(static_cast<size_t>(nranks), -1);  // segment running on the rank
  size_t done = 0;
  double t = 0.0;
  auto ready = [&](int i) {
    const int d = segs[static_cast<size_t>(i)].dep;
    return d < 0 || (segs[static_cast<size_t>(d)].fin >= 0 && segs[static_cast<size_t>(d)].fin <= t);
  };
  while (done < segs.size()) {
    // retire segments finishing by t
    for (int r = 0; r < nranks; ++r) {
      const int b = busy[static_cast<size_t>(r)];
      if (b >= 0 && segs[static_cast<size_t>(b)].fin <= t) {
        busy[static_cast<size_t>(r)] = -1;
        ++done;
        const Seg& g = segs[static_cast<size_t>(b)];
        if (g.phase && --bleft[static_cast<size_t>(r)][static_cast<size_t>(g.k)] == 0) --inflight[static_cast<size_t>(r)];
      }
    }
    bool progressed = false;
    for (int r = 0; r < nranks; ++r) {
      if (busy[static_cast<size_t>(r)] >= 0) continue;
      const size_t ru = static_cast<size_t>(r);
      int pick = -1;
      if (pb[ru] < qb[ru].size() && ready(qb[ru][pb[ru]])) {
        pick = qb[ru][pb[ru]++];
      } else if (pf[ru] < qf[ru].size() && ready(qf[ru][pf[ru]])) {
        const int c = qf[ru][pf[ru]];
        const int k = segs[static_cast<size_t>(c)].k;
        if (started[ru][static_cast<size_t>(k)] || inflight[ru] < limit) {
          if (!started[ru][static_cast<size_t>(k)]) {
            started[ru][static_cast<size_t>(k)] = 1;
            if (bleft[ru][static_cast<size_t>(k)] > 0) ++inflight[ru];
          }
          pick = qf[ru][pf[ru]++];
        }
      }
      if (pick < 0) continue;
      Seg& g = segs[static_cast<size_t>(pick)];
      g.start = t;
      g.fin = t + std::max(g.dur, 1e-9);
      busy[ru] = pick;
      progressed = true;
    }
    // next event: the earliest running segment's finish
    double nt = -1.0;
    for (int r = 0; r < nranks; ++r) {
      const int b = busy[static_cast<size_t>(r)];
      if (b >= 0 && (nt < 0 || segs[static_cast<size_t>(b)].fin < nt)) nt = segs[static_cast<size_t>(b)].fin;
    }
    if (nt < 0) {
      if (done < segs.size()) fail(1, "pipeline plan: 1F1B simulation stalled (internal error)");
      break;
    }
    if (!progressed || nt > t) t = nt;
  }
  // flatten: segments at (start, 1, rank), transfers at (producer finish, 0, src)
  struct Item {
    double time;
    int cls, rank;
    size_t seq;
    std::vector<PlanOp> ops;
  };
  std::vector<Item> items;
  for (size_t i = 0; i < segs.size(); ++i) {
    const Seg& g = segs[i];
    items.push_back({g.start, 1, g.rank, i, g.ops});
    // the transfer to the next segment of the same microbatch (if it runs on another rank)
    for (size_t j = i + 1; j < segs.size() && segs[j].k == g.k; ++j) {
      if (segs[j].dep != static_cast<int>(i)) continue;
      if (segs[j].rank != g.rank) items.push_back({g.fin, 0, g.rank, i, {{segs[j].phase, g.k, PlanOp::kXfer, g.rank,
                                                                          segs[j].rank, segs[j].phase}}});
      break;
    }
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    if (a.time != b.time) return a.time < b.time;
    if (a.cls != b.cls) return a.cls < b.cls;
    if (a.rank != b.rank) return a.rank < b.rank;
    return a.seq < b.seq;
  });
  for (auto& it : items) ops.insert(ops.end(), it.ops.begin(), it.ops.end());
  return ops;
}

}  // namespace ckf::host
