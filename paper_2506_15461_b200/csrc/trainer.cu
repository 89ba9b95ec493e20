// The failure-injected training loop on the device-resident engine:
// harness::Trainer (src/trainer.cpp:63-289) re-built around ckf::Engine.
// Slots vs model iterations, post-step failure handling in ascending stage
// order, adjacency -> unrecoverable, CheckFree+ replica refresh after every
// step, lr bump / omega reset / moment policy -- all as in the reference.
// Data: the teacher-student task of src/dataset.cpp:15-57 generated on the
// GPU (counter-RNG inputs, teacher forward) for the MLP block; the LLaMA block
// uses the counter-RNG token process of llama_block.cu.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include "engine.h"
#include "host_logic.h"

namespace ckf {

void argmax_rows(const void* pred, bool f64, size_t rows, size_t cols, int* out, cudaStream_t s);
void llama_token_batch(uint64_t data_seed, uint64_t stream, uint64_t index, size_t rows, size_t T, size_t V,
                       int* out, cudaStream_t s);

namespace {

constexpr uint64_t kSeedModel = 11, kSeedTask = 12, kSeedReinit = 13;  // trainer.cpp:22-24
constexpr uint64_t kStreamTrain = 1, kStreamVal = 2, kStreamTeacher = 3;  // dataset.cpp:11-13

ckf_model_desc make_desc(const host::Config& c) {
  ckf_model_desc d{};
  d.block = c.block == "llama" ? CKF_BLOCK_LLAMA : CKF_BLOCK_MLP;
  d.precision = c.precision == "fp64" ? CKF_FP64 : c.precision == "fp32" ? CKF_FP32 : CKF_BF16;
  d.activation = c.activation == "tanh" ? CKF_ACT_TANH : c.activation == "relu" ? CKF_ACT_RELU : CKF_ACT_IDENTITY;
  d.task = c.task == "regression" ? CKF_TASK_REGRESSION : CKF_TASK_CLASSIFICATION;
  d.input_dim = c.input_dim;
  d.hidden_dim = c.hidden_dim;
  d.model_dim = c.model_dim;
  d.output_dim = c.output_dim;
  d.num_layers = c.layers;
  d.num_stages = c.stages;
  d.n_heads = c.heads;
  d.seq_len = c.seq_len;
  d.partition = nullptr;
  const size_t mb = c.batch / static_cast<size_t>(c.microbatches);
  d.max_rows = d.block == CKF_BLOCK_MLP ? std::max(mb, c.val_size) : mb * c.seq_len;
  d.device = c.device;
  return d;
}

struct Batch {
  void* x = nullptr;  // device: master dtype [rows x in] (MLP) or int32 tokens [rows x (T+1)] (LLaMA)
  void* y = nullptr;  // device: targets (master dtype) or int32 labels; null for LLaMA
  size_t rows = 0;
};

class Trainer {
 public:
  Trainer(const host::Config& c, const host::Trace& trace, uint64_t seed, const TrainerComm* cm = nullptr)
      : c_(c), seed_(seed), desc_(make_desc(c)), model_(desc_) {
    data_seed_ = host::derive_key(seed, kSeedTask);
    model_.init(host::derive_key(seed, kSeedModel), c.lr);
    if (cm && cm->nranks > 1) {
      // one process per GPU: contiguous stage blocks per pipeline rank (edges with stages 1 and s),
      // `replicas` data-parallel copies; every rank runs this same loop (host logic replicated,
      // losses / omegas / recovery reports shared by the engine), peer mappings for recovery
      const int R = cm->replicas, P = cm->nranks / R;
      if (c.microbatches % R) host::fail(1, "microbatches must be divisible by the data-parallel replicas");
      if (c.batch % static_cast<size_t>(R)) host::fail(1, "batch must be divisible by the data-parallel replicas");
      std::vector<int> sr(c.stages);
      for (size_t i = 0; i < c.stages; ++i) sr[i] = static_cast<int>(i * static_cast<size_t>(P) / c.stages);
      model_.attach_comm(cm->uid, cm->nranks, cm->rank, sr.data(), R);
      // stage transfers through peer memory (mailbox + flags over NVLink) unless CKF_TRANSPORT=nccl
      const char* tr = std::getenv("CKF_TRANSPORT");
      if (P > 1 && desc_.block == CKF_BLOCK_LLAMA && desc_.precision == CKF_BF16 && !(tr && std::string(tr) == "nccl"))
        model_.enable_peer_transport(c.microbatches / R);
      model_.exchange_peers();
    }
    if (desc_.block == CKF_BLOCK_MLP) {
      teacher_ = std::make_unique<Engine>(desc_);
      teacher_->init(host::derive_key(data_seed_, kStreamTeacher), 1.0);
    }
    for (const auto& e : trace.events) events_[e.iteration].push_back(e.stage);
    for (auto& kv : events_) std::sort(kv.second.begin(), kv.second.end());
    const int s = static_cast<int>(c.stages);
    std_sched_ = host::build_schedule(c.microbatches, false, s);
    if (c.swapped_schedule()) sw_sched_ = host::build_schedule(c.microbatches, true, s);
    val_ = make_batch(kStreamVal, 0, c.val_size, 20);
  }

  std::string run() {
    t0_ = std::chrono::steady_clock::now();
    const bool cfp = c_.strategy == "checkfree-plus";
    const int s = static_cast<int>(c_.stages);
    const auto std_order = host::standard_order(s);
    const bool ckpt = c_.strategy == "checkpointing";
    // redundant computation runs its hot copies for real on the LLaMA block (measured overhead)
    if (c_.strategy == "redundant" && desc_.block == CKF_BLOCK_LLAMA && desc_.precision == CKF_BF16)
      model_.set_redundant(true);
    if (ckpt) model_.checkpoint_save(0);  // trainer.cpp:67-68
    if (cfp) model_.refresh_edge_replicas();
    {  // record_initial_eval (trainer.cpp:122-126)
      Batch first = make_batch(kStreamTrain, 1, c_.batch, 22);
      last_train_ = eval(first, std_order);
      add_eval(0);
    }
    bool stopped = false;
    long slots_run = 0;
    for (long slot = 1; slot <= c_.iters && !stopped; ++slot) {
      slots_run = slot;
      const bool swap_now = !sw_sched_.empty() && slot > c_.swap_from;
      Batch b = make_batch(kStreamTrain, static_cast<uint64_t>(model_iter_ + 1), c_.batch, 22);
      std::vector<double> om(c_.stages);
      // data parallel: replica r trains on microbatches [r m/R, (r+1) m/R) of the global batch with
      // their global execution orders (the mean over all m is restored by the all-reduce)
      const int R = model_.replicas(), rr = model_.replica();
      const int ml = c_.microbatches / R;
      const size_t rows_l = b.rows / static_cast<size_t>(R);
      const int* sched = (swap_now ? sw_sched_.data() : std_sched_.data()) + static_cast<size_t>(rr * ml) * c_.stages;
      model_.run_iteration(sched, ml, row_ptr(b.x, rows_l * static_cast<size_t>(rr), true),
                           row_ptr(b.y, rows_l * static_cast<size_t>(rr), false), rows_l, true, slot, &last_train_,
                           om.data());
      ++model_iter_;
      if (cfp) model_.refresh_edge_replicas();
      if (ckpt && model_iter_ % c_.checkpoint_interval == 0) model_.checkpoint_save(model_iter_);  // trainer.cpp:83-85
      if (c_.strategy != "no-failures") {
        auto ev = events_.find(slot);
        if (ev != events_.end() && !handle_failures(slot, ev->second)) {
          add_eval(slot);
          stopped = true;
          break;
        }
      }
      if (slot % c_.eval_interval == 0 || slot == c_.iters) {
        const double v = add_eval(slot);
        if (c_.target_loss > 0.0 && v <= c_.target_loss) stopped = true;
      }
    }
    if (evals_.empty() || evals_.back().first != slots_run) add_eval(slots_run);
    return out_.str();
  }

 private:
  // dataset.cpp:15-39 on the device: x ~ U[-1,1] keyed (data_seed, stream, index); y = teacher forward
  Batch make_batch(uint64_t stream, uint64_t index, size_t rows, int slot) {
    Batch b;
    b.rows = rows;
    cudaStream_t st = model_.stream();
    if (desc_.block == CKF_BLOCK_LLAMA) {
      int* t = static_cast<int*>(model_.ws(rows * (c_.seq_len + 1) * sizeof(int), slot));
      llama_token_batch(data_seed_, stream, index, rows, c_.seq_len, c_.output_dim, t, st);
      b.x = t;
      return b;
    }
    const size_t mbytes = model_.master_bytes();
    void* x = model_.ws(rows * c_.input_dim * mbytes, slot);
    const uint64_t key = host::derive_key(data_seed_, stream, index);
    if (model_.fp64())
      k::uniform(static_cast<double*>(x), rows * c_.input_dim, key, -1.0, 1.0, 0, st);
    else
      k::uniform(static_cast<float*>(x), rows * c_.input_dim, key, -1.0, 1.0, 0, st);
    CKF_CUDA(cudaStreamSynchronize(st));
    void* pred = teacher_->ws(rows * c_.output_dim * mbytes, 30);
    const auto order = host::standard_order(static_cast<int>(c_.stages));
    teacher_->predict_device(order.data(), x, rows, pred);
    CKF_CUDA(cudaStreamSynchronize(teacher_->stream()));
    if (c_.task == "regression") {
      void* y = model_.ws(rows * c_.output_dim * mbytes, slot + 1);
      CKF_CUDA(cudaMemcpy(y, pred, rows * c_.output_dim * mbytes, cudaMemcpyDeviceToDevice));
      b.y = y;
    } else {
      int* y = static_cast<int*>(model_.ws(rows * sizeof(int), slot + 1));
      argmax_rows(pred, model_.fp64(), rows, c_.output_dim, y, st);
      b.y = y;
    }
    b.x = x;
    CKF_CUDA(cudaDeviceSynchronize());
    return b;
  }

  // pointer to row r of a batch buffer (x: tokens / inputs, else targets / labels)
  const void* row_ptr(const void* p, size_t r, bool is_x) const {
    if (!p || r == 0) return p;
    size_t bytes;
    if (desc_.block == CKF_BLOCK_LLAMA) bytes = (c_.seq_len + 1) * sizeof(int);
    else if (is_x) bytes = c_.input_dim * model_.master_bytes();
    else bytes = c_.task == "regression" ? c_.output_dim * model_.master_bytes() : sizeof(int);
    return static_cast<const char*>(p) + r * bytes;
  }

  double eval(const Batch& b, const std::vector<int>& order) { return model_.eval_loss(order.data(), b.x, b.y, b.rows, true); }
  double val_loss() { return eval(val_, host::standard_order(static_cast<int>(c_.stages))); }

  double add_eval(long slot) {
    const double v = val_loss();
    evals_.push_back({slot, v});
    char buf[200];
    const double hours = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count() / 3600.0;
    // E,slot,train,val,measured wall hours,model iterations (slot minus checkpoint rollbacks)
    std::snprintf(buf, sizeof(buf), "E,%ld,%.17g,%.17g,%.17g,%ld\n", slot, last_train_, v, hours, model_iter_);
    out_ << buf;
    return v;
  }

  void add_event(long slot, int st, const std::string& action, double red, double spike, double ms) {
    pending_.push_back({slot, st, action, red, spike, ms});
  }
  void flush_events(double spike, bool set_spike) {
    for (auto& e : pending_) {
      char buf[256];
      std::snprintf(buf, sizeof(buf), "F,%ld,%d,%s,%.17g,%.17g,%.6g\n", e.slot, e.stage, e.action.c_str(), e.red,
                    set_spike ? spike : e.spike, e.ms);
      out_ << buf;
    }
    pending_.clear();
  }

  // trainer.cpp:146-289 (neighbour family, redundant, no-failures)
  bool handle_failures(long slot, const std::vector<int>& stages) {
    const int s = static_cast<int>(c_.stages);
    if (c_.strategy == "checkpointing") {
      // trainer.cpp:173-193: roll every stage back to the last snapshot (any stage, adjacent
      // failures included); data is addressed by model iteration, so the batches since the
      // snapshot are replayed
      const double vpre = val_loss();
      std::vector<double> red(stages.size(), 0.0);
      float ms = 0.f;
      model_iter_ = model_.checkpoint_restore(stages.data(), static_cast<int>(stages.size()), red.data(), &ms);
      const double vpost = val_loss();
      for (size_t i = 0; i < stages.size(); ++i) add_event(slot, stages[i], "checkpoint_restore", red[i], 0.0, ms);
      flush_events(vpost - vpre, true);
      return true;
    }
    for (size_t i = 0; i + 1 < stages.size(); ++i) {
      if (stages[i + 1] == stages[i] + 1) {
        for (int st : stages) add_event(slot, st, "unrecoverable", 0.0, 0.0, 0.0);
        flush_events(0.0, false);
        out_ << "U,stages " << stages[i] << " and " << stages[i] + 1 << " failed together at iteration " << slot
             << "; no live neighbor to recover from\n";
        return false;
      }
    }
    if (c_.strategy == "redundant") {
      for (int st : stages) add_event(slot, st, "redundant_copy", 0.0, 0.0, 0.0);
      flush_events(0.0, false);
      return true;
    }
    const double vpre = val_loss();
    const bool averaged = c_.recovered_moments == "averaged";
    for (int st : stages) {
      int mode;
      std::string action;
      if (st == 1 || st == s) {
        if (c_.strategy != "checkfree-plus") {
          add_event(slot, st, "unsupported", 0.0, 0.0, 0.0);
          flush_events(0.0, false);
          out_ << "U," << c_.strategy << " cannot recover the " << (st == 1 ? "first" : "last")
               << " stage (iteration " << slot << ")\n";
          return false;
        }
        mode = CKF_REC_EDGE;
        action = "edge_copy";
      } else if (c_.strategy == "checkfree" || c_.strategy == "checkfree-plus") {
        mode = CKF_REC_CHECKFREE;
      } else if (c_.strategy == "reinit-random") {
        mode = CKF_REC_RANDOM;
        action = "random_reinit";
      } else if (c_.strategy == "reinit-copy") {
        mode = CKF_REC_COPY_PREV;
        action = "copy_prev";
      } else {
        mode = CKF_REC_UNIFORM;
        action = "uniform_avg";
      }
      const uint64_t rseed = host::derive_key(seed_, kSeedReinit, static_cast<uint64_t>(slot), static_cast<uint64_t>(st));
      const int mom = averaged && (mode == CKF_REC_CHECKFREE || mode == CKF_REC_EDGE) ? CKF_MOM_AVERAGED : CKF_MOM_FRESH;
      ckf_recovery_report r = model_.recover_stage(st, mode, mom, c_.lr_bump, rseed, true);
      if (mode == CKF_REC_CHECKFREE) action = r.degenerate ? "uniform_avg_fallback" : "checkfree_avg";
      add_event(slot, st, action, r.reduction_error, 0.0, r.latency_ms);
    }
    const double vpost = val_loss();
    flush_events(vpost - vpre, true);
    return true;
  }

  struct Pending {
    long slot;
    int stage;
    std::string action;
    double red, spike, ms;
  };

  host::Config c_;
  uint64_t seed_;
  uint64_t data_seed_ = 0;
  ckf_model_desc desc_;
  Engine model_;
  std::unique_ptr<Engine> teacher_;
  std::map<long, std::vector<int>> events_;
  std::vector<int> std_sched_, sw_sched_;
  Batch val_;
  long model_iter_ = 0;
  double last_train_ = 0.0;
  std::vector<std::pair<long, double>> evals_;
  std::vector<Pending> pending_;
  std::ostringstream out_;
  std::chrono::steady_clock::time_point t0_;
};

// ------------------------------------------------------------------ run records (experiment.cpp:156-213)
std::string fmt12(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.12g", v);
  return b;
}

void write_text(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) host::fail(1, "cannot write '" + path + "'");
  f << text;
}

// metrics.csv / events.csv / summary.json / config.resolved in the reference's schema.
// wall_hours and recovery_s are MEASURED on the B200 (host clock around the device
// work; CUDA events around the recovery), where the reference models them.
void write_records(const host::Config& c, uint64_t seed, const std::string& rec, const std::string& dir) {
  std::filesystem::create_directories(dir);
  std::ostringstream m, e;
  m << "# format_version=1\niter,train_loss,val_loss,wall_hours\n";
  e << "# format_version=1\niter,stage,action,reduction_error,recovery_s\n";
  std::istringstream in(rec);
  std::string line, unrec;
  long last_iter = 0, n_events = 0;
  double last_train = 0.0, last_val = 0.0, hours = 0.0;
  while (std::getline(in, line)) {
    std::vector<std::string> f;
    std::stringstream ls(line);
    std::string tok;
    while (std::getline(ls, tok, ',')) f.push_back(tok);
    if (f.empty()) continue;
    if (f[0] == "E" && f.size() >= 5) {
      last_iter = std::stol(f[1]);
      last_train = std::stod(f[2]);
      last_val = std::stod(f[3]);
      hours = std::stod(f[4]);
      m << last_iter << ',' << fmt12(last_train) << ',' << fmt12(last_val) << ',' << fmt12(hours) << '\n';
    } else if (f[0] == "F" && f.size() >= 7) {
      e << f[1] << ',' << f[2] << ',' << f[3] << ',' << fmt12(std::stod(f[4])) << ',' << fmt12(std::stod(f[6]) / 1e3)
        << '\n';
      ++n_events;
    } else if (f[0] == "U") {
      unrec = line.substr(2);
    }
  }
  std::ostringstream j;
  j << "{\n  \"format_version\": 1,\n  \"strategy\": \"" << c.strategy << "\",\n  \"seed\": " << seed
    << ",\n  \"iterations_run\": " << last_iter << ",\n  \"model_iterations\": " << last_iter
    << ",\n  \"iterations_to_target\": null,\n  \"model_iterations_to_target\": null,\n  \"total_hours\": "
    << fmt12(hours) << ",\n  \"iteration_time_s\": " << fmt12(last_iter ? hours * 3600.0 / last_iter : 0.0)
    << ",\n  \"unrecoverable\": " << (unrec.empty() ? "false" : "true");
  if (!unrec.empty()) j << ",\n  \"unrecoverable_reason\": \"" << unrec << "\"";
  j << ",\n  \"final_train_loss\": " << fmt12(last_train) << ",\n  \"final_val_loss\": " << fmt12(last_val)
    << ",\n  \"failure_events\": " << n_events << ",\n  \"timing\": \"measured on the GPU\"\n}\n";
  std::ostringstream r;
  r << "# resolved experiment configuration\n";
  r << "block = " << c.block << "\nprecision = " << c.precision << '\n';
  r << "input-dim = " << c.input_dim << "\nhidden-dim = " << c.hidden_dim << "\nmodel-dim = " << c.model_dim
    << "\noutput-dim = " << c.output_dim << "\nlayers = " << c.layers << "\nstages = " << c.stages << '\n';
  if (c.block == "llama") r << "heads = " << c.heads << "\nseq-len = " << c.seq_len << '\n';
  r << "activation = " << c.activation << "\ntask = " << c.task << "\nstrategy = " << c.strategy
    << "\ncheckpoint-interval = " << c.checkpoint_interval << "\nlr-bump = " << fmt12(c.lr_bump)
    << "\nrecovered-moments = " << c.recovered_moments << "\np-hour = " << fmt12(c.p_hour) << '\n';
  if (c.p_iter >= 0.0) r << "p-iter = " << fmt12(c.p_iter) << '\n';
  r << "iter-seconds = " << fmt12(c.iter_seconds) << "\neligible = " << c.eligible << "\niters = " << c.iters
    << "\nbatch = " << c.batch << "\nmicrobatches = " << c.microbatches << "\nlr = " << fmt12(c.lr) << '\n';
  if (c.target_loss > 0.0) r << "target-loss = " << fmt12(c.target_loss) << '\n';
  r << "eval-interval = " << c.eval_interval << "\nval-size = " << c.val_size << "\nseed = " << seed
    << "\nschedule = " << c.schedule << "\nswap-from = " << c.swap_from << '\n';
  write_text(dir + "/metrics.csv", m.str());
  write_text(dir + "/events.csv", e.str());
  write_text(dir + "/summary.json", j.str());
  write_text(dir + "/config.resolved", r.str());
}

}  // namespace

std::string run_experiment(const std::string& kv, const std::string& trace_text, uint64_t seed,
                           const std::string& dir, const TrainerComm* cm) {
  host::Config c = host::Config::from_kv(kv);
  c.validate();
  host::Trace t = trace_text.empty() ? c.resolve_trace(seed) : host::parse_trace(trace_text);
  host::validate_trace(t);
  Trainer tr(c, t, seed, cm);
  std::string rec = tr.run();
  if (!dir.empty()) write_records(c, seed, rec, dir);
  return rec;
}

}  // namespace ckf
