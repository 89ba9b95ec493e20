// Reference-parity block: the reference's residual MLP, embed -> L x
// [h += act(h W1) W2] -> de-embed (model.hpp:55-60, model.cpp:211-378), on
// the GPU in fp64 (bit-level parity mode) or fp32.  Gradients accumulate
// straight into the stage accumulators (GEMM beta = 1), replacing
// Gradients::accumulate (model.cpp:299-305).
#include <vector>

#include "engine.h"

namespace ckf {

namespace {
__global__ void argmax_rows_kernel(const double* __restrict__ p, size_t rows, size_t cols, int* __restrict__ out) {
  const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  size_t best = 0;  // first maximum wins (dataset.cpp:30-33)
  for (size_t j = 1; j < cols; ++j)
    if (p[r * cols + j] > p[r * cols + best]) best = j;
  out[r] = static_cast<int>(best);
}
__global__ void argmax_rows_kernel_f(const float* __restrict__ p, size_t rows, size_t cols, int* __restrict__ out) {
  const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  size_t best = 0;
  for (size_t j = 1; j < cols; ++j)
    if (p[r * cols + j] > p[r * cols + best]) best = j;
  out[r] = static_cast<int>(best);
}
}  // namespace

void argmax_rows(const void* pred, bool f64, size_t rows, size_t cols, int* out, cudaStream_t s) {
  if (f64)
    argmax_rows_kernel<<<grid_for(rows, 128), 128, 0, s>>>(static_cast<const double*>(pred), rows, cols, out);
  else
    argmax_rows_kernel_f<<<grid_for(rows, 128), 128, 0, s>>>(static_cast<const float*>(pred), rows, cols, out);
  CKF_LAUNCH_CHECK();
}

struct MlpBlock final : BlockImpl {
  explicit MlpBlock(Engine* e) : BlockImpl(e) {}

  size_t blk_params() const { return 2 * eng->desc().d * eng->desc().hid; }
  size_t stage_params(int sid) const override { return eng->desc().part[static_cast<size_t>(sid - 1)].count() * blk_params(); }
  size_t embed_params() const override { return eng->desc().in * eng->desc().d; }
  size_t deembed_params() const override { return eng->desc().d * eng->desc().out; }

  template <typename T>
  void sample(T* w, size_t n, size_t fan_in, size_t fan_out, uint64_t key) {
    // sample_uniform (model.cpp:27-33): U[-a, a], a = sqrt(6/(fan_in+fan_out))
    const double a = std::sqrt(6.0 / static_cast<double>(fan_in + fan_out));
    k::uniform(w, n, key, -a, a, 0, eng->stream());
  }

  template <typename T>
  void init_stage_t(int sid, uint64_t seed, T* w) {
    const Desc& d = eng->desc();
    const Range& r = d.part[static_cast<size_t>(sid - 1)];
    size_t off = 0;
    for (size_t layer = r.first; layer <= r.last; ++layer) {  // tags 2l / 2l+1 (model.cpp:24-25,159-172)
      sample(w + off, d.d * d.hid, d.d, d.hid, derive_key(seed, 2 * layer));
      off += d.d * d.hid;
      sample(w + off, d.hid * d.d, d.hid, d.d, derive_key(seed, 2 * layer + 1));
      off += d.hid * d.d;
    }
  }
  void init_stage(int sid, uint64_t seed, void* w) override {
    if (eng->fp64())
      init_stage_t(sid, seed, static_cast<double*>(w));
    else
      init_stage_t(sid, seed, static_cast<float*>(w));
  }
  template <typename T>
  void init_edges_t(uint64_t seed, T* e, T* de) {
    const Desc& d = eng->desc();
    if (e) sample(e, d.in * d.d, d.in, d.d, derive_key(seed, 0));      // kTagEmbed
    if (de) sample(de, d.d * d.out, d.d, d.out, derive_key(seed, 1));  // kTagDeembed
  }
  void init_edges(uint64_t seed, void* e, void* de) override {
    if (eng->fp64())
      init_edges_t(seed, static_cast<double*>(e), static_cast<double*>(de));
    else
      init_edges_t(seed, static_cast<float*>(e), static_cast<float*>(de));
  }

  // CUDA-core GEMM, timed as KC_GEMM when the engine's kernel timing is on
  template <typename T>
  void gemm(bool ta, bool tb, size_t M, size_t N, size_t K, const T* A, size_t lda, const T* B, size_t ldb, T* C,
            size_t ldc, bool acc) {
    eng->kt_begin();
    k::gemm_simt<T>(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, acc, eng->stream());
    eng->kt_end(KC_GEMM, 2.0 * M * N * K,
                sizeof(T) * (static_cast<double>(M) * K + static_cast<double>(K) * N + (acc ? 2.0 : 1.0) * M * N));
  }

  // Workspace slots (>= 8; 0-3 belong to the engine's upload paths).
  template <typename T>
  T* buf(int slot, size_t elems) {
    return static_cast<T*>(eng->ws(elems * sizeof(T), slot));
  }

  // Per-slot state kept from forward to backward: the applied-block caches
  // (block input, hidden activation) and dL/dh_final.
  static int slot_id(int mb, int k) { return 1000 + 8 * mb + k; }

  template <typename T>
  void fwd(int mb, const int* order, const T* x, const void* y, size_t b, bool train, double* loss_dev, T* pred_out) {
    const Desc& d = eng->desc();
    cudaStream_t st = eng->stream();
    const size_t L = d.L;
    T* h = buf<T>(8, b * d.d);
    T* cache_in = buf<T>(slot_id(mb, 0), L * b * d.d);
    T* cache_z = buf<T>(slot_id(mb, 1), L * b * d.hid);
    T* dh = buf<T>(slot_id(mb, 2), b * d.d);
    T* pre = buf<T>(11, b * d.hid);
    T* pred = pred_out ? pred_out : buf<T>(12, b * d.out);
    T* dpred = buf<T>(13, b * d.out);

    // ---- forward (model.cpp:226-253)
    int at = 0;  // pipeline position of h (0 = embedding)
    if (eng->mine(eng->owner_of_embed()))
      gemm<T>(false, false, b, d.d, d.in, x, d.in, static_cast<const T*>(eng->embed().w), d.d, h, d.d, false);
    size_t slot = 0;
    for (size_t oi = 0; oi < d.s; ++oi) {
      const int sid = order[oi];
      const int own = eng->owner_of_stage(sid);
      eng->move(h, b * d.d * sizeof(T), at, sid);
      at = sid;
      const Range& r = d.part[static_cast<size_t>(sid - 1)];
      for (size_t bi = 0; bi < r.count(); ++bi, ++slot) {
        if (!eng->mine(own)) continue;
        const T* w1 = static_cast<const T*>(eng->stage(sid).w) + bi * blk_params();
        const T* w2 = w1 + d.d * d.hid;
        T* cin = cache_in + slot * b * d.d;
        T* cz = cache_z + slot * b * d.hid;
        CKF_CUDA(cudaMemcpyAsync(cin, h, b * d.d * sizeof(T), cudaMemcpyDeviceToDevice, st));
        gemm<T>(false, false, b, d.hid, d.d, h, d.d, w1, d.hid, pre, d.hid, false);
        k::act_fwd<T>(d.act, pre, cz, b * d.hid, st);
        gemm<T>(false, false, b, d.d, d.hid, cz, d.hid, w2, d.d, h, d.d, true);
      }
    }
    eng->move(h, b * d.d * sizeof(T), at, static_cast<int>(d.s) + 1);
    if (!eng->mine(eng->owner_of_deembed())) return;
    gemm<T>(false, false, b, d.out, d.d, h, d.d, static_cast<const T*>(eng->deembed().w), d.out, pred, d.out, false);
    if (loss_dev) {
      if (d.task == CKF_TASK_REGRESSION)
        k::mse_loss_grad<T>(pred, static_cast<const T*>(y), b, d.out, train ? dpred : nullptr, loss_dev,
                            eng->scratch(), st);
      else
        k::xent_loss_grad<T>(pred, static_cast<const int*>(y), b, d.out, train ? dpred : nullptr, loss_dev,
                             eng->scratch(), st);
    }
    if (!train) return;
    // head backward (model.cpp:322-342); h holds h_final on the de-embedding GPU
    gemm<T>(true, false, d.d, d.out, b, h, d.d, dpred, d.out, static_cast<T*>(eng->deembed().g), d.out, true);
    gemm<T>(false, true, b, d.d, d.out, dpred, d.out, static_cast<const T*>(eng->deembed().w), d.out, dh, d.d,
            false);
  }

  template <typename T>
  void bwd(int mb, const int* order, const T* x, size_t b) {
    const Desc& d = eng->desc();
    cudaStream_t st = eng->stream();
    const size_t L = d.L;
    const T* cache_in = buf<T>(slot_id(mb, 0), L * b * d.d);
    const T* cache_z = buf<T>(slot_id(mb, 1), L * b * d.hid);
    T* dh = buf<T>(slot_id(mb, 2), b * d.d);
    T* dz = buf<T>(15, b * d.hid);
    T* da = buf<T>(16, b * d.hid);
    struct Applied {
      int sid;
      size_t bi;
    };
    std::vector<Applied> applied;
    for (size_t oi = 0; oi < d.s; ++oi) {
      const Range& r = d.part[static_cast<size_t>(order[oi] - 1)];
      for (size_t bi = 0; bi < r.count(); ++bi) applied.push_back({order[oi], bi});
    }
    // ---- backward (model.cpp:344-372), reverse application order
    int at = static_cast<int>(d.s) + 1;  // dL/dh_final sits at the de-embedding
    for (size_t ai = applied.size(); ai-- > 0;) {
      const Applied& a = applied[ai];
      const int own = eng->owner_of_stage(a.sid);
      eng->move(dh, b * d.d * sizeof(T), at, a.sid);
      at = a.sid;
      if (!eng->mine(own)) continue;
      const T* w1 = static_cast<const T*>(eng->stage(a.sid).w) + a.bi * blk_params();
      const T* w2 = w1 + d.d * d.hid;
      T* gw1 = static_cast<T*>(eng->stage(a.sid).g) + a.bi * blk_params();
      T* gw2 = gw1 + d.d * d.hid;
      const T* cin = cache_in + ai * b * d.d;
      const T* cz = cache_z + ai * b * d.hid;
      gemm<T>(false, true, b, d.hid, d.d, dh, d.d, w2, d.d, dz, d.hid, false);   // dz = dh W2^T
      k::act_bwd<T>(d.act, cz, dz, da, b * d.hid, st);                         // da = dz act'(z)
      gemm<T>(true, false, d.d, d.hid, b, cin, d.d, da, d.hid, gw1, d.hid, true);  // gW1 += in^T da
      gemm<T>(true, false, d.hid, d.d, b, cz, d.hid, dh, d.d, gw2, d.d, true);     // gW2 += z^T dh
      gemm<T>(false, true, b, d.d, d.hid, da, d.hid, w1, d.hid, dh, d.d, true);    // dh += da W1^T
    }
    eng->move(dh, b * d.d * sizeof(T), at, 0);
    if (eng->mine(eng->owner_of_embed()))
      gemm<T>(true, false, d.in, d.d, b, x, d.in, dh, d.d, static_cast<T*>(eng->embed().g), d.d, true);
  }

  void mb_forward(int mb, const int* order, const void* x, const void* y, size_t rows, bool train,
                  double* loss_dev) override {
    const int slot = train ? mb : 0;
    if (eng->fp64())
      fwd<double>(slot, order, static_cast<const double*>(x), y, rows, train, loss_dev, nullptr);
    else
      fwd<float>(slot, order, static_cast<const float*>(x), y, rows, train, loss_dev, nullptr);
  }
  void mb_backward(int mb, const int* order, const void* x, size_t rows) override {
    if (eng->fp64())
      bwd<double>(mb, order, static_cast<const double*>(x), rows);
    else
      bwd<float>(mb, order, static_cast<const float*>(x), rows);
  }
  void predict(const int* order, const void* x, size_t rows, void* pred) override {
    if (eng->fp64())
      fwd<double>(0, order, static_cast<const double*>(x), nullptr, rows, false, nullptr, static_cast<double*>(pred));
    else
      fwd<float>(0, order, static_cast<const float*>(x), nullptr, rows, false, nullptr, static_cast<float*>(pred));
  }
};

std::unique_ptr<BlockImpl> make_mlp_block(Engine* e) { return std::make_unique<MlpBlock>(e); }

}  // namespace ckf
