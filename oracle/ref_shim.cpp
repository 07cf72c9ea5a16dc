// ref_shim.cpp -- C ABI over the UNMODIFIED reference library (xcls::, /root/reference/proj).
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  `make -C oracle ref` (oracle/Makefile) compiles this file with
// the reference's own sources (read in place from /root/reference/proj/src, never copied) into
// oracle/_ref/libxcls_ref.so.  It is used (1) to pin the C restatement in oracle/xknn_oracle.c,
// (2) to generate the golden fixtures under tests/golden/, and (3) as bench.py's
// `--impl reference` / cpu_baseline arm, which times the reference's stock
// HybridSim::train_step (parallel.cpp:433-677) in SoftmaxMode::kKnn.
//
// Every entry point catches xcls::Error and returns the status code of include/xknn.h.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "xcls/errors.hpp"
#include "xcls/knn_graph.hpp"
#include "xcls/knn_softmax.hpp"
#include "xcls/matrix.hpp"
#include "xcls/parallel.hpp"
#include "xcls/softmax.hpp"
#include "xcls/sparsify.hpp"

using namespace xcls;

namespace {

int code_of(const std::exception& e) {
  if (dynamic_cast<const ShapeMismatch*>(&e)) return 1;
  if (dynamic_cast<const ZeroNormRow*>(&e)) return 2;
  if (dynamic_cast<const LabelOutOfRange*>(&e)) return 3;
  if (dynamic_cast<const KTooLarge*>(&e)) return 4;
  if (dynamic_cast<const EmptyShard*>(&e)) return 5;
  if (dynamic_cast<const MTooSmall*>(&e)) return 6;
  if (dynamic_cast<const LabelNotActive*>(&e)) return 7;
  if (dynamic_cast<const InvalidArgument*>(&e)) return 8;
  return 99;
}

#define GUARD(...)                                   \
  try {                                              \
    __VA_ARGS__;                                          \
    return 0;                                        \
  } catch (const ZeroNormRow& e) {                   \
    g_bad_row = e.row;                               \
    return 2;                                        \
  } catch (const std::exception& e) {                \
    return code_of(e);                               \
  }

thread_local uint64_t g_bad_row = 0;

DenseMatrix mat(uint64_t r, uint64_t c, const float* p) {
  return DenseMatrix(r, c, std::vector<float>(p, p + r * c));
}

std::vector<CompressedKnnGraph> shards_of(uint64_t n, uint64_t p, const uint32_t* const* kpc,
                                          const uint64_t* const* off,
                                          const uint32_t* const* flat) {
  std::vector<CompressedKnnGraph> v(p);
  ShardLayout layout{n, p};
  for (uint64_t s = 0; s < p; ++s) {
    auto& cg = v[s];
    cg.num_classes = n;
    cg.shard = s;
    auto [b, e] = layout.class_range(s);
    for (auto c = b; c < e; ++c) cg.shard_classes.push_back(static_cast<uint32_t>(c));
    cg.k_per_class.assign(kpc[s], kpc[s] + n);
    cg.offsets.assign(off[s], off[s] + n);
    uint64_t total = n ? off[s][n - 1] + kpc[s][n - 1] : 0;
    cg.flat_neighbors.assign(flat[s], flat[s] + total);
  }
  return v;
}

}  // namespace

extern "C" {

uint64_t ref_last_bad_row() { return g_bad_row; }

int ref_l2_normalize_rows(uint64_t rows, uint64_t cols, const float* in, float* out,
                          float* norms) {
  GUARD({
    auto r = l2_normalize_rows_cached(mat(rows, cols, in));
    std::memcpy(out, r.normalized.data.data(), rows * cols * sizeof(float));
    std::memcpy(norms, r.norms.data(), rows * sizeof(float));
  })
}

int ref_softmax_xent(uint64_t m, uint64_t c, const float* logits, const uint32_t* labels,
                     double* loss, float* grad) {
  GUARD({
    auto r = softmax_xent(mat(m, c, logits), std::span<const uint32_t>(labels, m));
    *loss = r.loss;
    std::memcpy(grad, r.grad_logits.data.data(), m * c * sizeof(float));
  })
}

int ref_build_graph_bruteforce(uint64_t n, uint64_t d, const float* w, uint64_t k,
                               uint32_t* out) {
  GUARD({
    auto g = build_graph_bruteforce(mat(n, d, w), k);
    std::memcpy(out, g.flat.data(), n * k * sizeof(uint32_t));
  })
}

int ref_build_graph_ring(uint64_t n, uint64_t d, const float* w, uint64_t p, uint64_t k,
                         uint64_t kprime, int threaded, uint32_t* out) {
  GUARD({
    auto blocks = split_rows(mat(n, d, w), ShardLayout{n, p});
    auto g = build_graph_ring(blocks, k, kprime, nullptr, threaded != 0);
    std::memcpy(out, g.flat.data(), n * k * sizeof(uint32_t));
  })
}

// topk_divide_conquer / CompressionState (sparsify.cpp)
int ref_topk(uint64_t len, const float* t, uint64_t k, uint64_t m_chunks, uint64_t* out_idx,
             float* out_val) {
  GUARD({
    auto r = topk_divide_conquer(std::span<const float>(t, len), k, m_chunks);
    std::memcpy(out_idx, r.indices.data(), r.indices.size() * sizeof(uint64_t));
    std::memcpy(out_val, r.values.data(), r.values.size() * sizeof(float));
  })
}

void* ref_dgc_create(double ratio, float momentum) {
  try {
    return new CompressionState(ratio, momentum);
  } catch (...) {
    return nullptr;
  }
}

int ref_dgc_step(void* h, uint32_t layer, uint64_t len, const float* g, uint64_t m_chunks,
                 uint64_t* out_idx, float* out_val, uint64_t* count) {
  GUARD({
    auto s = static_cast<CompressionState*>(h)->compress_step(
        layer, std::span<const float>(g, len), m_chunks);
    std::memcpy(out_idx, s.indices.data(), s.indices.size() * sizeof(uint64_t));
    std::memcpy(out_val, s.values.data(), s.values.size() * sizeof(float));
    *count = s.indices.size();
  })
}

int ref_dgc_set_sparsity(void* h, double r) {
  GUARD({ static_cast<CompressionState*>(h)->set_sparsity_ratio(r); })
}

int ref_dgc_residual(void* h, uint32_t layer, uint64_t len, float* out) {
  GUARD({
    auto r = static_cast<CompressionState*>(h)->residual(layer);
    if (r.size() != len) throw ShapeMismatch("residual length");
    std::memcpy(out, r.data(), len * sizeof(float));
  })
}

void ref_dgc_destroy(void* h) { delete static_cast<CompressionState*>(h); }

// save_graph / load_graph (knn_graph.cpp:276-311).  load: *n and *k out; flat (>= n*k) may be
// NULL to query the sizes only.
int ref_save_graph(const char* path, uint64_t n, uint64_t k, const uint32_t* g_flat) {
  GUARD({
    KnnGraph g;
    g.num_classes = n;
    g.k = k;
    g.flat.assign(g_flat, g_flat + n * k);
    save_graph(g, path);
  })
}

int ref_load_graph(const char* path, uint64_t* n, uint64_t* k, uint32_t* flat) {
  GUARD({
    auto g = load_graph(path);
    *n = g.num_classes;
    *k = g.k;
    if (flat) std::memcpy(flat, g.flat.data(), g.flat.size() * sizeof(uint32_t));
  })
}

// Returns Σ kept through *total; arrays sized by caller (flat_out ≥ n*k).
int ref_compress_graph(uint64_t n, uint64_t k, const uint32_t* g_flat, uint64_t p, uint64_t shard,
                       uint32_t* kpc, uint64_t* offsets, uint32_t* flat_out, uint64_t* total) {
  GUARD({
    KnnGraph g;
    g.num_classes = n;
    g.k = k;
    g.flat.assign(g_flat, g_flat + n * k);
    auto cg = compress_graph(g, ShardLayout{n, p}, shard);
    std::memcpy(kpc, cg.k_per_class.data(), n * sizeof(uint32_t));
    std::memcpy(offsets, cg.offsets.data(), n * sizeof(uint64_t));
    std::memcpy(flat_out, cg.flat_neighbors.data(), cg.flat_neighbors.size() * sizeof(uint32_t));
    *total = cg.flat_neighbors.size();
  })
}

int ref_select_active_full(uint64_t n, uint64_t k, const uint32_t* g_flat, const uint32_t* labels,
                           uint64_t b, uint64_t m_active, uint64_t seed, uint32_t* out,
                           uint64_t* count, int* contains_all) {
  GUARD({
    KnnGraph g;
    g.num_classes = n;
    g.k = k;
    g.flat.assign(g_flat, g_flat + n * k);
    auto a = select_active_classes(g, std::span<const uint32_t>(labels, b),
                                   SelectionConfig{m_active, seed}, n);
    std::memcpy(out, a.class_indices.data(), a.size() * sizeof(uint32_t));
    *count = a.size();
    *contains_all = a.contains_all_labels;
  })
}

int ref_select_active_shards(uint64_t n, uint64_t p, const uint32_t* const* kpc,
                             const uint64_t* const* off, const uint32_t* const* flat,
                             const uint32_t* labels, uint64_t b, uint64_t m_active, uint64_t seed,
                             uint32_t* out, uint64_t* count, int* contains_all) {
  GUARD({
    auto shards = shards_of(n, p, kpc, off, flat);
    auto a = select_active_classes(std::span<const CompressedKnnGraph>(shards),
                                   std::span<const uint32_t>(labels, b),
                                   SelectionConfig{m_active, seed}, n);
    std::memcpy(out, a.class_indices.data(), a.size() * sizeof(uint32_t));
    *count = a.size();
    *contains_all = a.contains_all_labels;
  })
}

int ref_knn_softmax_forward_backward(uint64_t b, uint64_t n, uint64_t d, const float* x_norm,
                                     const float* w_norm, const uint32_t* labels,
                                     const uint32_t* active, uint64_t m_act, float scale,
                                     double* loss, float* grad_logits, float* grad_features,
                                     float* grad_weights) {
  GUARD({
    ActiveSet a;
    a.class_indices.assign(active, active + m_act);
    auto r = knn_softmax_forward_backward(mat(b, d, x_norm), mat(n, d, w_norm),
                                          std::span<const uint32_t>(labels, b), a, scale);
    *loss = r.loss;
    if (grad_logits)
      std::memcpy(grad_logits, r.grad_logits.data.data(), b * m_act * sizeof(float));
    if (grad_features)
      std::memcpy(grad_features, r.grad_features.data.data(), b * d * sizeof(float));
    if (grad_weights)
      std::memcpy(grad_weights, r.grad_weights.data.data(), n * d * sizeof(float));
  })
}

int ref_distributed_softmax_xent(uint64_t p, uint64_t m, uint64_t n, const float* const* logits,
                                 const uint32_t* labels, double* loss, float* const* grads) {
  GUARD({
    ShardLayout layout{n, p};
    std::vector<DenseMatrix> sl;
    for (uint64_t s = 0; s < p; ++s) sl.push_back(mat(m, layout.shard_size(s), logits[s]));
    auto r = distributed_softmax_xent(sl, std::span<const uint32_t>(labels, m), layout);
    *loss = r.loss;
    for (uint64_t s = 0; s < p; ++s)
      std::memcpy(grads[s], r.grad_slices[s].data.data(), r.grad_slices[s].size() * sizeof(float));
  })
}

// Feature-side gradient of one micro-batch step, composed from the reference's own free
// functions exactly as HybridSim::train_step does (parallel.cpp:479-503, :544-585):
// grad_feat = l2_normalize_backward(f̂, norms, all_reduce_sum_w(s·G_w·W_sub_w)).
int ref_fc_feature_grad(uint64_t n, uint64_t d, uint64_t p, const float* w, const float* x,
                        const uint32_t* labels, uint64_t b, const uint32_t* active,
                        uint64_t m_act, float scale, double* loss, float* grad_feat) {
  GUARD({
    ShardLayout layout{n, p};
    std::vector<std::vector<uint32_t>> cols(p);
    std::vector<DenseMatrix> w_sub(p), logits(p);
    auto f = l2_normalize_rows_cached(mat(b, d, x));
    for (uint64_t s = 0; s < p; ++s) {
      auto [bg, en] = layout.class_range(s);
      for (uint64_t i = 0; i < m_act; ++i)
        if (active[i] >= bg && active[i] < en) cols[s].push_back(active[i]);
      auto wn = l2_normalize_rows_cached(mat(en - bg, d, w + bg * d));
      DenseMatrix sub(cols[s].size(), d);
      for (size_t i = 0; i < cols[s].size(); ++i)
        std::copy_n(wn.normalized.data.data() + (cols[s][i] - bg) * d, d,
                    sub.data.data() + i * d);
      w_sub[s] = std::move(sub);
      DenseMatrix lg = matmul(f.normalized, w_sub[s], true);
      for (float& v : lg.data) v *= scale;
      logits[s] = std::move(lg);
    }
    auto sm = distributed_softmax_xent_cols(logits, cols, std::span<const uint32_t>(labels, b));
    std::vector<DenseMatrix> part(p);
    for (uint64_t s = 0; s < p; ++s) {
      DenseMatrix gf = matmul(sm.grad_slices[s], w_sub[s]);
      for (float& v : gf.data) v *= scale;
      part[s] = std::move(gf);
    }
    auto red = all_reduce_sum(part);
    auto g = l2_normalize_backward(f.normalized, f.norms, red[0]);
    *loss = sm.loss;
    std::memcpy(grad_feat, g.data.data(), b * d * sizeof(float));
  })
}

// ---- The stock HybridSim trainer (the reference arm of bench.py) ----------------------------
// The feature extractor is configured as a single D×D linear layer and loaded with the identity
// (exact: x·Iᵀ + 0 == x in fp32), so the fc half sees exactly the supplied features.
struct RefSim {
  HybridSim sim;
  uint64_t n, d;
};

void* ref_sim_create(uint64_t n, uint64_t d, uint64_t p, int threads, float scale, float momentum,
                     float wd, const float* w) {
  try {
    MlpConfig mc;
    mc.input_dim = d;
    mc.hidden = {};
    mc.output_dim = d;
    SimOptions o;
    o.scale = scale;
    o.momentum = momentum;
    o.weight_decay = wd;
    o.worker_threads = threads != 0;
    auto* r = new RefSim{HybridSim(WorkerTopology::make(p, n), mc, 1, 2, o), n, d};
    HybridSim::ModelView v = r->sim.model();
    auto& W = v.mlp.weights[0];
    std::fill(W.data.begin(), W.data.end(), 0.0f);
    for (uint64_t i = 0; i < d; ++i) W.at(i, i) = 1.0f;
    std::fill(v.mlp.biases[0].data.begin(), v.mlp.biases[0].data.end(), 0.0f);
    v.fc_weight = mat(n, d, w);
    r->sim.load_model(v);
    return r;
  } catch (...) {
    return nullptr;
  }
}

// Re-installs the identity feature extractor (train_step's FE optimizer moves it every step);
// the fc shards and their velocity are untouched (load_model keeps Worker::fc_opt).  Parity
// tests call this between steps; the timed baseline does not.
int ref_sim_reset_fe(void* h) {
  auto* r = static_cast<RefSim*>(h);
  GUARD({
    HybridSim::ModelView v = r->sim.model();
    auto& W = v.mlp.weights[0];
    std::fill(W.data.begin(), W.data.end(), 0.0f);
    for (uint64_t i = 0; i < r->d; ++i) W.at(i, i) = 1.0f;
    std::fill(v.mlp.biases[0].data.begin(), v.mlp.biases[0].data.end(), 0.0f);
    r->sim.load_model(v);
  })
}

int ref_sim_set_graphs(void* h, uint64_t p, const uint32_t* const* kpc, const uint64_t* const* off,
                       const uint32_t* const* flat) {
  auto* r = static_cast<RefSim*>(h);
  GUARD(r->sim.set_shard_graphs(shards_of(r->n, p, kpc, off, flat)))
}

int ref_sim_step_mb(void* h, const float* x, const uint32_t* labels, uint64_t b,
                    uint64_t m_active, uint64_t seed, float lr, uint64_t micro_batches,
                    double* loss, uint64_t* active_classes) {
  auto* r = static_cast<RefSim*>(h);
  GUARD({
    LabeledBatch batch{mat(b, r->d, x), std::vector<uint32_t>(labels, labels + b)};
    StepOptions so;
    so.mode = SoftmaxMode::kKnn;
    so.lr = lr;
    so.micro_batches = micro_batches;
    so.selection = SelectionConfig{m_active, seed};
    auto res = r->sim.train_step(batch, so);
    *loss = res.loss;
    *active_classes = res.active_classes;
  })
}

int ref_sim_step(void* h, const float* x, const uint32_t* labels, uint64_t b, uint64_t m_active,
                 uint64_t seed, float lr, double* loss, uint64_t* active_classes) {
  auto* r = static_cast<RefSim*>(h);
  GUARD({
    LabeledBatch batch{mat(b, r->d, x), std::vector<uint32_t>(labels, labels + b)};
    StepOptions so;
    so.mode = SoftmaxMode::kKnn;
    so.lr = lr;
    so.micro_batches = 1;
    so.selection = SelectionConfig{m_active, seed};
    auto res = r->sim.train_step(batch, so);
    *loss = res.loss;
    *active_classes = res.active_classes;
  })
}

int ref_sim_get_weights(void* h, float* out) {
  auto* r = static_cast<RefSim*>(h);
  GUARD({
    auto w = r->sim.fc_weights();
    std::memcpy(out, w.data.data(), w.size() * sizeof(float));
  })
}

void ref_sim_destroy(void* h) { delete static_cast<RefSim*>(h); }

}  // extern "C"
