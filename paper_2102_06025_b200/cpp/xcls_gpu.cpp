// xcls_gpu.cpp -- the C++ shim of include/xcls_gpu.hpp over the C ABI (include/xknn.h).
// Host matrices go to the current CUDA device through a small RAII buffer, the libxknn.so entry
// points run there, results come back.  No arithmetic of the path runs here: the shim only moves
// data and assembles the reference's host-side types (CSR layout, dense gradient rows).
#include "xcls_gpu.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

namespace xcls_gpu {

void check(xknn_status_t s) {
  if (s == XKNN_OK) return;
  const std::string m = xknn_last_error_message();
  switch (s) {
    case XKNN_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
    case XKNN_ERR_ZERO_NORM_ROW: throw ZeroNormRow(m, xknn_last_error_row());
    case XKNN_ERR_LABEL_OUT_OF_RANGE: throw LabelOutOfRange(m);
    case XKNN_ERR_K_TOO_LARGE: throw KTooLarge(m);
    case XKNN_ERR_EMPTY_SHARD: throw EmptyShard(m);
    case XKNN_ERR_M_TOO_SMALL: throw MTooSmall(m);
    case XKNN_ERR_LABEL_NOT_ACTIVE: throw LabelNotActive(m);
    case XKNN_ERR_INVALID_ARGUMENT: throw InvalidArgument(m);
    case XKNN_ERR_IO: throw IoError(m);
    case XKNN_ERR_CONFIG: throw ConfigError(m);
    default: throw DeviceError(std::string(xknn_status_string(s)) + ": " + m);
  }
}

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
struct DevBuf {  // device copy of a host array (or scratch of n elements)
  T* p = nullptr;
  std::size_t n = 0;
  explicit DevBuf(std::size_t count) : n(count) {
    cuda_check(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)), "cudaMalloc");
  }
  DevBuf(const T* host, std::size_t count) : DevBuf(count) {
    if (count)
      cuda_check(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  void to_host(T* host, std::size_t count) const {
    if (count)
      cuda_check(cudaMemcpy(host, p, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// P shards' slices of every class concatenated in shard order, each entry ranked within its own
// slice: the span<CompressedKnnGraph> selection on one layer (xknn_layer_set_graph_csr_ranked)
void merge_shards(std::span<const CompressedKnnGraph> shards, std::size_t n,
                  std::vector<std::uint32_t>& kpc, std::vector<std::uint64_t>& off,
                  std::vector<std::uint32_t>& flat, std::vector<std::uint32_t>& rank) {
  kpc.assign(n, 0);
  off.assign(n, 0);
  std::size_t total = 0;
  for (const auto& cg : shards) {
    if (cg.k_per_class.size() != n || cg.offsets.size() != n)
      throw ShapeMismatch("select_active_classes: shard graph size disagrees with class count");
    total += cg.flat_neighbors.size();
  }
  flat.clear();
  rank.clear();
  flat.reserve(total);
  rank.reserve(total);
  for (std::size_t c = 0; c < n; ++c) {
    off[c] = flat.size();
    for (const auto& cg : shards) {
      const auto sl = cg.slice(static_cast<std::uint32_t>(c));
      for (std::size_t r = 0; r < sl.size(); ++r) {
        flat.push_back(sl[r]);
        rank.push_back(static_cast<std::uint32_t>(r));
      }
    }
    kpc[c] = static_cast<std::uint32_t>(flat.size() - off[c]);
  }
}

}  // namespace

// ---- ShardLayout / graphs -------------------------------------------------------------------
std::pair<std::size_t, std::size_t> ShardLayout::class_range(std::size_t s) const {
  std::uint64_t b = 0, e = 0;
  check(xknn_shard_range(num_classes, num_shards, s, &b, &e));
  return {b, e};
}
std::size_t ShardLayout::shard_size(std::size_t s) const {
  auto [b, e] = class_range(s);
  return e - b;
}
std::size_t ShardLayout::shard_of(std::uint32_t cls) const {
  if (cls >= num_classes) throw LabelOutOfRange("ShardLayout::shard_of: class out of range");
  const std::size_t base = num_classes / num_shards, rem = num_classes % num_shards;
  const std::size_t big = rem * (base + 1);
  return cls < big ? cls / (base + 1) : rem + (cls - big) / base;
}

std::span<const std::uint32_t> CompressedKnnGraph::slice(std::uint32_t label) const {
  if (label >= num_classes) throw LabelOutOfRange("CompressedKnnGraph::slice: label out of range");
  return {flat_neighbors.data() + offsets[label], k_per_class[label]};
}

CompressedKnnGraph compress_graph(const KnnGraph& g, const ShardLayout& layout, std::size_t shard) {
  if (layout.num_classes != g.num_classes)
    throw ShapeMismatch("compress_graph: layout and graph disagree on the class count");
  auto [b, e] = layout.class_range(shard);
  CompressedKnnGraph cg;
  cg.num_classes = g.num_classes;
  cg.shard = shard;
  for (std::size_t c = b; c < e; ++c) cg.shard_classes.push_back(static_cast<std::uint32_t>(c));
  cg.k_per_class.assign(g.num_classes, 0);
  cg.offsets.assign(g.num_classes, 0);
  for (std::size_t c = 0; c < g.num_classes; ++c) {
    cg.offsets[c] = cg.flat_neighbors.size();
    for (std::uint32_t v : g.neighbors(c))
      if (v >= b && v < e) cg.flat_neighbors.push_back(v);
    cg.k_per_class[c] = static_cast<std::uint32_t>(cg.flat_neighbors.size() - cg.offsets[c]);
  }
  return cg;
}

std::vector<std::span<const std::uint32_t>> quick_access(const CompressedKnnGraph& cg,
                                                         std::span<const std::uint32_t> labels) {
  std::vector<std::span<const std::uint32_t>> out;
  out.reserve(labels.size());
  for (std::uint32_t y : labels) out.push_back(cg.slice(y));
  return out;
}

void save_graph(const KnnGraph& g, const std::string& path) {
  check(xknn_graph_save_rows(path.c_str(), g.num_classes, static_cast<std::uint32_t>(g.k), 0,
                             g.num_classes, g.flat.data(), 0, 1));
}

KnnGraph load_graph(const std::string& path) {
  std::uint32_t k = 0;
  // header first (class count and k), then the rows
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("load_graph: cannot open " + path);
  char hdr[16];
  const bool ok = std::fread(hdr, 1, 16, f) == 16;
  std::fclose(f);
  if (!ok) throw IoError("load_graph: truncated header");
  std::uint64_t n = 0;
  std::memcpy(&n, hdr + 8, 8);
  check(xknn_graph_load_rows(path.c_str(), n, 0, n, nullptr, 0, 0, &k));
  KnnGraph g;
  g.num_classes = n;
  g.k = k;
  g.flat.resize(n * k);
  check(xknn_graph_load_rows(path.c_str(), n, 0, n, g.flat.data(), g.flat.size(), 0, &k));
  return g;
}

KnnGraph build_graph_bruteforce(const DenseMatrix& w_norm, std::size_t k) {
  if (k > w_norm.rows) throw KTooLarge("build_graph: k exceeds class count");
  if (k == 0) throw InvalidArgument("build_graph: k must be positive");
  DevBuf<float> w(w_norm.data.data(), w_norm.data.size());
  DevBuf<std::uint32_t> out(w_norm.rows * k);
  std::uint64_t unc = 0;
  check(xknn_graph_bruteforce(w.p, w_norm.rows, w_norm.cols, static_cast<std::uint32_t>(k), 0,
                              out.p, nullptr, &unc));
  KnnGraph g;
  g.num_classes = w_norm.rows;
  g.k = k;
  g.flat.resize(w_norm.rows * k);
  out.to_host(g.flat.data(), g.flat.size());
  return g;
}

// ---- selection ------------------------------------------------------------------------------
std::optional<std::size_t> ActiveSet::position_of(std::uint32_t cls) const {
  auto it = std::lower_bound(class_indices.begin(), class_indices.end(), cls);
  if (it == class_indices.end() || *it != cls) return std::nullopt;
  return static_cast<std::size_t>(it - class_indices.begin());
}

ActiveSet full_active_set(std::size_t n_total) {
  ActiveSet a;
  a.class_indices.resize(n_total);
  for (std::size_t i = 0; i < n_total; ++i) a.class_indices[i] = static_cast<std::uint32_t>(i);
  a.contains_all_labels = true;
  return a;
}

ActiveSet select_active_classes(const KnnGraph& g, std::span<const std::uint32_t> labels,
                                const SelectionConfig& cfg, std::size_t n_total) {
  if (g.num_classes != n_total)
    throw ShapeMismatch("select_active_classes: graph size disagrees with class count");
  DevBuf<std::uint32_t> dg(g.flat.data(), g.flat.size());
  DevBuf<std::uint32_t> dl(labels.data(), labels.size());
  DevBuf<std::uint32_t> out(cfg.m_active);
  std::uint64_t cnt = 0;
  int all = 0;
  check(xknn_select_full_graph(dg.p, n_total, static_cast<std::uint32_t>(g.k), dl.p,
                               labels.size(), cfg.m_active, cfg.rng_seed, out.p, &cnt, &all,
                               nullptr));
  ActiveSet a;
  a.class_indices.resize(cnt);
  out.to_host(a.class_indices.data(), cnt);
  a.contains_all_labels = all != 0;
  return a;
}

ActiveSet select_active_classes(std::span<const CompressedKnnGraph> shards,
                                std::span<const std::uint32_t> labels,
                                const SelectionConfig& cfg, std::size_t n_total) {
  if (shards.empty()) throw InvalidArgument("select_active_classes: no shards");
  if (labels.empty()) throw InvalidArgument("select_active_classes: empty batch");
  std::vector<std::uint32_t> kpc, flat, rank;
  std::vector<std::uint64_t> off;
  merge_shards(shards, n_total, kpc, off, flat, rank);
  xknn_config_t c{};
  c.scale = 1.f;
  c.m_active = cfg.m_active;
  c.rng_seed = cfg.rng_seed;
  c.max_batch = labels.size();
  c.precision = XKNN_PREC_FP32_EXACT;
  c.flags = XKNN_FLAG_SELECT_ONLY | XKNN_FLAG_NO_GRAPH;
  xknn_layer_t* h = nullptr;
  check(xknn_layer_create(0, 1, n_total, 128, &c, nullptr, nullptr, &h));
  struct Guard {
    xknn_layer_t* h;
    ~Guard() { xknn_layer_destroy(h); }
  } guard{h};
  check(xknn_layer_set_graph_csr_ranked(h, kpc.data(), off.data(), flat.data(), rank.data(),
                                        flat.size(), 0));
  DevBuf<std::uint32_t> dl(labels.data(), labels.size());
  DevBuf<std::uint32_t> out(std::max<std::size_t>(cfg.m_active, 1));
  std::uint64_t cnt = 0;
  int all = 0;
  check(xknn_select(h, dl.p, labels.size(), out.p, &cnt, &all));
  ActiveSet a;
  a.class_indices.resize(cnt);
  out.to_host(a.class_indices.data(), cnt);
  a.contains_all_labels = all != 0;
  return a;
}

// ---- softmax --------------------------------------------------------------------------------
LossAndGrad knn_softmax_forward_backward(const DenseMatrix& x_norm, const DenseMatrix& w_norm,
                                         std::span<const std::uint32_t> labels,
                                         const ActiveSet& active, float scale) {
  if (x_norm.cols != w_norm.cols) throw ShapeMismatch("knn_softmax: feature dims disagree");
  if (labels.size() != x_norm.rows) throw ShapeMismatch("knn_softmax: one label per row required");
  if (active.size() == 0) throw InvalidArgument("knn_softmax: empty active set");
  const std::size_t b = x_norm.rows, d = x_norm.cols, n = w_norm.rows, m = active.size();
  DevBuf<float> dx(x_norm.data.data(), x_norm.data.size());
  DevBuf<float> dw(w_norm.data.data(), w_norm.data.size());
  DevBuf<std::uint32_t> dl(labels.data(), labels.size());
  DevBuf<std::uint32_t> da(active.class_indices.data(), m);
  DevBuf<float> gl(b * m), gf(b * d), gw(m * d);
  LossAndGrad out;
  check(xknn_knn_softmax_fwd_bwd(dx.p, b, dw.p, n, d, dl.p, da.p, m, scale, &out.loss, gl.p, gf.p,
                                 gw.p, nullptr));
  out.grad_logits = DenseMatrix(b, m);
  gl.to_host(out.grad_logits.data.data(), b * m);
  out.grad_features = DenseMatrix(b, d);
  gf.to_host(out.grad_features.data.data(), b * d);
  std::vector<float> rows(m * d);
  gw.to_host(rows.data(), m * d);
  out.grad_weights = DenseMatrix(n, d);  // dense N x D, zero outside the active rows
  for (std::size_t i = 0; i < m; ++i)
    std::memcpy(out.grad_weights.row(active.class_indices[i]), rows.data() + i * d,
                d * sizeof(float));
  return out;
}

LossAndGrad full_softmax_forward_backward(const DenseMatrix& x_norm, const DenseMatrix& w_norm,
                                          std::span<const std::uint32_t> labels, float scale) {
  return knn_softmax_forward_backward(x_norm, w_norm, labels, full_active_set(w_norm.rows), scale);
}

// ---- HybridSimFc ----------------------------------------------------------------------------
HybridSimFc::HybridSimFc(std::size_t num_classes, std::size_t dim, const FcOptions& opt, int rank,
                         int world, void* nccl_comm)
    : n_(num_classes), d_(dim), rank_(rank), world_(world) {
  xknn_config_t c{};
  c.scale = opt.scale;
  c.momentum = opt.momentum;
  c.weight_decay = opt.weight_decay;
  c.m_active = opt.selection.m_active;
  c.rng_seed = opt.selection.rng_seed;
  c.max_batch = opt.max_batch;
  c.precision = opt.precision;
  c.active_capacity = opt.active_capacity;
  cudaStream_t s = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_ = s;
  const xknn_status_t st = xknn_layer_create(rank, world, num_classes, dim, &c, nccl_comm, s, &h_);
  if (st != XKNN_OK) {
    cudaStreamDestroy(s);
    check(st);
  }
  std::uint64_t b = 0, e = 0;
  check(xknn_layer_shard(h_, &b, &e));
  begin_ = b;
  end_ = e;
}

HybridSimFc::~HybridSimFc() {
  if (h_) xknn_layer_destroy(h_);
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

void HybridSimFc::set_shard_graphs(std::span<const CompressedKnnGraph> shards) {
  if (world_ > 1) {
    const CompressedKnnGraph& cg = shards.size() == 1 ? shards[0] : shards[rank_];
    if (shards.size() != 1 && shards.size() != static_cast<std::size_t>(world_))
      throw ShapeMismatch("set_shard_graphs: need this rank's shard or one per rank");
    check(xknn_layer_set_graph_csr(h_, cg.k_per_class.data(), cg.offsets.data(),
                                   cg.flat_neighbors.data(), cg.flat_neighbors.size(), 0));
    return;
  }
  if (shards.empty()) throw InvalidArgument("set_shard_graphs: no shards");
  if (shards.size() == 1) {
    const CompressedKnnGraph& cg = shards[0];
    check(xknn_layer_set_graph_csr(h_, cg.k_per_class.data(), cg.offsets.data(),
                                   cg.flat_neighbors.data(), cg.flat_neighbors.size(), 0));
    return;
  }
  std::vector<std::uint32_t> kpc, flat, rank;
  std::vector<std::uint64_t> off;
  merge_shards(shards, n_, kpc, off, flat, rank);
  check(xknn_layer_set_graph_csr_ranked(h_, kpc.data(), off.data(), flat.data(), rank.data(),
                                        flat.size(), 0));
}

void HybridSimFc::load_model(const DenseMatrix& w) {
  if (w.rows != end_ - begin_ || w.cols != d_) throw ShapeMismatch("load_model: shard shape");
  check(xknn_layer_set_weights(h_, w.data.data(), 0));
}

DenseMatrix HybridSimFc::fc_weights() const {
  DenseMatrix w(end_ - begin_, d_);
  check(xknn_layer_get_weights(h_, w.data.data(), 0));
  return w;
}

DenseMatrix HybridSimFc::velocity() const {
  DenseMatrix v(end_ - begin_, d_);
  check(xknn_layer_get_velocity(h_, v.data.data(), 0));
  return v;
}

FcStepResult HybridSimFc::train_step(const DenseMatrix& features,
                                     std::span<const std::uint32_t> labels, float lr,
                                     DenseMatrix* grad_features) {
  if (features.cols != d_ || labels.size() != features.rows)
    throw ShapeMismatch("train_step: features / labels shape");
  DevBuf<float> x(features.data.data(), features.data.size());
  DevBuf<std::uint32_t> y(labels.data(), labels.size());
  DevBuf<double> loss(1);
  DevBuf<float> gf(grad_features ? features.data.size() : 1);
  check(xknn_step(h_, x.p, y.p, features.rows, lr, loss.p, grad_features ? gf.p : nullptr));
  check(xknn_layer_sync(h_));
  FcStepResult r;
  loss.to_host(&r.loss, 1);
  std::uint64_t tot = 0, loc = 0;
  check(xknn_layer_last_active(h_, &tot, &loc));
  r.active_classes = tot;
  if (grad_features) {
    *grad_features = DenseMatrix(features.rows, d_);
    gf.to_host(grad_features->data.data(), grad_features->data.size());
  }
  return r;
}

}  // namespace xcls_gpu
