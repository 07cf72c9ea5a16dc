// xcls_gpu.hpp -- C++ drop-in shim for the reference's hot-path API (namespace xcls,
// /root/reference/proj/include/xcls) over the C ABI of include/xknn.h.
//
// The types and functions keep the reference's names, argument meaning, host-side data layout
// (row-major std::vector<float> matrices, u32 class ids, CSR graphs) and error behaviour
// (exceptions derived from Error, one per errors.hpp:10-54 class).  A caller switches with
//     namespace xcls = xcls_gpu;
// and links libxcls_gpu.so (+ libxknn.so).  Every call copies its host inputs to the current CUDA
// device, runs the sm_100a kernels of libxknn.so, and copies the results back; the large-N path
// (one process per GPU, device-resident shards, no host matrices) is xknn.h / HybridSimFc.
//
//   reference                                             here
//   ShardLayout                 knn_graph.hpp:30-41       ShardLayout (xknn_shard_range)
//   KnnGraph, CompressedKnnGraph knn_graph.hpp:15-55      KnnGraph, CompressedKnnGraph (host CSR)
//   ActiveSet, SelectionConfig  knn_softmax.hpp:15-30     same
//   select_active_classes(KnnGraph)        :37-38        xknn_select_full_graph
//   select_active_classes(span<Compressed>) :44-46       a select-only layer holding the P
//                                                         shards' slices with per-slice ranks
//   knn_softmax_forward_backward            :51-53       xknn_knn_softmax_fwd_bwd
//   full_softmax_forward_backward           :56-57       the same over full_active_set
//   build_graph_bruteforce      knn_graph.hpp:57          xknn_graph_bruteforce
//   HybridSim (fc half)         parallel.hpp:170-224      HybridSimFc (xknn_layer_*, xknn_step)
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "xknn.h"

namespace xcls_gpu {

// ---- errors.hpp:10-54 ---------------------------------------------------------------------
class Error : public std::runtime_error {
 public:
  Error(xknn_status_t code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  xknn_status_t code() const { return code_; }

 private:
  xknn_status_t code_;
};
#define XCLS_GPU_ERROR(Name, Code)                                                 \
  class Name : public Error {                                                      \
   public:                                                                         \
    explicit Name(const std::string& m) : Error(Code, m) {}                        \
  };
XCLS_GPU_ERROR(ShapeMismatch, XKNN_ERR_SHAPE_MISMATCH)
XCLS_GPU_ERROR(LabelOutOfRange, XKNN_ERR_LABEL_OUT_OF_RANGE)
XCLS_GPU_ERROR(KTooLarge, XKNN_ERR_K_TOO_LARGE)
XCLS_GPU_ERROR(EmptyShard, XKNN_ERR_EMPTY_SHARD)
XCLS_GPU_ERROR(MTooSmall, XKNN_ERR_M_TOO_SMALL)
XCLS_GPU_ERROR(LabelNotActive, XKNN_ERR_LABEL_NOT_ACTIVE)
XCLS_GPU_ERROR(InvalidArgument, XKNN_ERR_INVALID_ARGUMENT)
XCLS_GPU_ERROR(IoError, XKNN_ERR_IO)
XCLS_GPU_ERROR(ConfigError, XKNN_ERR_CONFIG)
XCLS_GPU_ERROR(DeviceError, XKNN_ERR_CUDA)  // CUDA / NCCL / out of device memory / unsupported
#undef XCLS_GPU_ERROR
class ZeroNormRow : public Error {
 public:
  ZeroNormRow(const std::string& m, std::size_t row) : Error(XKNN_ERR_ZERO_NORM_ROW, m), row(row) {}
  std::size_t row;
};
// throws the exception class of a failed xknn call (message: xknn_last_error_message)
void check(xknn_status_t s);

// ---- matrices and graphs ------------------------------------------------------------------
struct DenseMatrix {  // row-major fp32, as matrix.hpp
  std::size_t rows = 0, cols = 0;
  std::vector<float> data;
  DenseMatrix() = default;
  DenseMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0f) {}
  float* row(std::size_t i) { return data.data() + i * cols; }
  const float* row(std::size_t i) const { return data.data() + i * cols; }
};

struct ShardLayout {  // contiguous class blocks, the first num_classes % num_shards one larger
  std::size_t num_classes = 0, num_shards = 1;
  std::pair<std::size_t, std::size_t> class_range(std::size_t shard) const;
  std::size_t shard_size(std::size_t shard) const;
  std::size_t shard_of(std::uint32_t cls) const;
};

struct KnnGraph {  // num_classes x k row-major, row c = neighbours of class c (self first)
  std::size_t num_classes = 0, k = 0;
  std::vector<std::uint32_t> flat;
  std::span<const std::uint32_t> neighbors(std::size_t c) const { return {flat.data() + c * k, k}; }
  bool operator==(const KnnGraph& o) const {
    return num_classes == o.num_classes && k == o.k && flat == o.flat;
  }
};

struct CompressedKnnGraph {  // one shard's CSR over all N classes: only its own neighbours kept
  std::size_t num_classes = 0;
  std::size_t shard = 0;
  std::vector<std::uint32_t> shard_classes;   // classes owned by this shard, sorted
  std::vector<std::uint32_t> k_per_class;     // [num_classes]
  std::vector<std::uint64_t> offsets;         // [num_classes], exclusive prefix of k_per_class
  std::vector<std::uint32_t> flat_neighbors;  // [sum k_per_class]
  // the neighbours of `label` owned by this shard; LabelOutOfRange past num_classes
  std::span<const std::uint32_t> slice(std::uint32_t label) const;
};

// compress_graph (knn_graph.cpp:235-266) and quick_access (:268-274) on the host
CompressedKnnGraph compress_graph(const KnnGraph& g, const ShardLayout& layout, std::size_t shard);
std::vector<std::span<const std::uint32_t>> quick_access(const CompressedKnnGraph& cg,
                                                         std::span<const std::uint32_t> labels);
// save_graph / load_graph (knn_graph.cpp:276-311): XKNN v1 files (xknn_graph_save_rows/_load_rows)
void save_graph(const KnnGraph& g, const std::string& path);
KnnGraph load_graph(const std::string& path);

// ---- selection ----------------------------------------------------------------------------
struct ActiveSet {
  std::vector<std::uint32_t> class_indices;  // sorted, unique
  bool contains_all_labels = false;
  std::size_t size() const { return class_indices.size(); }
  std::optional<std::size_t> position_of(std::uint32_t cls) const;
};
ActiveSet full_active_set(std::size_t n_total);

struct SelectionConfig {
  std::size_t m_active = 0;
  std::uint64_t rng_seed = 0;
};

ActiveSet select_active_classes(const KnnGraph& g, std::span<const std::uint32_t> labels,
                                const SelectionConfig& cfg, std::size_t n_total);
ActiveSet select_active_classes(std::span<const CompressedKnnGraph> shards,
                                std::span<const std::uint32_t> labels,
                                const SelectionConfig& cfg, std::size_t n_total);

// ---- softmax ------------------------------------------------------------------------------
struct LossAndGrad {
  double loss = 0.0;
  DenseMatrix grad_logits;    // B x |active|
  DenseMatrix grad_features;  // B x D, w.r.t. x_norm
  DenseMatrix grad_weights;   // N x D, zero outside the active rows
};
LossAndGrad knn_softmax_forward_backward(const DenseMatrix& x_norm, const DenseMatrix& w_norm,
                                         std::span<const std::uint32_t> labels,
                                         const ActiveSet& active, float scale);
LossAndGrad full_softmax_forward_backward(const DenseMatrix& x_norm, const DenseMatrix& w_norm,
                                          std::span<const std::uint32_t> labels, float scale);

// build_graph_bruteforce (knn_graph.cpp:124-145): exact, bit-identical rows
KnnGraph build_graph_bruteforce(const DenseMatrix& w_norm, std::size_t k);

// ---- the fc half of HybridSim -------------------------------------------------------------
struct FcOptions {  // SimOptions (parallel.hpp:130-146) fields of the fc layer
  float scale = 30.0f;
  float momentum = 0.9f;
  float weight_decay = 0.0f;
  SelectionConfig selection;
  std::size_t max_batch = 0;          // largest global batch
  int precision = XKNN_PREC_BF16;     // xknn_precision_t
  std::size_t active_capacity = 0;    // xknn_config_t::active_capacity (0 = worst case)
};
struct FcStepResult {
  double loss = 0.0;
  std::size_t active_classes = 0;   // |ActiveSet|
};

// HybridSim (parallel.hpp:170-224) restricted to the fc layer of one worker/GPU: its class shard
// of ShardLayout(num_classes, world), the SgdMomentum velocity and the CompressedKnnGraph, all
// device resident.  world > 1: one process per GPU over an NCCL communicator (ncclComm_t).
// train_step takes the already-extracted features of this rank's B/P rows (the reference's
// feature extractor is outside this path) and returns d loss / d features for them.
class HybridSimFc {
 public:
  HybridSimFc(std::size_t num_classes, std::size_t dim, const FcOptions& opt, int rank = 0,
              int world = 1, void* nccl_comm = nullptr);
  ~HybridSimFc();
  HybridSimFc(const HybridSimFc&) = delete;
  HybridSimFc& operator=(const HybridSimFc&) = delete;

  // set_shard_graphs (parallel.cpp:381-388).  world == 1: all P shards of the reference's
  // simulated workers (selection over their slices, ranks within each slice); world > 1:
  // shards[rank] (this process's shard) or a span of exactly this one.
  void set_shard_graphs(std::span<const CompressedKnnGraph> shards);
  // load_model / fc_weights (parallel.cpp:401-431) for this rank's shard rows
  void load_model(const DenseMatrix& w_shard);
  DenseMatrix fc_weights() const;
  DenseMatrix velocity() const;
  FcStepResult train_step(const DenseMatrix& features, std::span<const std::uint32_t> labels,
                          float lr, DenseMatrix* grad_features = nullptr);
  std::pair<std::size_t, std::size_t> shard_range() const { return {begin_, end_}; }

 private:
  xknn_layer_t* h_ = nullptr;
  void* stream_ = nullptr;
  std::size_t n_, d_, begin_ = 0, end_ = 0;
  int rank_, world_;
};

}  // namespace xcls_gpu
