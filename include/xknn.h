/*
 * xknn.h -- C ABI of the B200-native (sm_100a) model-parallel KNN-softmax layer.
 *
 * Drop-in boundary for the reference's fc hot path (namespace xcls, /root/reference/proj):
 * one layer object per GPU owns that GPU's contiguous class shard (ShardLayout,
 * knn_graph.cpp:94-115), its weight rows, momentum velocity and compressed KNN graph, and runs
 * the fc half of HybridSim::train_step (parallel.cpp:455-572, :638-668) on device: active-class
 * selection -> active-row gather/normalize -> logit GEMM + distributed softmax-CE -> feature- and
 * weight-gradient GEMMs -> sparse momentum-SGD row update.  Collectives are NCCL over
 * NVLink/NVSwitch on a caller-provided communicator.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "_dev" pointers are device memory of the layer's GPU,
 *    "_host" pointers host memory.  Row-major fp32 matrices, u32 class ids, u64 offsets.
 *  - Every call is ordered on the layer's CUDA stream.  Calls that return host values
 *    (counts, loss) synchronize that stream; the rest are asynchronous.
 *  - Errors are the xcls::Error classes of errors.hpp:10-54, one code each, checked before
 *    state changes as the reference does.  xknn_last_error_row() carries ZeroNormRow::row.
 *  - Thread-safety: a layer is single-owner (like HybridSim); distinct layers are independent.
 */
#ifndef XKNN_H_
#define XKNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:10-54 -> status codes */
typedef enum {
  XKNN_OK = 0,
  XKNN_ERR_SHAPE_MISMATCH = 1,     /* ShapeMismatch   */
  XKNN_ERR_ZERO_NORM_ROW = 2,      /* ZeroNormRow     */
  XKNN_ERR_LABEL_OUT_OF_RANGE = 3, /* LabelOutOfRange */
  XKNN_ERR_K_TOO_LARGE = 4,        /* KTooLarge       */
  XKNN_ERR_EMPTY_SHARD = 5,        /* EmptyShard      */
  XKNN_ERR_M_TOO_SMALL = 6,        /* MTooSmall       */
  XKNN_ERR_LABEL_NOT_ACTIVE = 7,   /* LabelNotActive  */
  XKNN_ERR_INVALID_ARGUMENT = 8,   /* InvalidArgument */
  XKNN_ERR_IO = 9,                 /* IoError         */
  XKNN_ERR_CONFIG = 10,            /* ConfigError     */
  XKNN_ERR_CUDA = 20,
  XKNN_ERR_NCCL = 21,
  XKNN_ERR_OUT_OF_MEMORY = 22,
  XKNN_ERR_UNSUPPORTED = 23
} xknn_status_t;

/* Arithmetic of the three fc GEMMs.  Selection, indices and the update are identical in all. */
typedef enum {
  /* tcgen05/TMEM tensor cores, bf16 operands, fp32 accumulation (the performance path; stated
     bf16 bound).  Needs 0 < scale <= 40 (fixed softmax stabilizer). */
  XKNN_PREC_BF16 = 0,
  /* CUDA-core fp32 with the reference's summation order (matrix.cpp:57-98), logits
     materialized and bit-identical; any scale */
  XKNN_PREC_FP32_EXACT = 1,
  /* tcgen05/TMEM tensor cores at fp32 accuracy from split operands, fp32 accumulation: logits
     GEMM tf32 leading product + two bf16 cross terms, gradient GEMMs bf16x3 (environment
     XKNN_FP32_GEMM=3xtf32: 3xTF32 throughout); within 1e-5 relative of the fp32 reference.
     Needs 0 < scale <= 40 (fixed softmax stabilizer). */
  XKNN_PREC_FP32 = 2
} xknn_precision_t;

typedef struct {
  float scale;           /* SimOptions::scale (parallel.hpp:140), cosine logit scale s      */
  float momentum;        /* SimOptions::momentum (parallel.hpp:141)                          */
  float weight_decay;    /* SimOptions::weight_decay (parallel.hpp:142)                      */
  uint64_t m_active;     /* SelectionConfig::m_active (knn_softmax.hpp:27), global M         */
  uint64_t rng_seed;     /* SelectionConfig::rng_seed (knn_softmax.hpp:28)                   */
  uint64_t max_batch;    /* largest global batch B a step will see (sizes scratch)           */
  int32_t precision;     /* xknn_precision_t                                                 */
  int32_t flags;         /* XKNN_FLAG_*                                                      */
  /* per-shard capacity of the active set (sizes W_sub, P~ and dW: P~ alone is max_batch x
     capacity); 0 = min(shard size, m_active), the worst case.  With uniform labels a shard
     holds ~m_active / world active classes; a step whose selection puts more on this shard
     fails with XKNN_ERR_OUT_OF_MEMORY before any parameter is touched.  C4 on 4 GPUs needs it
     (worst case: 8192 x 10M x 2 B = 164 GB of P~ per GPU). */
  uint64_t active_capacity;
} xknn_config_t;

/* The step's device work (selection .. update) is captured once per batch size into a CUDA
   graph and replayed; this flag launches it kernel by kernel instead. */
#define XKNN_FLAG_NO_GRAPH 1
/* A selection-only layer: graph + Algorithm-1 selection state, no weight/velocity shard and no
   step scratch (xknn_select only; parameter and step calls return XKNN_ERR_UNSUPPORTED). */
#define XKNN_FLAG_SELECT_ONLY 2

typedef struct xknn_layer xknn_layer_t;

/* Status of the last failing call on this thread, human readable. */
const char* xknn_status_string(xknn_status_t s);
const char* xknn_last_error_message(void);
/* ZeroNormRow::row of the last XKNN_ERR_ZERO_NORM_ROW (errors.hpp:18-22). */
uint64_t xknn_last_error_row(void);

/* ShardLayout::class_range (knn_graph.cpp:102-115), host-only, no GPU needed. */
xknn_status_t xknn_shard_range(uint64_t num_classes, uint64_t num_shards, uint64_t shard,
                               uint64_t* begin, uint64_t* end);

/* NCCL bootstrap helpers (plumbing for callers without nccl.h, e.g. ctypes/cgo):
   rank 0 calls xknn_nccl_unique_id, the caller broadcasts the 128 bytes, every rank calls
   xknn_nccl_comm_init on its device.  The returned handle is an ncclComm_t. */
xknn_status_t xknn_nccl_unique_id(uint8_t out_id[128]);
xknn_status_t xknn_nccl_comm_init(const uint8_t id[128], int world, int rank, void** comm);
xknn_status_t xknn_nccl_comm_destroy(void* comm);

/* HybridSim ctor (parallel.cpp:351-379) restricted to the fc shard of `rank`.
   comm: ncclComm_t over `world` ranks (NULL iff world == 1).  stream: cudaStream_t (NULL =
   the legacy default stream).  The velocity starts at zero (SgdMomentum::ensure_state,
   fccs.cpp:58-62).  The weights must be set before the first step. */
xknn_status_t xknn_layer_create(int rank, int world, uint64_t num_classes, uint64_t dim,
                                const xknn_config_t* cfg, void* comm, void* stream,
                                xknn_layer_t** out);
xknn_status_t xknn_layer_destroy(xknn_layer_t* h);
xknn_status_t xknn_layer_shard(const xknn_layer_t* h, uint64_t* begin, uint64_t* end);
xknn_status_t xknn_layer_set_config(xknn_layer_t* h, const xknn_config_t* cfg);

/* Weights of this shard, (end-begin) x dim fp32 row-major.  HybridSim::load_model /
   fc_weights (parallel.cpp:401-409, :425-431).  on_device selects the pointer space. */
xknn_status_t xknn_layer_set_weights(xknn_layer_t* h, const float* w, int on_device);
xknn_status_t xknn_layer_get_weights(xknn_layer_t* h, float* w, int on_device);
xknn_status_t xknn_layer_get_velocity(xknn_layer_t* h, float* v, int on_device);
/* Device pointer to the resident weight shard (for callers that initialise in place). */
xknn_status_t xknn_layer_weights_ptr(xknn_layer_t* h, float** w_dev);

/* HybridSim::set_shard_graphs (parallel.cpp:381-388): this shard's CompressedKnnGraph
   (knn_graph.hpp:46-55): k_per_class[num_classes], offsets[num_classes], flat[flat_len]. */
xknn_status_t xknn_layer_set_graph_csr(xknn_layer_t* h, const uint32_t* k_per_class,
                                       const uint64_t* offsets, const uint32_t* flat,
                                       uint64_t flat_len, int on_device);

/* In-place graph install for shards too large to stage twice (C4: ~10 GB of entries per GPU):
   xknn_layer_graph_buffers drops the installed graph and returns the layer-owned device arrays
   k_per_class[num_classes], offsets[num_classes], flat[flat_len] for the caller to fill (on any
   stream; synchronize before committing); xknn_layer_graph_commit validates them as
   xknn_layer_set_graph_csr does and installs them (collective when world > 1). */
xknn_status_t xknn_layer_graph_buffers(xknn_layer_t* h, uint64_t flat_len, uint32_t** k_per_class_dev,
                                       uint64_t** offsets_dev, uint32_t** flat_dev);
xknn_status_t xknn_layer_graph_commit(xknn_layer_t* h);

/* xknn_layer_set_graph_csr with a per-entry rank (rank[flat_len], NULL = the position within
   the class's list): lets one layer hold several shards' slices of a label concatenated into one
   list, each entry ranked within its own slice -- select_active_classes(span<CompressedKnnGraph>)
   (knn_softmax.cpp:117-134) over P shards on one device. */
xknn_status_t xknn_layer_set_graph_csr_ranked(xknn_layer_t* h, const uint32_t* k_per_class,
                                              const uint64_t* offsets, const uint32_t* flat,
                                              const uint32_t* rank, uint64_t flat_len,
                                              int on_device);

/* select_active_classes(span<CompressedKnnGraph>, ...) (knn_softmax.cpp:117-134 +
   finish_selection :17-81) for the global batch `labels_dev` (B u32, identical on every
   rank), executed shard-parallel.  Writes this shard's slice of the ActiveSet (sorted global
   class ids; the rank-order concatenation over ranks is ActiveSet::class_indices) to
   out_active_dev (capacity >= min(shard size, m_active)) and its length to *count_host;
   *contains_all_host = ActiveSet::contains_all_labels restricted to labels this shard owns.
   Synchronizes. */
xknn_status_t xknn_select(xknn_layer_t* h, const uint32_t* labels_dev, uint64_t batch,
                          uint32_t* out_active_dev, uint64_t* count_host,
                          int* contains_all_host);

/* One synchronous step of the fc half of HybridSim::train_step in SoftmaxMode::kKnn with one
   micro-batch (parallel.cpp:455-572, :638-668):
     features_local_dev : this rank's B/P rows of extracted features (fp32, dim wide), in the
                          reference's rank-major slicing (parallel.cpp:447-453)
     labels_local_dev   : the matching B/P labels (u32, global class ids)
   The layer all-gathers features and labels, selects the active classes, computes the
   distributed softmax cross-entropy, updates its active weight rows with momentum SGD at
   learning rate lr, and writes d loss / d features for its own B/P rows (through the row
   normalization, the tensor handed to mlp_backward at parallel.cpp:585-586) to
   grad_features_local_dev (may be NULL).  loss_dev (a double in device or pinned host memory, may be NULL) receives the
   mean loss, identical on all ranks.  Asynchronous: use xknn_layer_sync to collect errors. */
xknn_status_t xknn_step(xknn_layer_t* h, const float* features_local_dev,
                        const uint32_t* labels_local_dev, uint64_t batch_local, float lr,
                        double* loss_dev, float* grad_features_local_dev);

/* xknn_step with StepOptions::micro_batches = micro_batches (parallel.cpp:444, :505-591): one
   selection and one weight update per step, as the reference; the micro-batches (the balanced
   split of every rank's B/P rows, min(micro_batches, B/P) of them, 0 meaning 1) share one fused
   pass on the device -- the loss (sum of weight_c * loss_c = the batch mean) and the weight
   gradient (sum of scale * weight_c * G_c^T F_c) are the same sums -- and grad_features rows of
   micro-batch c are the tensor the reference hands to mlp_backward for them, whose softmax
   gradient carries 1/m_c: the caller scales its feature-extractor gradients by
   weight_c = m_c / B as the reference does (fe_acc.add_scaled, parallel.cpp:587). */
xknn_status_t xknn_step_micro(xknn_layer_t* h, const float* features_local_dev,
                              const uint32_t* labels_local_dev, uint64_t batch_local, float lr,
                              uint32_t micro_batches, double* loss_dev,
                              float* grad_features_local_dev);

/* Pipelined selection: starts the NEXT step's label all-gather and active-class selection on
   the layer's side stream now, so that it overlaps the step still in flight (its GEMMs and the
   HBM-bound row update) -- selection depends only on the labels and the graph.  The next
   xknn_step with the same batch size uses the result and skips its own selection; its
   labels_local must hold the labels given here.  ready_stream (may be NULL): the stream on which
   labels_local becomes valid (its current work is waited for); NULL = already valid.
   Collective when world > 1 (uses a communicator split from the layer's). */
xknn_status_t xknn_prepare(xknn_layer_t* h, const uint32_t* labels_local_dev,
                           uint64_t batch_local, void* ready_stream);

/* select_active_classes(const KnnGraph&, labels, cfg, n_total) (knn_softmax.cpp:100-115 +
   finish_selection :17-81) on one device: graph_dev is the uncompressed KnnGraph (num_classes x
   k u32, row-major, device), candidate ranks are positions in the full lists (equal to the shard
   overload only when P = 1, knn_softmax.hpp:40-43).  out_active_dev (capacity m_active) receives
   ActiveSet::class_indices (sorted), *count_host its size, *contains_all_host
   ActiveSet::contains_all_labels.  Errors as the reference: LabelOutOfRange, MTooSmall,
   InvalidArgument (M > N), ShapeMismatch (an id >= num_classes in the graph).  Synchronizes
   `stream`. */
xknn_status_t xknn_select_full_graph(const uint32_t* graph_dev, uint64_t num_classes, uint32_t k,
                                     const uint32_t* labels_dev, uint64_t batch,
                                     uint64_t m_active, uint64_t seed, uint32_t* out_active_dev,
                                     uint64_t* count_host, int* contains_all_host, void* stream);

/* knn_softmax_forward_backward(x_norm, w_norm, labels, active, scale) (knn_softmax.cpp:136-186),
   the single-shard free function, on device in fp32 with the reference's summation order
   (logits bit-identical; loss and gradients within 1e-5):
     x_norm_dev  batch x dim fp32 (already normalized), w_norm_dev num_classes x dim fp32,
     labels_dev  batch u32, active_dev m_act u32 (ActiveSet::class_indices, sorted, unique).
   Outputs: *loss_host (LossAndGrad::loss); grad_logits_dev (batch x m_act, may be NULL);
   grad_features_dev (batch x dim, d loss / d x_norm, times scale); grad_w_active_dev (m_act x
   dim: the active rows of LossAndGrad::grad_weights, which is zero elsewhere).  Errors:
   InvalidArgument (empty active set), LabelOutOfRange (active class >= num_classes),
   LabelNotActive (xknn_last_error_row = the batch row), ShapeMismatch.  Synchronizes. */
xknn_status_t xknn_knn_softmax_fwd_bwd(const float* x_norm_dev, uint64_t batch,
                                       const float* w_norm_dev, uint64_t num_classes,
                                       uint64_t dim, const uint32_t* labels_dev,
                                       const uint32_t* active_dev, uint64_t m_act, float scale,
                                       double* loss_host, float* grad_logits_dev,
                                       float* grad_features_dev, float* grad_w_active_dev,
                                       void* stream);

/* Replaces the padding draw's raw 64-bit word stream -- by default std::mt19937_64(rng_seed)
   re-seeded on every selection as the reference does (knn_softmax.cpp:43) -- with `count`
   caller-given words (count >= m_active; NULL restores the default).  The words feed
   std::uniform_int_distribution<size_t>'s Lemire draw (uniform_int_dist.h:257-274) exactly as
   engine output would, including its rejection loop (a zero word is always rejected unless the
   range is a power of two), so a crafted stream drives that rare path deterministically: a
   parity hook for tests, also usable to replay another engine's output.  Synchronizes. */
xknn_status_t xknn_layer_set_draw_stream(xknn_layer_t* h, const uint64_t* words, uint64_t count);

/* Synchronizes the layer stream, returns the first device-side error of the preceding
   asynchronous calls (label range, ZeroNormRow, MTooSmall, ...) and clears it. */
xknn_status_t xknn_layer_sync(xknn_layer_t* h);

/* Diagnostics of the last step (host values, synchronizes): |ActiveSet| (global), this
   shard's active row count. */
xknn_status_t xknn_layer_last_active(xknn_layer_t* h, uint64_t* active_global,
                                     uint64_t* active_local);

/* Copies the last step's logits (B x active_local, fp32) -- FP32_EXACT precision only; for
   parity tests of the logit GEMM (matmul(f_hat, w_sub, T) * scale, parallel.cpp:550-551). */
xknn_status_t xknn_layer_last_logits(xknn_layer_t* h, float* out_host, uint64_t capacity);

/* Phase profiler.  xknn_layer_profile(h, 1) resets and starts recording CUDA events on the
   layer stream at the phase boundaries of every step (asynchronous; no extra syncs in the step
   loop); xknn_layer_phase_ms returns the accumulated milliseconds per phase over the recorded
   steps (synchronizes; with the CUDA-graph step, the phases of the last step):
   0 feature/label all-gather, 1 selection, 2 operand normalize/gather, 3 logit GEMM (+ fused
   softmax epilogue in BF16), 4 softmax statistics + all-reduce + loss, 5 weight-gradient GEMM,
   6 feature-gradient GEMM, 7 feature-gradient reduce(-scatter), 8 normalize-backward +
   momentum-SGD row update (BF16: the wait for it), 9 feature normalize-backward, 11 the BF16
   row update itself (it runs on a side stream concurrently with phase 6). */
xknn_status_t xknn_layer_profile(xknn_layer_t* h, int enable);
xknn_status_t xknn_layer_phase_ms(xknn_layer_t* h, double* out_ms, int n, uint64_t* steps);

/* build_graph_bruteforce (knn_graph.cpp:124-145): the exact KNN graph of the normalized class
   weights w_norm_dev (num_classes x dim fp32, device), k neighbours per class, self first, then
   descending inner product (the reference's fp32 ascending-d sum), ties to the lower index.
   Bit-exact: an fp16 tensor-core pass keeps up to kprime candidates per row (0 = default,
   max(2k, k+32)) above a cut, the window that can reach the top k is re-scored exactly, and
   rows whose certificate fails are recomputed by an exact scan (*uncertified_rows counts them).  out_dev: num_classes x k u32.  Synchronizes `stream`. */
xknn_status_t xknn_graph_bruteforce(const float* w_norm_dev, uint64_t num_classes, uint64_t dim,
                                    uint32_t k, uint32_t kprime, uint32_t* out_dev, void* stream,
                                    uint64_t* uncertified_rows);

/* build_graph_ring (knn_graph.cpp:147-233) over the class blocks of `world` ranks, one process
   per GPU: w_norm_local_dev holds this rank's block of the ShardLayout(num_classes, world)
   (knn_graph.cpp:94-115) -- its normalized class weights, (end - begin) x dim fp32, device.
   The blocks travel around the ring over `comm` (ncclComm_t; rank -> rank+1, world-1 hops,
   RingBuildStats::transfer_steps) while every rank scores its own rows against them.  Writes
   rows [begin, end) of the graph (x k u32, global ids) to out_rows_dev; identical to
   build_graph_bruteforce on the concatenated blocks (bit-exact, see xknn_graph_bruteforce).
   k' >= k (else InvalidArgument, as the reference); it only sizes the candidate lists here.
   Collective: every rank calls it.  dim must be 512 when world > 1.  Synchronizes `stream`. */
xknn_status_t xknn_graph_ring(const float* w_norm_local_dev, uint64_t num_classes, uint64_t dim,
                             uint32_t k, uint32_t kprime, int rank, int world, void* comm,
                             void* stream, uint32_t* out_rows_dev, uint64_t* uncertified_rows,
                             uint64_t* transfer_steps);

/* The graph builds (xknn_graph_ring / _bruteforce / xknn_layer_rebuild_graph / classify) take
   their scratch from the device's default CUDA memory pool and leave it cached there for the
   next build (no driver map/unmap of GBs per rebuild).  This returns the cached blocks to the
   driver (cf. torch.cuda.empty_cache()).  Synchronizes the device.  No reference counterpart. */
xknn_status_t xknn_graph_release_cache(void);

/* compress_graph (knn_graph.cpp:235-266) + HybridSim::set_shard_graphs (parallel.cpp:381-388)
   from the row-distributed full graph: every rank passes its rows [begin, end) x k (global ids,
   device), entries are exchanged all-to-all by owning shard, and each layer installs its
   CompressedKnnGraph.  Collective.  Synchronizes. */
xknn_status_t xknn_layer_set_graph_rows(xknn_layer_t* h, const uint32_t* rows_dev, uint32_t k);

/* The periodic graph refresh of the paper on the live layer: l2_normalize_rows of every rank's
   weight shard (matrix.cpp:12-29, bit-exact; ZeroNormRow), xknn_graph_ring over the shards,
   then xknn_layer_set_graph_rows.  rows_out_dev (may be NULL) receives this rank's rows
   [begin, end) x k of the full graph (e.g. for xknn_graph_save_rows).  Collective.
   Synchronizes. */
xknn_status_t xknn_layer_rebuild_graph(xknn_layer_t* h, uint32_t k, uint32_t kprime,
                                       uint32_t* rows_out_dev, uint64_t* uncertified_rows);

/* save_graph (knn_graph.cpp:276-291) for a row-distributed KnnGraph: writes classes
   [begin, end) (rows: (end - begin) x k u32, host or device) as XKNN v1 records ("XKNN", u32
   version 1, u64 num_classes, then per class u32 k + k u32 ids, little-endian) at their byte
   offsets.  create != 0 creates/truncates the file and writes the header: one writer (rank 0)
   does that first, then every shard writes its own rows (records have a fixed size).  IoError
   on open/write failure. */
xknn_status_t xknn_graph_save_rows(const char* path, uint64_t num_classes, uint32_t k,
                                   uint64_t begin, uint64_t end, const uint32_t* rows,
                                   int on_device, int create);

/* load_graph (knn_graph.cpp:293-311) restricted to classes [begin, end): IoError for a file that
   cannot be opened, a bad magic, an unsupported version, truncation, or a record whose k differs
   from class 0's ("per-class k varies; not a full graph"); ShapeMismatch when the file's class
   count differs from num_classes (compress_graph's layout check).  *k_out receives the file's
   k; rows (capacity entries, host or device; NULL: header only) receives (end - begin) x k ids. */
xknn_status_t xknn_graph_load_rows(const char* path, uint64_t num_classes, uint64_t begin,
                                   uint64_t end, uint32_t* rows, uint64_t capacity, int on_device,
                                   uint32_t* k_out);

/* The installed CompressedKnnGraph of this shard (knn_graph.hpp:46-55): k_per_class and
   offsets [num_classes], flat [*flat_len] (flat_capacity >= *flat_len, else ShapeMismatch);
   NULL arrays are skipped.  Synchronizes. */
xknn_status_t xknn_layer_get_graph(xknn_layer_t* h, uint32_t* k_per_class, uint64_t* offsets,
                                   uint32_t* flat, uint64_t flat_capacity, uint64_t* flat_len,
                                   int on_device);

/* classify_retrieval (the paper's retrieval evaluation): the nearest class of
   each query among the L2-normalized class weights of all shards = the argmax of the fp32 cosine
   logits (matmul(q_hat, w_hat, T) order), ties to the lower class id.  Every rank scores its
   shard (fp16 tensor-core candidates, exact re-score of the certified window, exact scans
   otherwise) and the ranks' winners are merged over NCCL.  queries_dev: n_queries x dim fp32
   (normalized here, bit-exact with l2_normalize_rows; ZeroNormRow); out_class_dev: n_queries
   u32, out_score_dev (may be NULL): the winning cosine; identical on every rank.  Collective.
   Synchronizes. */
xknn_status_t xknn_layer_classify(xknn_layer_t* h, const float* queries_dev, uint64_t n_queries,
                                  uint32_t* out_class_dev, float* out_score_dev);

/* ---- DGC gradient sparsification (the paper's Table 6 path, beside the fc layer) ---------- */

/* topk_divide_conquer (sparsify.cpp:41-80): exact top-k of values_dev (len fp32) by |value|
   descending, ties to the lower index, in that selection order -- the reference's result is the
   same for every chunk count, so there is no chunk parameter.  KTooLarge (k > len),
   InvalidArgument (k == 0).  out_idx_dev / out_val_dev: k each.  Synchronizes `stream`. */
xknn_status_t xknn_topk(const float* values_dev, uint64_t len, uint64_t k, uint64_t* out_idx_dev,
                        float* out_val_dev, void* stream);

/* selected_count (sparsify.cpp:98-103): clamp(ceil((1 - ratio) * len), 1, len), 0 for len 0. */
uint64_t xknn_dgc_selected_count(double sparsity_ratio, uint64_t len);

/* CompressionState (sparsify.hpp:46-75) with the per-layer velocity and residual in HBM. */
typedef struct xknn_dgc xknn_dgc_t;
xknn_status_t xknn_dgc_create(double sparsity_ratio, float momentum, void* stream,
                              xknn_dgc_t** out);
xknn_status_t xknn_dgc_set_sparsity(xknn_dgc_t* h, double sparsity_ratio);
/* compress_step (sparsify.cpp:120-161): velocity = momentum*velocity + grad, residual +=
   velocity, emit the top selected_count(ratio, len) residual entries (indices strictly
   increasing, u64) and zero residual and velocity there.  *count = entries written.  Errors:
   InvalidArgument (empty gradient), ShapeMismatch (a layer's length changed).  Synchronizes. */
xknn_status_t xknn_dgc_compress(xknn_dgc_t* h, uint32_t layer_id, const float* grad_dev,
                                uint64_t len, uint64_t* out_idx_dev, float* out_val_dev,
                                uint64_t* count);
/* residual() / velocity() of a layer (zeros before its first compress_step), device copies. */
xknn_status_t xknn_dgc_state(xknn_dgc_t* h, uint32_t layer_id, float* residual_dev,
                             float* velocity_dev, uint64_t len);
xknn_status_t xknn_dgc_destroy(xknn_dgc_t* h);

/* Kernel launch counter (all kernels this library launched on this layer since creation). */
uint64_t xknn_layer_kernel_launches(const xknn_layer_t* h);

#ifdef __cplusplus
}
#endif
#endif /* XKNN_H_ */
