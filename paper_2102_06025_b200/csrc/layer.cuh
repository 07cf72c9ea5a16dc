// layer.cuh -- the per-GPU layer object behind the xknn C ABI.
//
// One Layer owns one contiguous class shard [begin, end) of the global fc weight matrix
// (ShardLayout, knn_graph.cpp:94-115) and everything HybridSim keeps per worker for that
// shard (parallel.cpp:204-215): weight rows, SgdMomentum velocity, the CompressedKnnGraph.
//
// HBM layout (N_w = end-begin rows, D = dim, B = max global batch, M_w = min(N_w, M)):
//   W, V            N_w x D fp32 (row-major, 2 KiB rows at D=512, 16-B aligned)
//   graph           k_per_class u32[N], offsets u64[N], flat u32[sum k]   (knn_graph.hpp:50-53)
//   sel_best/occ    u32[N_w] each, pool_bits/act_bits/lab_bits  u32[ceil(N_w/32)]
//   mt_cache        u64[M + 64]: the mt19937_64(rng_seed) stream -- the reference re-seeds
//                   per call (knn_softmax.cpp:43), so the stream is a constant of the layer
//   active          u32[M_w] sorted global ids of this shard's active classes
//   X (gathered)    B x D fp32, X_hat bf16 B x D, x_norm fp32[B]
//   W_sub           M_w x D bf16 (normalized active rows) + w_norm fp32[M_w]
//   P_tilde         B x M_w_pad bf16 (exp(s*logit - c), BF16 precision only)
//   dW              M_w x D fp32; dX partials fp32
#pragma once
#include <nccl.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace xknn {

xknn_status_t fail_msg(xknn_status_t s, const char* msg);  // sets xknn_last_error_message
xknn_status_t fail_row(xknn_status_t s, const char* msg, uint64_t row);  // + last_error_row

struct SelState {
  unsigned long long pool_local;   // |pool ∩ shard|
  unsigned long long pool_total;   // |pool|
  unsigned long long nd;           // distinct batch labels
  unsigned long long need;         // M - |pool| (padding branch)
  unsigned long long csize;        // N - |pool|
  unsigned long long cbase;        // first global complement position owned here
  unsigned long long compl_local;  // N_w - pool_local
  unsigned long long take;         // over-full: M - nd
  unsigned long long tie_quota;    // over-full: ties this shard keeps
  unsigned int branch;             // 0 padding, 1 exact fit, 2 over-full
  unsigned int first_rej;          // first Lemire rejection index (padding), kNone if none
  unsigned int r_star, o_star;     // over-full thresholds
  unsigned int pool_count;         // compacted local pool list length
  unsigned int active_count;       // compacted local active list length
  unsigned int labels_local;       // distinct labels owned here
  unsigned int labels_found;       // of those, present in the active set
  unsigned long long active_total; // |ActiveSet|
  double loss;                     // last loss
};

enum Branch : unsigned { kPad = 0, kExact = 1, kOverfull = 2 };

// The softmax statistics all-reduce over NVLink peer memory (peer.cu).
struct PeerAllreduce {
  int rank = 0, world = 0;
  uint64_t cap = 0;
  double* buf = nullptr;         // [2 slots][world][cap], written by every rank
  uint64_t* flags = nullptr;     // [world]: the epoch each rank last published here
  uint64_t* epoch = nullptr;     // this rank's all-reduce count
  double** peer_bufs = nullptr;  // device table: every rank's buf as mapped here
  uint64_t** peer_flags = nullptr;
  std::vector<void*> opened;
  bool ready = false;
  xknn_status_t setup(int rank, int world, uint64_t cap, ncclComm_t comm, cudaStream_t s);
  cudaError_t launch(double* data, uint64_t n, unsigned long long* err, cudaStream_t s) const;
  void release();
};

struct Layer {
  // ---- topology / config
  int rank = 0, world = 1, device = 0;
  uint64_t n = 0, d = 0, begin = 0, end = 0, nw = 0;
  xknn_config_t cfg{};
  ncclComm_t comm = nullptr;
  PeerAllreduce par_ar;               // P > 1: the B x 3 softmax statistics all-reduce
  bool par_ar_tried = false;
  ncclComm_t comm_ag = nullptr;       // split of comm: the feature all-gather, which overlaps
                                      // the selection's own collectives on comm
  cudaEvent_t ev_in = nullptr, ev_feat = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;        // overlaps the row update with the feature-gradient GEMM
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint64_t launches = 0;

  // ---- persistent state
  float* W = nullptr;
  float* V = nullptr;
  uint32_t* g_kpc = nullptr;
  uint64_t* g_off = nullptr;
  uint32_t* g_flat = nullptr;
  uint32_t* g_rank = nullptr;         // optional per-entry rank (merged multi-shard slices)
  bool select_only = false;           // XKNN_FLAG_SELECT_ONLY: no parameters, no step scratch
  uint64_t g_flat_len = 0;
  uint32_t g_kmax = 0;
  bool has_graph = false, has_weights = false;

  // ---- selection scratch
  uint32_t* sel_best = nullptr;
  uint32_t* sel_occ = nullptr;
  uint32_t* pool_bits = nullptr;
  uint32_t* act_bits = nullptr;
  uint32_t* lab_bits = nullptr;
  uint64_t nwords = 0;
  uint32_t* pool_list = nullptr;      // sorted local pool (global ids), cap nw
  uint32_t* pool_samp = nullptr;      // every 64th pool position p: (pool_list[p]-begin) - p
  uint32_t* pos_of = nullptr;         // local class -> position in `active` (valid if active)
  uint32_t* active = nullptr;         // sorted local active (global ids), cap mw_cap
  uint64_t mw_cap = 0;
  uint32_t* blk_counts = nullptr;     // compaction block counts / offsets
  uint64_t* mt_cache = nullptr;       // u64[m_active + 64]
  uint64_t mt_len = 0, mt_seed = 0;
  bool mt_injected = false;           // xknn_layer_set_draw_stream replaced the stream
  uint32_t* pick_key = nullptr;       // j_i        [M]
  uint32_t* pick_val = nullptr;       // next-in-group links [M]
  uint32_t* pick_head = nullptr;      // [N] group heads per complement position
  uint32_t* pred = nullptr;           // [M]
  uint32_t* lw = nullptr;             // [M]
  uint32_t* labels_all = nullptr;     // [B]
  int32_t* label_col = nullptr;       // [B] column of label in local active list, -1 if not local
  unsigned long long* pool_counts = nullptr;  // [2*world]: pool size, distinct labels
  unsigned long long* tie_counts = nullptr;   // [world]
  uint32_t* hist = nullptr;           // over-full histograms [hist_len]
  uint64_t hist_len = 0;
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  SelState* st = nullptr;             // device
  unsigned long long* err = nullptr;  // device error word

  // ---- step scratch
  uint64_t bmax = 0;
  float* X = nullptr;                 // gathered features B x D fp32
  float* Xhat = nullptr;              // B x D fp32 (exact)
  __nv_bfloat16* Xhat16 = nullptr;    // B x D bf16 (fast)
  __nv_bfloat16* Xs16 = nullptr;      // B x D bf16, rows scaled by s*r_i (fast)
  float* xnorm = nullptr;             // [B]
  float* Wsub = nullptr;              // M_w x D fp32 (exact)
  __nv_bfloat16* Wsub16 = nullptr;    // M_w x D bf16 (fast)
  float* wnorm = nullptr;             // [M_w]
  float* logits = nullptr;            // B x M_w fp32 (exact) ; G in place
  __nv_bfloat16* Pt = nullptr;        // B x ldp bf16 (fast)
  uint64_t ldp = 0;
  float* rowstat = nullptr;           // per-row partials
  double* rowred = nullptr;           // [3B] reduced (denom, label term, owner)
  float* rowmax = nullptr;            // [B]
  float* dW = nullptr;                // M_w x D fp32
  float* dX = nullptr;                // B x D fp32 (summed partial)
  float* dXpart = nullptr;            // split-K partials
  uint64_t dxpart_splits = 0;
  double* loss_dev = nullptr;         // [1]
  float* lr_dev = nullptr;            // [1] learning rate of the current step
  // CUDA graphs of run_core per batch size: [selection set][selection prepared]
  cudaGraphExec_t core_graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  uint64_t core_graph_b[2][2] = {{0, 0}, {0, 0}}, core_graph_launches[2][2] = {{0, 0}, {0, 0}};
  bool core_graph_prof[2][2] = {{false, false}, {false, false}};
  bool graph_mode = false;
  void drop_graphs();

  // ---- pipelined selection (xknn_prepare).  The selection of step t+1 needs only its labels and
  // the graph, so xknn_prepare runs it on the side stream while step t is still busy (its GEMMs
  // and the HBM-bound row update).  Its outputs that the rest of a step reads live in two sets;
  // the step after a prepare waits on ev_prep and skips its own selection.
  struct SelSet {
    SelState* st = nullptr;
    uint32_t* active = nullptr;
    int32_t* label_col = nullptr;
  };
  SelSet ss[2];
  int par = 0;                        // the set the next step (or prepare) uses
  int last_par = 0;                   // the set of the last step
  bool prepared = false;
  uint64_t prepared_b = 0;
  bool core_prepared = false;         // run_core: the selection was done by xknn_prepare
  cudaEvent_t ev_sel_done = nullptr;  // the last step's selection finished (scratch reusable)
  cudaEvent_t ev_prep = nullptr, ev_ready = nullptr;
  cudaGraphExec_t sel_graph[2] = {nullptr, nullptr};
  uint64_t sel_graph_b[2] = {0, 0}, sel_graph_launches[2] = {0, 0};
  void use_set(int p);
  xknn_status_t cancel_prepared();    // drop a pending xknn_prepare result (graph/seed changed)
  xknn_status_t run_prepare(const uint32_t* labels_local, uint64_t batch_local, cudaStream_t ready);
  xknn_status_t record_external(cudaEvent_t ev, cudaStream_t on);
  xknn_status_t wait_external(cudaEvent_t ev, cudaStream_t on);
  uint64_t last_b = 0;

  std::string last_msg;

  // ---- methods (layer.cu / select.cu / step.cu)
  xknn_status_t init(int rank, int world, uint64_t n, uint64_t d, const xknn_config_t* cfg,
                     void* comm, void* stream);
  void free_all();
  xknn_status_t ensure_mt_cache();
  xknn_status_t run_selection(uint64_t batch);    // labels_all already on device
  xknn_status_t run_core(uint64_t batch);
  xknn_status_t ensure_graph(uint64_t batch);
  xknn_status_t wait_features();
  xknn_status_t run_step(const float* feats_local, const uint32_t* labels_local,
                         uint64_t batch_local, float lr, double* loss_out, float* gfeat_local, uint32_t micros = 1);
  xknn_status_t nccl_ok(ncclResult_t r);
  xknn_status_t cuda_ok(cudaError_t e, const char* file = "", int line = 0,
                        const char* expr = "");

  // phase profiler: CUDA events recorded on the layer stream at phase boundaries (a ring of
  // per-step event sets, read back lazily so the timed loop stays asynchronous)
  static constexpr int kMarks = 13;  // 0..10 main stream, 11..12 the side-stream update
  static constexpr int kRing = 64;
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<double> prof_ms;
  uint64_t prof_steps = 0, prof_done = 0;
  void mark(int i, cudaStream_t on = nullptr);
  void prof_collect(bool all);

  // BF16 tensor-core path (fast.cu)
  void* fast = nullptr;
  xknn_status_t init_fast();
  void free_fast();
  xknn_status_t run_fast_core(uint64_t batch);
  xknn_status_t reset_fast_scratch();

  // FP32 (3xTF32) tensor-core path (fast32.cu)
  void* fast32 = nullptr;
  xknn_status_t init_fast32();
  void free_fast32();
  xknn_status_t run_fast32_core(uint64_t batch);
  xknn_status_t reset_fast32_scratch();
};

}  // namespace xknn

// the opaque handle of the C ABI
struct xknn_layer {
  xknn::Layer L;
};

// error helpers usable inside Layer methods
#define XK_CUDA(expr)                                                      \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) return cuda_ok(_e, __FILE__, __LINE__, #expr);  \
  } while (0)
#define XK_NCCL(expr)                                  \
  do {                                                 \
    ncclResult_t _r = (expr);                          \
    if (_r != ncclSuccess) return nccl_ok(_r);         \
  } while (0)
#define XK_TRY(expr)                                   \
  do {                                                 \
    xknn_status_t _s = (expr);                         \
    if (_s != XKNN_OK) return _s;                      \
  } while (0)
#define XK_TRY_H(expr)                                 \
  do {                                                 \
    xknn_status_t _s = (expr);                         \
    if (_s != XKNN_OK) return _s;                      \
  } while (0)
#define XK_CUDA_H(expr)                                                        \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) return h->L.cuda_ok(_e, __FILE__, __LINE__, #expr); \
  } while (0)
// XKNN_DEBUG_SYNC=1 (diagnostics): no CUDA graphs, and a device sync after every launch site, so
// a faulting kernel is reported at its own XK_LAUNCH line
inline bool debug_sync() {
  static const bool on = getenv("XKNN_DEBUG_SYNC") != nullptr;
  return on;
}
#define XK_LAUNCH()                                         \
  do {                                                      \
    ++launches;                                             \
    XK_CUDA(cudaGetLastError());                            \
    if (debug_sync()) XK_CUDA(cudaDeviceSynchronize());     \
  } while (0)
