// layer.cu -- the xknn C ABI (include/xknn.h) and the per-step orchestration.
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <random>
#include <string>

#include "kernels.cuh"

namespace xknn {

static thread_local std::string g_msg;
static thread_local uint64_t g_row = 0;

static xknn_status_t fail(xknn_status_t s, const std::string& msg) {
  g_msg = msg;
  return s;
}

xknn_status_t fail_msg(xknn_status_t s, const char* msg) { return fail(s, msg); }
xknn_status_t fail_row(xknn_status_t s, const char* msg, uint64_t row) {
  g_row = row;
  return fail(s, msg);
}

xknn_status_t Layer::cuda_ok(cudaError_t e, const char* file, int line, const char* expr) {
  if (e == cudaSuccess) return XKNN_OK;
  (void)cudaGetLastError();  // clear non-sticky errors so the caller's runtime stays clean
  const std::string where = std::string(" at ") + file + ":" + std::to_string(line) + " " + expr;
  if (e == cudaErrorMemoryAllocation)
    return fail(XKNN_ERR_OUT_OF_MEMORY, std::string("cuda: ") + cudaGetErrorString(e) + where);
  return fail(XKNN_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e) + where);
}

xknn_status_t Layer::nccl_ok(ncclResult_t r) {
  if (r == ncclSuccess) return XKNN_OK;
  return fail(XKNN_ERR_NCCL, std::string("nccl: ") + ncclGetErrorString(r));
}


xknn_status_t Layer::init(int rank_, int world_, uint64_t n_, uint64_t d_,
                          const xknn_config_t* cfg_, void* comm_, void* stream_) {
  rank = rank_;
  world = world_;
  n = n_;
  d = d_;
  cfg = *cfg_;
  comm = static_cast<ncclComm_t>(comm_);
  stream = static_cast<cudaStream_t>(stream_);
  XK_CUDA(cudaGetDevice(&device));
  const uint64_t base = n / world, rem = n % world;  // ShardLayout::class_range
  if ((uint64_t)rank < rem) {
    begin = rank * (base + 1);
    end = begin + base + 1;
  } else {
    begin = rem * (base + 1) + (rank - rem) * base;
    end = begin + base;
  }
  nw = end - begin;
  nwords = (nw + 31) / 32;
  bmax = cfg.max_batch;
  mw_cap = std::min<uint64_t>(nw, cfg.m_active);
  if (cfg.active_capacity) mw_cap = std::min<uint64_t>(mw_cap, cfg.active_capacity);

  select_only = (cfg.flags & XKNN_FLAG_SELECT_ONLY) != 0;
  if (!select_only) {
    XK_CUDA(dalloc(&W, nw * d));
    XK_CUDA(dalloc(&V, nw * d));
    XK_CUDA(cudaMemsetAsync(V, 0, nw * d * sizeof(float), stream));
  }
  XK_CUDA(dalloc(&sel_best, nw));
  XK_CUDA(dalloc(&sel_occ, nw));
  XK_CUDA(cudaMemsetAsync(sel_best, 0xff, nw * sizeof(uint32_t), stream));
  XK_CUDA(cudaMemsetAsync(sel_occ, 0, nw * sizeof(uint32_t), stream));
  XK_CUDA(dalloc(&pool_bits, 3 * nwords));  // pool | act | labels, cleared by one memset
  act_bits = pool_bits + nwords;
  lab_bits = pool_bits + 2 * nwords;
  XK_CUDA(dalloc(&pos_of, nw));
  XK_CUDA(dalloc(&pool_list, nw));
  XK_CUDA(dalloc(&pool_samp, nw / 64 + 2));
  for (int q = 0; q < 2; ++q) {
    XK_CUDA(dalloc(&ss[q].active, mw_cap + 32));
    XK_CUDA(dalloc(&ss[q].st, 1));
    XK_CUDA(cudaMemsetAsync(ss[q].st, 0, sizeof(SelState), stream));
    XK_CUDA(dalloc(&ss[q].label_col, bmax));
  }
  use_set(0);
  const uint64_t nblocks = (nwords + 255) / 256;
  XK_CUDA(dalloc(&blk_counts, 2 * (nblocks + 2)));
  XK_CUDA(cudaMemsetAsync(blk_counts, 0, 2 * (nblocks + 2) * sizeof(uint32_t), stream));
  const uint64_t m = cfg.m_active;
  XK_CUDA(dalloc(&pick_key, m));
  XK_CUDA(dalloc(&pick_val, m));
  XK_CUDA(dalloc(&pick_head, n));  // per complement position, kNone between steps
  XK_CUDA(cudaMemsetAsync(pick_head, 0xff, n * sizeof(uint32_t), stream));
  XK_CUDA(dalloc(&pred, m));
  XK_CUDA(dalloc(&lw, m));
  XK_CUDA(dalloc(&labels_all, bmax));
  XK_CUDA(dalloc(&pool_counts, 2 * world));
  XK_CUDA(dalloc(&tie_counts, world));
  XK_CUDA(dalloc(&err, 1));
  XK_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned long long), stream));
  XK_CUDA(dalloc(&loss_dev, 1));
  XK_CUDA(dalloc(&lr_dev, 1));
  XK_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  XK_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  XK_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  XK_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
  XK_CUDA(cudaEventCreateWithFlags(&ev_feat, cudaEventDisableTiming));
  XK_CUDA(cudaEventCreateWithFlags(&ev_sel_done, cudaEventDisableTiming));
  XK_CUDA(cudaEventCreateWithFlags(&ev_prep, cudaEventDisableTiming));
  XK_CUDA(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));

  // cub temp: max over the sorts/scans/selects we run
  size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b3, blk_counts, blk_counts, (int)(nblocks + 1), stream);
  cub_tmp_bytes = std::max(std::max(b1, b2), std::max(b3, b4)) + 256;
  XK_CUDA(cudaMalloc(&cub_tmp, cub_tmp_bytes));

  // step scratch
  if (select_only) {
    XK_CUDA(cudaStreamSynchronize(stream));
    return XKNN_OK;
  }
  XK_CUDA(dalloc(&X, bmax * d));
  XK_CUDA(dalloc(&xnorm, bmax));
  XK_CUDA(dalloc(&wnorm, mw_cap));
  XK_CUDA(dalloc(&rowmax, bmax));
  XK_CUDA(dalloc(&rowred, 3 * bmax));
  XK_CUDA(dalloc(&dX, bmax * d));
  if (cfg.precision == XKNN_PREC_FP32_EXACT) {
    XK_CUDA(dalloc(&dW, mw_cap * d));
    XK_CUDA(dalloc(&Xhat, bmax * d));
    XK_CUDA(dalloc(&Wsub, mw_cap * d));
    XK_CUDA(dalloc(&logits, bmax * mw_cap * 2));  // logits, then G
    XK_CUDA(dalloc(&dXpart, bmax * d));
  } else if (cfg.precision == XKNN_PREC_FP32) {
    XK_TRY(init_fast32());
  } else {
    XK_TRY(init_fast());
  }
  XK_CUDA(cudaStreamSynchronize(stream));
  return XKNN_OK;
}

void Layer::free_all() {
  void* ptrs[] = {W, V, g_kpc, g_off, g_flat, g_rank, sel_best, sel_occ, pool_bits, pos_of,
                  pool_list, pool_samp, blk_counts, mt_cache, pick_key, pick_val, pick_head,
                  pred, lw, labels_all, pool_counts, tie_counts, hist, cub_tmp, err, X, Xhat, Xhat16,
                  Xs16, xnorm, Wsub, Wsub16, wnorm, logits, Pt, rowstat, rowred, rowmax, dW, dX,
                  dXpart, loss_dev};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto e : prof_ev) cudaEventDestroy(e);
  prof_ev.clear();
  drop_graphs();
  for (auto& q : ss) {
    void* pp[] = {q.st, q.active, q.label_col};
    for (void* p : pp)
      if (p) cudaFree(p);
    q = SelSet{};
  }
  for (cudaEvent_t e : {ev_sel_done, ev_prep, ev_ready})
    if (e) cudaEventDestroy(e);
  if (lr_dev) cudaFree(lr_dev);
  if (side) cudaStreamDestroy(side);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_in) cudaEventDestroy(ev_in);
  if (ev_feat) cudaEventDestroy(ev_feat);
  if (comm_ag) ncclCommDestroy(comm_ag);
  par_ar.release();
  free_fast();
  free_fast32();
}

// The padding draw's raw stream: std::mt19937_64(rng_seed), re-seeded by the reference on every
// select_active_classes call (knn_softmax.cpp:43) -- generated here with the same libstdc++
// engine, once per (seed, M).
xknn_status_t Layer::ensure_mt_cache() {
  if (mt_injected) return XKNN_OK;  // xknn_layer_set_draw_stream
  const uint64_t want = cfg.m_active + 64;
  if (mt_cache && mt_len == want && mt_seed == cfg.rng_seed) return XKNN_OK;
  if (mt_cache) cudaFree(mt_cache);
  mt_cache = nullptr;
  std::vector<uint64_t> h(want);
  std::mt19937_64 g(cfg.rng_seed);
  for (auto& v : h) v = g();
  XK_CUDA(dalloc(&mt_cache, want));
  XK_CUDA(cudaMemcpyAsync(mt_cache, h.data(), want * sizeof(uint64_t), cudaMemcpyHostToDevice,
                          stream));
  XK_CUDA(cudaStreamSynchronize(stream));
  mt_len = want;
  mt_seed = cfg.rng_seed;
  return XKNN_OK;
}

__global__ void k_set_f32(float* p, float v) {
  griddep_wait();
  griddep_launch(); *p = v; }

// P = 1 step inputs in one kernel: the caller's features (and labels, unless a prepared
// selection already holds them) into the layer's buffers, and the learning rate into device
// memory -- instead of two copy-engine nodes and a kernel between the step graphs
__global__ void k_stage_inputs(float4* __restrict__ X, const float4* __restrict__ xs,
                               uint64_t n4, uint32_t* __restrict__ lab,
                               const uint32_t* __restrict__ ls, uint64_t nl, float* lr_dev,
                               float lr) {
  griddep_wait();
  griddep_launch();
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = t0; i < n4; i += stride) X[i] = xs[i];
  if (lab)
    for (uint64_t i = t0; i < nl; i += stride) lab[i] = ls[i];
  if (t0 == 0) *lr_dev = lr;
}

// the step's loss to the caller's double (device or pinned host memory, through UVA): a kernel
// in the stream's launch chain instead of a copy-engine node between two step graphs
__global__ void k_copy_loss(double* dst, const double* src) {
  griddep_wait();
  griddep_launch();
  *dst = *src;
}

void Layer::mark(int i, cudaStream_t on) {
  if (!prof_on) return;
  cudaStream_t stream = on ? on : this->stream;
  const uint64_t slot = graph_mode ? 0 : (prof_steps % kRing);
  // inside a stream capture an External record becomes an event-record node fired on replay
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(prof_ev[slot * kMarks + i], stream, cudaEventRecordExternal);
  else
    cudaEventRecord(prof_ev[slot * kMarks + i], stream);
}

// Accumulates the phase durations of finished steps (all = wait for every recorded step).  In
// graph mode the in-graph marks are fixed event nodes: the phases of the last replay count.
void Layer::prof_collect(bool all) {
  if (graph_mode) {
    if (!all || prof_steps == 0) return;
    cudaEvent_t* e = &prof_ev[0];
    cudaEventSynchronize(e[10]);
    prof_ms.assign(kMarks, 0.0);
    for (int i = 0; i + 1 < kMarks; ++i) {
      float ms = 0.f;
      if (i != 10 && cudaEventElapsedTime(&ms, e[i], e[i + 1]) == cudaSuccess) prof_ms[i] = ms;
    }
    prof_done = 1;
    (void)cudaGetLastError();  // never leave a stale error for the caller's runtime
    return;
  }
  while (prof_done < prof_steps) {
    if (!all && prof_steps - prof_done < kRing) break;
    cudaEvent_t* e = &prof_ev[(prof_done % kRing) * kMarks];
    cudaEventSynchronize(e[10]);
    for (int i = 0; i + 1 < kMarks; ++i) {
      float ms = 0.f;
      if (i != 10 && cudaEventElapsedTime(&ms, e[i], e[i + 1]) == cudaSuccess) prof_ms[i] += ms;
    }
    ++prof_done;
  }
  (void)cudaGetLastError();
}

// Everything between the input all-gather and the caller-facing outputs: selection, operands,
// the three GEMMs with the distributed softmax, the feature-gradient reduce(-scatter) and the
// sparse update.  Touches only layer-owned buffers, so it is captured once per batch size into
// a CUDA graph and replayed (the learning rate is read from device memory).
xknn_status_t Layer::run_core(uint64_t B) {
  const uint32_t D = (uint32_t)d;
  const uint64_t bl = B / world;
  // (1) Algorithm 1 selection -> this shard's sorted active rows (or xknn_prepare's result)
  if (core_prepared)
    XK_TRY(wait_external(ev_prep, stream));
  else
    XK_TRY(run_selection(B));
  XK_TRY(record_external(ev_sel_done, stream));  // the next prepare may reuse the scratch
  mark(2);
  unsigned int* cnt = &st->active_count;
  // feature rows normalized; active weight rows gathered + normalized (only M_w rows, never the
  // whole shard as parallel.cpp:490-492 does -- row-wise identical)
  // (the BF16 core waits for the feature all-gather only after its weight-row gather)
  if (world > 1 && cfg.precision == XKNN_PREC_FP32_EXACT) XK_TRY(wait_features());
  if (cfg.precision == XKNN_PREC_FP32_EXACT) {
    XK_CUDA(launch_normalize_rows(X, B, D, nullptr, nullptr, 0, Xhat, nullptr, xnorm, err, stream));
    ++launches;
    XK_CUDA(launch_normalize_rows(W, mw_cap, D, active, cnt, begin, Wsub, nullptr, wnorm, err,
                                  stream));
    ++launches;
    float* L = logits;
    float* G = logits + bmax * mw_cap;
    mark(3);
    // (3) logits
    XK_CUDA(launch_logits_exact(Xhat, Wsub, B, cnt, mw_cap, D, cfg.scale, L, stream));
    ++launches;
    mark(4);
    // (4) distributed softmax-CE: global row max, then [exp-sum, label term, owner] sums
    XK_CUDA(launch_rowmax(L, B, cnt, rowmax, stream));
    ++launches;
    if (world > 1) XK_NCCL(ncclAllReduce(rowmax, rowmax, B, ncclFloat, ncclMax, comm, stream));
    XK_CUDA(launch_rowsum(L, B, cnt, rowmax, label_col, rowred, stream));
    ++launches;
    if (world > 1) XK_NCCL(ncclAllReduce(rowred, rowred, 3 * B, ncclDouble, ncclSum, comm, stream));
    XK_CUDA(launch_loss(rowred, B, loss_dev, st, err, stream));
    ++launches;
    XK_CUDA(cudaMemcpyAsync(G, L, B * mw_cap * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    XK_CUDA(launch_softmax_grad(G, B, cnt, mw_cap, rowmax, rowred, label_col, stream));
    ++launches;
    mark(5);
    // (5) weight side and feature side
    XK_CUDA(launch_dw_exact(G, Xhat, B, cnt, mw_cap, D, cfg.scale * 1.0f, dW, stream));
    ++launches;
    mark(6);
    XK_CUDA(launch_dx_exact(G, Wsub, B, cnt, D, cfg.scale, dXpart, stream));
    ++launches;
    mark(7);
    if (world > 1)
      XK_NCCL(ncclReduceScatter(dXpart, dX, bl * d, ncclFloat, ncclSum, comm, stream));
    else
      XK_CUDA(cudaMemcpyAsync(dX, dXpart, B * d * sizeof(float), cudaMemcpyDeviceToDevice, stream));
  } else if (cfg.precision == XKNN_PREC_FP32) {
    XK_TRY(run_fast32_core(B));
  } else {
    XK_TRY(run_fast_core(B));
  }
  // (8) normalize-backward + momentum SGD on the active rows only (parallel.cpp:649-667);
  //     the BF16 path runs it at the end of run_fast_core (from its bf16 dW, or fused into
  //     the GEMM-dW epilogue)
  if (cfg.precision == XKNN_PREC_FP32_EXACT) {
    mark(8);
    XK_CUDA(launch_update_rows(W, V, dW, active, cnt, mw_cap, begin, D, wnorm, lr_dev,
                               cfg.momentum, cfg.weight_decay, err, stream));
    ++launches;
  }
  mark(9);
  return XKNN_OK;
}

// the core waits for the feature all-gather of run_step (an external event-wait node when the
// core is being captured into the step's CUDA graph)
xknn_status_t Layer::wait_features() {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  XK_CUDA(cudaStreamIsCapturing(stream, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    XK_CUDA(cudaStreamWaitEvent(stream, ev_feat, cudaEventWaitExternal));
  else
    XK_CUDA(cudaStreamWaitEvent(stream, ev_feat, 0));
  return XKNN_OK;
}

xknn_status_t Layer::ensure_graph(uint64_t B) {
  const int p = par, q = core_prepared ? 1 : 0;
  cudaGraphExec_t& gx = core_graph[p][q];
  if (gx && core_graph_b[p][q] == B && core_graph_prof[p][q] == prof_on) return XKNN_OK;
  if (gx) cudaGraphExecDestroy(gx);
  gx = nullptr;
  XK_TRY(ensure_mt_cache());
  const uint64_t l0 = launches;
  cudaGraph_t g = nullptr;
  XK_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  xknn_status_t s = run_core(B);
  cudaError_t e = cudaStreamEndCapture(stream, &g);
  if (s != XKNN_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  XK_CUDA(e);
  e = cudaGraphInstantiate(&gx, g, 0);
  cudaGraphDestroy(g);
  XK_CUDA(e);
  core_graph_b[p][q] = B;
  core_graph_prof[p][q] = prof_on;
  core_graph_launches[p][q] = launches - l0;
  launches = l0;
  return XKNN_OK;
}

void Layer::drop_graphs() {
  for (auto& row : core_graph)
    for (auto& g : row) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
  for (auto& g : sel_graph) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

xknn_status_t Layer::cancel_prepared() {
  if (!prepared) return XKNN_OK;
  XK_CUDA(cudaStreamWaitEvent(stream, ev_prep, 0));  // its side-stream work stays ordered
  prepared = false;
  return XKNN_OK;
}

void Layer::use_set(int p) {
  st = ss[p].st;
  active = ss[p].active;
  label_col = ss[p].label_col;
}

// an event record / wait that becomes an external event node when `on` is being captured
xknn_status_t Layer::record_external(cudaEvent_t ev, cudaStream_t on) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  XK_CUDA(cudaStreamIsCapturing(on, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    XK_CUDA(cudaEventRecordWithFlags(ev, on, cudaEventRecordExternal));
  else
    XK_CUDA(cudaEventRecord(ev, on));
  return XKNN_OK;
}
xknn_status_t Layer::wait_external(cudaEvent_t ev, cudaStream_t on) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  XK_CUDA(cudaStreamIsCapturing(on, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    XK_CUDA(cudaStreamWaitEvent(on, ev, cudaEventWaitExternal));
  else
    XK_CUDA(cudaStreamWaitEvent(on, ev, 0));
  return XKNN_OK;
}

// xknn_prepare: the next step's label all-gather and selection on the side stream, into the
// selection set that step will use, after the last step's selection released the scratch.
xknn_status_t Layer::run_prepare(const uint32_t* labels_local, uint64_t bl, cudaStream_t ready) {
  const uint64_t B = bl * world;
  if (prepared) XK_CUDA(cudaStreamWaitEvent(stream, ev_prep, 0));  // superseded: keep order
  if (world > 1 && !comm_ag) XK_NCCL(ncclCommSplit(comm, 0, rank, &comm_ag, nullptr));
  XK_TRY(ensure_mt_cache());
  use_set(par);
  if (ready) {
    XK_CUDA(cudaEventRecord(ev_ready, ready));
    XK_CUDA(cudaStreamWaitEvent(side, ev_ready, 0));
  }
  XK_CUDA(cudaStreamWaitEvent(side, ev_sel_done, 0));
  if (world > 1)
    XK_NCCL(ncclAllGather(labels_local, labels_all, bl, ncclUint32, comm_ag, side));
  else
    XK_CUDA(cudaMemcpyAsync(labels_all, labels_local, B * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, side));
  // the selection itself, on the side stream and the split communicator (the layer stream and
  // its communicator may be busy with the previous step), captured once per set and batch size
  cudaStream_t s0 = stream;
  ncclComm_t c0 = comm;
  stream = side;
  comm = world > 1 ? comm_ag : comm;
  xknn_status_t st_ = XKNN_OK;
  const bool use_graph = graph_mode || (!(cfg.flags & XKNN_FLAG_NO_GRAPH) && s0 != nullptr);
  if (use_graph) {
    cudaGraphExec_t& gx = sel_graph[par];
    if (!gx || sel_graph_b[par] != B) {
      if (gx) cudaGraphExecDestroy(gx);
      gx = nullptr;
      const uint64_t l0 = launches;
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamBeginCapture(side, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        st_ = run_selection(B);
        e = cudaStreamEndCapture(side, &g);
        if (st_ == XKNN_OK && e == cudaSuccess) e = cudaGraphInstantiate(&gx, g, 0);
        if (g) cudaGraphDestroy(g);
      }
      if (st_ == XKNN_OK && e != cudaSuccess) st_ = cuda_ok(e, __FILE__, __LINE__, "prepare");
      sel_graph_b[par] = B;
      sel_graph_launches[par] = launches - l0;
      launches = l0;
    }
    if (st_ == XKNN_OK) {
      cudaError_t e = cudaGraphLaunch(gx, side);
      if (e != cudaSuccess) st_ = cuda_ok(e, __FILE__, __LINE__, "prepare launch");
      launches += sel_graph_launches[par];
    }
  } else {
    st_ = run_selection(B);
  }
  stream = s0;
  comm = c0;
  XK_TRY(st_);
  XK_CUDA(cudaEventRecord(ev_prep, side));
  prepared = true;
  prepared_b = B;
  return XKNN_OK;
}

xknn_status_t Layer::run_step(const float* feats_local, const uint32_t* labels_local,
                              uint64_t bl, float lr, double* loss_out, float* gfeat_local,
                              uint32_t micros) {
  const uint64_t B = bl * world;
  const uint32_t D = (uint32_t)d;
  last_b = B;
  graph_mode = !(cfg.flags & XKNN_FLAG_NO_GRAPH) && stream != nullptr && !debug_sync();
  if (prof_on) prof_collect(false);
  mark(0);
  // this step's selection set; a prepared selection (xknn_prepare) for this batch size is used
  // instead of selecting again (its labels are the caller's promise)
  const int p = par;
  use_set(p);
  core_prepared = prepared && prepared_b == B;
  if (prepared && !core_prepared) XK_CUDA(cudaStreamWaitEvent(stream, ev_prep, 0));
  prepared = false;
  // (2) feature and label all-gather, rank-major (parallel.cpp:447-453, :544).  The labels go
  //     first on the layer stream (selection needs them); the features travel on the side
  //     stream over a split communicator while the selection runs, and the core waits for them
  //     right before the first kernel that reads X.
  if (world > 1) {
    if (!comm_ag) XK_NCCL(ncclCommSplit(comm, 0, rank, &comm_ag, nullptr));  // collective
    if (!par_ar.ready && !par_ar_tried && cfg.precision != XKNN_PREC_FP32_EXACT &&
        !getenv("XKNN_NCCL_ALLREDUCE")) {
      // collective; without CUDA IPC between the ranks the statistics go through NCCL
      par_ar_tried = true;
      if (par_ar.setup(rank, world, 3 * bmax, comm, stream) != XKNN_OK) {
        par_ar.release();
        (void)cudaGetLastError();
      }
    }
    if (!core_prepared)
      XK_NCCL(ncclAllGather(labels_local, labels_all, bl, ncclUint32, comm, stream));
    XK_CUDA(cudaEventRecord(ev_in, stream));
    XK_CUDA(cudaStreamWaitEvent(side, ev_in, 0));
    XK_NCCL(ncclAllGather(feats_local, X, bl * d, ncclFloat, comm_ag, side));
    XK_CUDA(cudaEventRecord(ev_feat, side));
  }
  // the learning rate travels through device memory so the captured core stays valid
  if (world == 1 && (reinterpret_cast<uintptr_t>(feats_local) & 15) == 0 && d % 4 == 0) {
    const uint64_t n4 = B * d / 4;
    launch_pdl(k_stage_inputs, grid_for(n4, 256, 148u * 8u), 256, 0, stream,
               reinterpret_cast<float4*>(X), reinterpret_cast<const float4*>(feats_local), n4,
               core_prepared ? (uint32_t*)nullptr : labels_all, labels_local, (uint64_t)B, lr_dev,
               lr);
    XK_LAUNCH();
  } else {
    if (world == 1) {
      XK_CUDA(cudaMemcpyAsync(X, feats_local, B * d * sizeof(float), cudaMemcpyDeviceToDevice,
                              stream));
      if (!core_prepared)
        XK_CUDA(cudaMemcpyAsync(labels_all, labels_local, B * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, stream));
    }
    launch_pdl(k_set_f32, 1, 1, 0, stream, lr_dev, lr);
    XK_LAUNCH();
  }
  mark(1);
  if (graph_mode) {
    XK_TRY(ensure_graph(B));
    const int q = core_prepared ? 1 : 0;
    XK_CUDA(cudaGraphLaunch(core_graph[p][q], stream));
    launches += core_graph_launches[p][q];
  } else {
    XK_TRY(run_core(B));
  }
  last_par = p;
  par = 1 - p;
  // (6) feature normalize-backward on this rank's rows (parallel.cpp:574-585)
  if (gfeat_local) {
    XK_CUDA(launch_feature_backward(X + (uint64_t)rank * bl * d, xnorm + (uint64_t)rank * bl, dX,
                                    bl, D, gfeat_local, stream, micros));
    ++launches;
  }
  mark(10);
  if (prof_on) ++prof_steps;
  if (loss_out) {
    cudaPointerAttributes pa{};
    double* dptr = nullptr;
    if (cudaPointerGetAttributes(&pa, loss_out) == cudaSuccess && pa.type != cudaMemoryTypeUnregistered)
      dptr = static_cast<double*>(pa.devicePointer);  // pinned host memory: its mapped address
    if (dptr) {
      launch_pdl(k_copy_loss, 1, 1, 0, stream, dptr, (const double*)loss_dev);
      XK_LAUNCH();
    } else {  // pageable host memory: the driver stages it
      XK_CUDA(cudaMemcpyAsync(loss_out, loss_dev, sizeof(double), cudaMemcpyDefault, stream));
    }
  }
  return XKNN_OK;
}

}  // namespace xknn

using xknn::Layer;
using xknn::fail;


// The tensor-core paths replace the row max by the fixed stabilizer c = s (fast.cu): every
// exp(s*cos - s) lies in [e^-2s, 1], which fp32 (and ex2.approx.ftz) represents for s <= 40.
// The reference works at any scale; FP32_EXACT (true row max) accepts any finite scale.
static xknn_status_t check_scale(const xknn_config_t* cfg) {
  if (!std::isfinite(cfg->scale)) return fail(XKNN_ERR_CONFIG, "scale must be finite");
  if (cfg->precision != XKNN_PREC_FP32_EXACT && !(cfg->scale > 0.f && cfg->scale <= 40.f))
    return fail(XKNN_ERR_CONFIG,
                "tensor-core precisions need 0 < scale <= 40 (fixed softmax stabilizer); use "
                "XKNN_PREC_FP32_EXACT for other scales");
  return XKNN_OK;
}

#define GUARD_H(h) \
  if (!(h)) return fail(XKNN_ERR_INVALID_ARGUMENT, "null layer handle")

extern "C" {

const char* xknn_status_string(xknn_status_t s) {
  switch (s) {
    case XKNN_OK: return "ok";
    case XKNN_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case XKNN_ERR_ZERO_NORM_ROW: return "ZeroNormRow";
    case XKNN_ERR_LABEL_OUT_OF_RANGE: return "LabelOutOfRange";
    case XKNN_ERR_K_TOO_LARGE: return "KTooLarge";
    case XKNN_ERR_EMPTY_SHARD: return "EmptyShard";
    case XKNN_ERR_M_TOO_SMALL: return "MTooSmall";
    case XKNN_ERR_LABEL_NOT_ACTIVE: return "LabelNotActive";
    case XKNN_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case XKNN_ERR_IO: return "IoError";
    case XKNN_ERR_CONFIG: return "ConfigError";
    case XKNN_ERR_CUDA: return "CudaError";
    case XKNN_ERR_NCCL: return "NcclError";
    case XKNN_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    case XKNN_ERR_UNSUPPORTED: return "Unsupported";
  }
  return "unknown";
}

const char* xknn_last_error_message(void) { return xknn::g_msg.c_str(); }
uint64_t xknn_last_error_row(void) { return xknn::g_row; }

xknn_status_t xknn_shard_range(uint64_t n, uint64_t p, uint64_t s, uint64_t* b, uint64_t* e) {
  if (p == 0 || s >= p) return fail(XKNN_ERR_INVALID_ARGUMENT, "ShardLayout: shard index out of range");
  const uint64_t base = n / p, rem = n % p;
  if (s < rem) {
    *b = s * (base + 1);
    *e = *b + base + 1;
  } else {
    *b = rem * (base + 1) + (s - rem) * base;
    *e = *b + base;
  }
  return XKNN_OK;
}

xknn_status_t xknn_nccl_unique_id(uint8_t out_id[128]) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(XKNN_ERR_NCCL, ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out_id, &id, 128);
  return XKNN_OK;
}

xknn_status_t xknn_nccl_comm_init(const uint8_t id[128], int world, int rank, void** comm) {
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, world, uid, rank);
  if (r != ncclSuccess) return fail(XKNN_ERR_NCCL, ncclGetErrorString(r));
  *comm = c;
  return XKNN_OK;
}

xknn_status_t xknn_nccl_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
  return XKNN_OK;
}

xknn_status_t xknn_layer_create(int rank, int world, uint64_t n, uint64_t d,
                                const xknn_config_t* cfg, void* comm, void* stream,
                                xknn_layer_t** out) {
  if (!cfg || !out) return fail(XKNN_ERR_INVALID_ARGUMENT, "null argument");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(XKNN_ERR_INVALID_ARGUMENT, "HybridSim: need >= 1 worker and 0 <= rank < world");
  if (world > 1 && !comm) return fail(XKNN_ERR_INVALID_ARGUMENT, "world > 1 needs an NCCL comm");
  if ((uint64_t)world > n) return fail(XKNN_ERR_EMPTY_SHARD, "more shards than classes");
  if (d == 0 || d % 128 != 0 || d > 1024)
    return fail(XKNN_ERR_SHAPE_MISMATCH, "dim must be a multiple of 128 and <= 1024");
  if (n >= 0xffffffffull) return fail(XKNN_ERR_INVALID_ARGUMENT, "class ids are u32");
  if (cfg->max_batch == 0 || cfg->max_batch % world)
    return fail(XKNN_ERR_INVALID_ARGUMENT, "max_batch must be a positive multiple of world");
  if (cfg->m_active > n) return fail(XKNN_ERR_INVALID_ARGUMENT, "M exceeds the class count");
  if (cfg->precision != XKNN_PREC_BF16 && cfg->precision != XKNN_PREC_FP32_EXACT &&
      cfg->precision != XKNN_PREC_FP32)
    return fail(XKNN_ERR_CONFIG, "unknown precision");
  if (xknn_status_t s = check_scale(cfg); s != XKNN_OK) return s;
  auto* h = new (std::nothrow) xknn_layer;
  if (!h) return fail(XKNN_ERR_OUT_OF_MEMORY, "host alloc");
  xknn_status_t s = h->L.init(rank, world, n, d, cfg, comm, stream);
  if (s != XKNN_OK) {
    h->L.free_all();
    delete h;
    return s;
  }
  *out = h;
  return XKNN_OK;
}

xknn_status_t xknn_layer_destroy(xknn_layer_t* h) {
  if (!h) return XKNN_OK;
  cudaStreamSynchronize(h->L.stream);
  h->L.free_all();
  delete h;
  return XKNN_OK;
}

xknn_status_t xknn_layer_shard(const xknn_layer_t* h, uint64_t* b, uint64_t* e) {
  GUARD_H(h);
  *b = h->L.begin;
  *e = h->L.end;
  return XKNN_OK;
}

xknn_status_t xknn_layer_set_config(xknn_layer_t* h, const xknn_config_t* cfg) {
  GUARD_H(h);
  Layer& L = h->L;
  if (cfg->m_active != L.cfg.m_active || cfg->max_batch != L.cfg.max_batch ||
      cfg->precision != L.cfg.precision || cfg->active_capacity != L.cfg.active_capacity)
    return fail(XKNN_ERR_CONFIG,
                "m_active, max_batch, precision and active_capacity are fixed at creation");
  XK_TRY_H(check_scale(cfg));
  // a prepared selection drew from the old rng_seed: the next step selects again
  XK_TRY_H(L.cancel_prepared());
  L.cfg.scale = cfg->scale;
  L.cfg.momentum = cfg->momentum;
  L.cfg.weight_decay = cfg->weight_decay;
  L.cfg.rng_seed = cfg->rng_seed;
  L.cfg.flags = cfg->flags;
  L.drop_graphs();
  return XKNN_OK;
}

static cudaMemcpyKind kind_in(int on_device) {
  return on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
}
static cudaMemcpyKind kind_out(int on_device) {
  return on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
}

xknn_status_t xknn_layer_set_draw_stream(xknn_layer_t* h, const uint64_t* words, uint64_t count) {
  GUARD_H(h);
  Layer& L = h->L;
  XK_TRY_H(L.cancel_prepared());
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  if (L.side) XK_CUDA_H(cudaStreamSynchronize(L.side));
  L.drop_graphs();  // the cache pointer is baked into the captured steps
  if (L.mt_cache) cudaFree(L.mt_cache);
  L.mt_cache = nullptr;
  L.mt_len = 0;
  L.mt_injected = false;
  if (!words) return XKNN_OK;  // back to mt19937_64(rng_seed)
  if (count < L.cfg.m_active)
    return fail(XKNN_ERR_INVALID_ARGUMENT, "draw stream shorter than m_active");
  XK_CUDA_H(xknn::dalloc(&L.mt_cache, count));
  XK_CUDA_H(cudaMemcpy(L.mt_cache, words, count * sizeof(uint64_t), cudaMemcpyHostToDevice));
  L.mt_len = count;
  L.mt_injected = true;
  return XKNN_OK;
}

xknn_status_t xknn_layer_set_weights(xknn_layer_t* h, const float* w, int on_device) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.select_only) return fail(XKNN_ERR_UNSUPPORTED, "select-only layer has no parameters");
  cudaError_t e = cudaMemcpyAsync(L.W, w, L.nw * L.d * sizeof(float), kind_in(on_device), L.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L.stream);
  L.has_weights = true;
  return L.cuda_ok(e);
}

xknn_status_t xknn_layer_get_weights(xknn_layer_t* h, float* w, int on_device) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.select_only) return fail(XKNN_ERR_UNSUPPORTED, "select-only layer has no parameters");
  cudaError_t e = cudaMemcpyAsync(w, L.W, L.nw * L.d * sizeof(float), kind_out(on_device), L.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L.stream);
  return L.cuda_ok(e);
}

xknn_status_t xknn_layer_get_velocity(xknn_layer_t* h, float* v, int on_device) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.select_only) return fail(XKNN_ERR_UNSUPPORTED, "select-only layer has no parameters");
  cudaError_t e = cudaMemcpyAsync(v, L.V, L.nw * L.d * sizeof(float), kind_out(on_device), L.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L.stream);
  return L.cuda_ok(e);
}

xknn_status_t xknn_layer_weights_ptr(xknn_layer_t* h, float** w_dev) {
  GUARD_H(h);
  if (h->L.select_only) return fail(XKNN_ERR_UNSUPPORTED, "select-only layer has no parameters");
  *w_dev = h->L.W;
  h->L.has_weights = true;
  return XKNN_OK;
}

namespace {
__global__ void k_graph_check(const uint32_t* kpc, const uint64_t* off, const uint32_t* flat,
                              uint64_t n, uint64_t flat_len, uint64_t begin, uint64_t end,
                              unsigned int* kmax, unsigned long long* bad) {
  xknn::griddep_wait();
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < n;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = kpc[c];
    const uint64_t o = off[c];
    atomicMax(kmax, k);
    if (o + k > flat_len || (c + 1 < n && off[c + 1] != o + k)) { atomicAdd(bad, 1ull); continue; }
    for (uint32_t r = 0; r < k; ++r) {
      const uint64_t v = flat[o + r];
      if (v < begin || v >= end) { atomicAdd(bad, 1ull); break; }
    }
  }
}
}  // namespace

xknn_status_t xknn_layer_graph_buffers(xknn_layer_t* h, uint64_t flat_len, uint32_t** kpc_dev,
                                       uint64_t** off_dev, uint32_t** flat_dev) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.g_kpc) cudaFree(L.g_kpc);
  if (L.g_off) cudaFree(L.g_off);
  if (L.g_flat) cudaFree(L.g_flat);
  if (L.g_rank) cudaFree(L.g_rank);
  L.g_kpc = nullptr;
  L.g_off = nullptr;
  L.g_flat = nullptr;
  L.g_rank = nullptr;
  L.g_flat_len = 0;
  L.has_graph = false;
  L.drop_graphs();  // graph buffers are baked into the graphs
  // a selection prepared from the old graph is never used after the graph changes (the
  // reference selects from the current graph at step time)
  XK_TRY_H(L.cancel_prepared());
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  XK_CUDA_H(xknn::dalloc(&L.g_kpc, L.n));
  XK_CUDA_H(xknn::dalloc(&L.g_off, L.n));
  XK_CUDA_H(xknn::dalloc(&L.g_flat, flat_len));
  L.g_flat_len = flat_len;
  if (kpc_dev) *kpc_dev = L.g_kpc;
  if (off_dev) *off_dev = L.g_off;
  if (flat_dev) *flat_dev = L.g_flat;
  return XKNN_OK;
}

xknn_status_t xknn_layer_graph_commit(xknn_layer_t* h) {
  GUARD_H(h);
  Layer& L = h->L;
  if (!L.g_kpc) return fail(XKNN_ERR_INVALID_ARGUMENT, "graph_commit: no graph buffers");
  const uint64_t flat_len = L.g_flat_len;
  unsigned int* dk;
  unsigned long long* db;
  XK_CUDA_H(cudaMalloc(&dk, 16));
  db = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(dk) + 8);
  XK_CUDA_H(cudaMemsetAsync(dk, 0, 16, L.stream));
  xknn::launch_pdl(k_graph_check, xknn::grid_for(L.n, 256), 256, 0, L.stream, L.g_kpc, L.g_off, L.g_flat, L.n,
                                                                 flat_len, L.begin, L.end, dk, db);
  ++L.launches;
  unsigned int kmax = 0;
  unsigned long long bad = 0;
  XK_CUDA_H(cudaMemcpyAsync(&kmax, dk, 4, cudaMemcpyDeviceToHost, L.stream));
  XK_CUDA_H(cudaMemcpyAsync(&bad, db, 8, cudaMemcpyDeviceToHost, L.stream));
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  cudaFree(dk);
  if (bad) return fail(XKNN_ERR_SHAPE_MISMATCH, "graph CSR inconsistent or entries outside shard");
  // global bound on one label's pooled slice length: sum over shards of their longest slice
  if (L.world > 1) {
    unsigned int* dv;
    XK_CUDA_H(cudaMalloc(&dv, 4));
    XK_CUDA_H(cudaMemcpyAsync(dv, &kmax, 4, cudaMemcpyHostToDevice, L.stream));
    ncclResult_t r = ncclAllReduce(dv, dv, 1, ncclUint32, ncclSum, L.comm, L.stream);
    if (r != ncclSuccess) return L.nccl_ok(r);
    XK_CUDA_H(cudaMemcpyAsync(&kmax, dv, 4, cudaMemcpyDeviceToHost, L.stream));
    XK_CUDA_H(cudaStreamSynchronize(L.stream));
    cudaFree(dv);
  }
  L.g_kmax = kmax;
  const uint64_t hl = (uint64_t)kmax + L.bmax + 2;
  if (hl > L.hist_len) {
    if (L.hist) cudaFree(L.hist);
    XK_CUDA_H(xknn::dalloc(&L.hist, hl));
    L.hist_len = hl;
  }
  L.has_graph = true;
  return XKNN_OK;
}

xknn_status_t xknn_layer_set_graph_csr_ranked(xknn_layer_t* h, const uint32_t* kpc,
                                              const uint64_t* off, const uint32_t* flat,
                                              const uint32_t* rank, uint64_t flat_len,
                                              int on_device) {
  GUARD_H(h);
  Layer& L = h->L;
  XK_TRY_H(xknn_layer_graph_buffers(h, flat_len, nullptr, nullptr, nullptr));
  XK_CUDA_H(cudaMemcpyAsync(L.g_kpc, kpc, L.n * 4, kind_in(on_device), L.stream));
  XK_CUDA_H(cudaMemcpyAsync(L.g_off, off, L.n * 8, kind_in(on_device), L.stream));
  if (flat_len)
    XK_CUDA_H(cudaMemcpyAsync(L.g_flat, flat, flat_len * 4, kind_in(on_device), L.stream));
  if (rank) {
    XK_CUDA_H(xknn::dalloc(&L.g_rank, flat_len));
    if (flat_len)
      XK_CUDA_H(cudaMemcpyAsync(L.g_rank, rank, flat_len * 4, kind_in(on_device), L.stream));
  }
  return xknn_layer_graph_commit(h);
}

xknn_status_t xknn_layer_set_graph_csr(xknn_layer_t* h, const uint32_t* kpc, const uint64_t* off,
                                       const uint32_t* flat, uint64_t flat_len, int on_device) {
  return xknn_layer_set_graph_csr_ranked(h, kpc, off, flat, nullptr, flat_len, on_device);
}

xknn_status_t xknn_select(xknn_layer_t* h, const uint32_t* labels_dev, uint64_t batch,
                          uint32_t* out_active_dev, uint64_t* count_host, int* contains_all) {
  GUARD_H(h);
  Layer& L = h->L;
  if (!L.has_graph) return fail(XKNN_ERR_INVALID_ARGUMENT, "knn mode without shard graphs");
  if (batch == 0 || batch > L.bmax) return fail(XKNN_ERR_INVALID_ARGUMENT, "batch outside (0, max_batch]");
  if (L.prepared) {  // a pending prepared selection is superseded
    XK_CUDA_H(cudaStreamWaitEvent(L.stream, L.ev_prep, 0));
    L.prepared = false;
  }
  L.use_set(L.par);
  XK_CUDA_H(cudaMemcpyAsync(L.labels_all, labels_dev, batch * 4, cudaMemcpyDeviceToDevice, L.stream));
  xknn_status_t s = L.run_selection(batch);
  if (s != XKNN_OK) return s;
  xknn::SelState hs;
  XK_CUDA_H(cudaMemcpyAsync(&hs, L.st, sizeof(hs), cudaMemcpyDeviceToHost, L.stream));
  s = xknn_layer_sync(h);
  if (s != XKNN_OK) return s;
  if (out_active_dev && hs.active_count)
    XK_CUDA_H(cudaMemcpyAsync(out_active_dev, L.active, hs.active_count * 4,
                              cudaMemcpyDeviceToDevice, L.stream));
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  if (count_host) *count_host = hs.active_count;
  if (contains_all) *contains_all = hs.labels_found == hs.labels_local;
  return XKNN_OK;
}

xknn_status_t xknn_prepare(xknn_layer_t* h, const uint32_t* labels_local, uint64_t bl,
                           void* ready_stream) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.select_only) return fail(XKNN_ERR_UNSUPPORTED, "select-only layer: no train step");
  if (!L.has_graph) return fail(XKNN_ERR_INVALID_ARGUMENT, "prepare: knn mode without shard graphs");
  if (bl == 0 || bl * L.world > L.bmax)
    return fail(XKNN_ERR_INVALID_ARGUMENT, "prepare: batch size must be a positive multiple of P (<= max_batch)");
  return L.run_prepare(labels_local, bl, static_cast<cudaStream_t>(ready_stream));
}

xknn_status_t xknn_step_micro(xknn_layer_t* h, const float* feats, const uint32_t* labels,
                              uint64_t bl, float lr, uint32_t micro_batches, double* loss_dev,
                              float* gfeat) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.select_only) return fail(XKNN_ERR_UNSUPPORTED, "select-only layer: no train step");
  if (!L.has_graph) return fail(XKNN_ERR_INVALID_ARGUMENT, "train_step: knn mode without shard graphs");
  if (bl == 0 || bl * L.world > L.bmax)
    return fail(XKNN_ERR_INVALID_ARGUMENT, "train_step: batch size must be a positive multiple of P (<= max_batch)");
  return L.run_step(feats, labels, bl, lr, loss_dev, gfeat, micro_batches);
}

xknn_status_t xknn_step(xknn_layer_t* h, const float* feats, const uint32_t* labels,
                        uint64_t bl, float lr, double* loss_dev, float* gfeat) {
  return xknn_step_micro(h, feats, labels, bl, lr, 1, loss_dev, gfeat);
}

xknn_status_t xknn_layer_sync(xknn_layer_t* h) {
  GUARD_H(h);
  Layer& L = h->L;
  unsigned long long w = 0;
  XK_CUDA_H(cudaMemcpyAsync(&w, L.err, 8, cudaMemcpyDeviceToHost, L.stream));
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  if (w) {
    XK_CUDA_H(cudaMemsetAsync(L.err, 0, 8, L.stream));
    XK_TRY_H(L.reset_fast_scratch());
    XK_TRY_H(L.reset_fast32_scratch());
    XK_CUDA_H(cudaStreamSynchronize(L.stream));
    const xknn_status_t code = (xknn_status_t)(w & 0xff);
    xknn::g_row = w >> 8;
    return fail(code, std::string(xknn_status_string(code)) + " (device, index " +
                          std::to_string(w >> 8) + ")");
  }
  return XKNN_OK;
}

xknn_status_t xknn_layer_last_active(xknn_layer_t* h, uint64_t* total, uint64_t* local) {
  GUARD_H(h);
  Layer& L = h->L;
  xknn::SelState hs;
  XK_CUDA_H(cudaMemcpyAsync(&hs, L.ss[L.last_par].st, sizeof(hs), cudaMemcpyDeviceToHost,
                            L.stream));
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  if (total) *total = hs.active_total;
  if (local) *local = hs.active_count;
  return XKNN_OK;
}

xknn_status_t xknn_layer_last_logits(xknn_layer_t* h, float* out, uint64_t capacity) {
  GUARD_H(h);
  Layer& L = h->L;
  if (L.cfg.precision != XKNN_PREC_FP32_EXACT)
    return fail(XKNN_ERR_UNSUPPORTED, "logits are only materialized in FP32_EXACT precision");
  xknn::SelState hs;
  XK_CUDA_H(cudaMemcpyAsync(&hs, L.st, sizeof(hs), cudaMemcpyDeviceToHost, L.stream));
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  const uint64_t cnt = L.last_b * hs.active_count;
  if (capacity < cnt) return fail(XKNN_ERR_SHAPE_MISMATCH, "capacity below B x active_local");
  XK_CUDA_H(cudaMemcpyAsync(out, L.logits, cnt * 4, cudaMemcpyDeviceToHost, L.stream));
  XK_CUDA_H(cudaStreamSynchronize(L.stream));
  return XKNN_OK;
}

uint64_t xknn_layer_kernel_launches(const xknn_layer_t* h) { return h ? h->L.launches : 0; }

xknn_status_t xknn_layer_profile(xknn_layer_t* h, int enable) {
  GUARD_H(h);
  Layer& L = h->L;
  if (enable && L.prof_ev.empty()) {
    L.prof_ev.resize(Layer::kRing * Layer::kMarks);
    for (auto& e : L.prof_ev) XK_CUDA_H(cudaEventCreate(&e));
  }
  L.prof_collect(true);
  L.prof_on = enable != 0;
  L.drop_graphs();  // re-capture with/without the marks
  L.prof_ms.assign(Layer::kMarks, 0.0);
  L.prof_steps = L.prof_done = 0;
  return XKNN_OK;
}

xknn_status_t xknn_layer_phase_ms(xknn_layer_t* h, double* out, int n, uint64_t* steps) {
  GUARD_H(h);
  Layer& L = h->L;
  L.prof_collect(true);
  for (int i = 0; i < n && i + 1 < Layer::kMarks; ++i)
    out[i] = L.prof_ms.empty() ? 0.0 : L.prof_ms[i];
  if (steps) *steps = L.prof_done;
  return XKNN_OK;
}

}  // extern "C"
