// graph.cuh -- device KNN graph build (graph.cu) and its distributed compression
// (layer_graph.cu), shared declarations.
#pragma once
#include <nccl.h>

#include "common.cuh"

namespace xknn {

struct GraphBuildStats {
  uint64_t uncertified_rows = 0;  // rows recomputed by exact scans (certificate failed)
  uint64_t transfer_steps = 0;    // ring hops (RingBuildStats::transfer_steps, knn_graph.hpp:63-68)
};

// The rows [begin, end) of the exact KNN graph (N x k u32, global ids) for this rank's class
// block of the ShardLayout(n_total, world) (knn_graph.cpp:94-115).  wn: this rank's normalized
// rows (end - begin) x d fp32, device.  Collective over `comm` when world > 1.  Synchronizes s.
xknn_status_t graph_build(const float* wn, uint64_t n_total, uint64_t d, uint32_t k,
                          uint32_t kprime, int rank, int world, ncclComm_t comm, cudaStream_t s,
                          uint32_t* out, GraphBuildStats* stats);

// classify_retrieval on one shard (graph.cu): best class (score, global id) of each query.
xknn_status_t retrieval_top1_local(const float* qn, uint32_t nq, const float* wn, uint32_t nw,
                                   uint32_t col_base, uint32_t d, cudaStream_t s,
                                   float* best_score, uint32_t* best_id, uint64_t* uncertified);

}  // namespace xknn
