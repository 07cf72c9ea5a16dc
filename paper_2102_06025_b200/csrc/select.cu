// select.cu -- Algorithm 1 active-class selection on device, bit-exact with
// select_active_classes(span<CompressedKnnGraph>) (knn_softmax.cpp:117-134) and
// finish_selection (knn_softmax.cpp:17-81), executed shard-parallel.
//
// Every shard holds the CSR graph pruned to its own classes (compress_graph,
// knn_graph.cpp:235-266), so the pool restricted to a shard is exactly the union of that
// shard's slices: each rank builds its part of the pool locally (bitmap over its class range,
// atomicMin rank / atomicAdd occurrence per candidate), and only P pool counts cross NVLink.
//
// Padding branch (|pool| < M, the default M = 10% N): the reference draws
// j_i = uniform_int_distribution<size_t>(i, |C|-1)(mt19937_64(seed)) and swaps C[i], C[j_i]
// over the ascending complement C (knn_softmax.cpp:39-49).  The reference re-seeds on every
// call, so the raw 64-bit stream is a constant of the layer (cached in HBM).  Each draw is
// Lemire's multiply-high (uniform_int_dist.h:257-274); rejections (p ~ range/2^64) are
// detected and replayed sequentially.  The Fisher-Yates result is resolved without the
// complement array: out[i] = C0[src(i)], where src follows "last writer" chains over the
// picks sorted by (j, i).  Positions map to classes by rank/select against the sorted pool.
//
// Over-full branch (|pool| > M): labels first, then the global top-(M - |labels|) by
// (best_rank asc, occurrences desc, class asc) (knn_softmax.cpp:61-67) via two histogram
// all-reduces and a rank-ordered tie split -- the keys are shard-local because every class
// lives in exactly one shard.
#include <cub/cub.cuh>

#include "layer.cuh"

namespace xknn {

namespace {

constexpr int kCompactBlock = 256;

// ---- pool marking: one warp per batch label, lanes stride the label's slice; lane 0 also
// marks the label (distinct labels of this shard counted as newly set bits).  A label's list is
// its slice of this shard's CompressedKnnGraph; with per-entry ranks it may be the concatenation
// of several shards' slices (the span<CompressedKnnGraph> overload on one device), each entry
// ranked within its own slice (knn_softmax.cpp:125-130).
__global__ void k_mark_pool(const uint32_t* __restrict__ labels, uint32_t batch, uint64_t n,
                            uint64_t begin, uint64_t nw, const uint32_t* __restrict__ kpc,
                            const uint64_t* __restrict__ off, const uint32_t* __restrict__ flat,
                            const uint32_t* __restrict__ rankv, uint32_t* pool_bits,
                            uint32_t* lab_bits, uint32_t* best, uint32_t* occ, SelState* st,
                            unsigned long long* err, int track) {
  griddep_wait();
  griddep_launch();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t newlab = 0;
  for (uint32_t i = warp; i < batch; i += nwarps) {
    const uint32_t y = labels[i];
    if (y >= n) {
      if (lane == 0) raise_error(err, XKNN_ERR_LABEL_OUT_OF_RANGE, i);
      continue;
    }
    if (lane == 0 && y >= begin && y - begin < nw) {
      const uint64_t lc = y - begin;
      const uint32_t bit = 1u << (lc & 31);
      if (!(atomicOr(&lab_bits[lc >> 5], bit) & bit)) ++newlab;
    }
    const uint32_t kk = kpc[y];
    const uint64_t o = off[y];
    for (uint32_t r = lane; r < kk; r += 32) {
      const uint64_t lc = (uint64_t)flat[o + r] - begin;
      if (lc >= nw) continue;  // validated at set_graph time
      atomicOr(&pool_bits[lc >> 5], 1u << (lc & 31));
      if (track) {  // candidate rank / occurrences: only the over-full branch ranks by them
        // rank = position within the slice, or the caller's per-entry rank (several shards'
        // slices merged into one list: xknn_layer_set_graph_csr_ranked)
        atomicMin(&best[lc], rankv ? rankv[o + r] : r);
        atomicAdd(&occ[lc], 1u);
      }
    }
  }
  newlab = warp_sum(newlab);
  if (lane == 0 && newlab) atomicAdd(&st->labels_local, newlab);
}

// ---- bitmap -> sorted list compaction (one 32-bit word per thread, block scan, sorted by
// construction).  mode 0: the pool bitmap.  mode 1: the final active set = act | pool (padding /
// exact fit, knn_softmax.cpp:32-51) or act | labels (over-full, :52-72).
__device__ __forceinline__ uint32_t final_word(int mode, const SelState* st, const uint32_t* act,
                                               const uint32_t* pool, const uint32_t* lab,
                                               uint64_t w) {
  if (mode == 0) return pool[w];
  return act[w] | (st->branch == kOverfull ? lab[w] : pool[w]);
}

// exclusive scan of the per-block counts (nblocks + 1 entries, last is the total), one CTA
__global__ void k_scan_blocks(const uint32_t* __restrict__ in, uint32_t n, uint32_t* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  using BS = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < n ? in[i] : 0;
    uint32_t x, tot;
    BS(tmp).ExclusiveSum(v, x, tot);
    if (i < n) out[i] = carry + x;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

__global__ void k_bits_count(int mode, SelState* st, const uint32_t* __restrict__ act,
                             const uint32_t* __restrict__ pool, const uint32_t* __restrict__ lab,
                             uint64_t nwords, uint32_t* blk_counts) {
  griddep_wait();
  griddep_launch();
  using BR = cub::BlockReduce<uint32_t, kCompactBlock>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ typename BR::TempStorage tmp2;
  const uint64_t w = (uint64_t)blockIdx.x * kCompactBlock + threadIdx.x;
  uint32_t word = 0, found = 0;
  if (w < nwords) {
    word = final_word(mode, st, act, pool, lab, w);
    if (mode == 1) found = __popc(word & lab[w]);
  }
  const uint32_t c = BR(tmp).Sum(__popc(word));
  if (threadIdx.x == 0) blk_counts[blockIdx.x] = c;
  if (mode == 1) {
    const uint32_t f = BR(tmp2).Sum(found);
    if (threadIdx.x == 0 && f) atomicAdd(&st->labels_found, f);
  }
}

__global__ void k_bits_write(int mode, SelState* st, const uint32_t* __restrict__ act,
                             const uint32_t* __restrict__ pool, const uint32_t* __restrict__ lab,
                             uint64_t nwords, const uint32_t* __restrict__ blk_off,
                             uint32_t nblocks, uint32_t base, uint32_t* __restrict__ out,
                             uint32_t* __restrict__ pos_of, unsigned long long* pool_counts,
                             int rank, uint32_t* __restrict__ samp,
                             unsigned long long* __restrict__ err, uint32_t cap) {
  griddep_wait();
  griddep_launch();
  using BS = cub::BlockScan<uint32_t, kCompactBlock>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t w = (uint64_t)blockIdx.x * kCompactBlock + threadIdx.x;
  // a step that already failed (MTooSmall, LabelOutOfRange, ...) gets an empty active set: the
  // reference throws before any of it runs, and an over-full set would not fit the capacity
  // a final set larger than the layer's active capacity (xknn_config_t::active_capacity) is not
  // written: OutOfMemory, as an allocation failure of the reference would be
  const bool over = mode == 1 && blk_off[nblocks] > cap;
  if (over && blockIdx.x == 0 && threadIdx.x == 0)
    raise_error(err, XKNN_ERR_OUT_OF_MEMORY, blk_off[nblocks]);
  const bool dead = mode == 1 && (over || *err != 0);
  uint32_t word = 0;
  if (w < nwords && !dead) word = final_word(mode, st, act, pool, lab, w);
  uint32_t pos;
  BS(tmp).ExclusiveSum(__popc(word), pos);
  pos += blk_off[blockIdx.x];
  while (word) {
    const uint32_t bit = __ffs(word) - 1;
    const uint32_t lc = (uint32_t)(w * 32 + bit);
    out[pos] = base + lc;
    if (pos_of) pos_of[lc] = pos;
    if (samp && (pos & 63) == 0) samp[pos >> 6] = lc - pos;  // g(pos) for k_pad_map
    ++pos;
    word &= word - 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t total = blk_off[nblocks];
    if (mode == 0) {
      st->pool_count = total;
      st->pool_local = total;
      pool_counts[2 * rank] = total;              // exchanged: [pool, distinct labels] per shard
      pool_counts[2 * rank + 1] = st->labels_local;
    } else {
      st->active_count = (dead || over) ? 0u : total;
    }
  }
}

// ---- the plan: which branch, how many pads, which complement positions this shard owns
__global__ void k_plan(SelState* st, const unsigned long long* pool_counts, int world, int rank,
                       uint64_t n, uint64_t m, uint64_t begin, uint64_t nw,
                       unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  unsigned long long total = 0, before = 0, nd = 0;
  for (int s = 0; s < world; ++s) {
    total += pool_counts[2 * s];
    nd += pool_counts[2 * s + 1];  // shards own disjoint class ranges
    if (s < rank) before += pool_counts[2 * s];
  }
  st->pool_total = total;
  st->nd = nd;
  st->csize = n - total;
  st->cbase = begin - before;
  st->compl_local = nw - pool_counts[2 * rank];
  st->first_rej = kNone;
  st->need = 0;
  st->take = 0;
  if (m < nd) raise_error(err, XKNN_ERR_M_TOO_SMALL);          // knn_softmax.cpp:24-27
  if (m > n) raise_error(err, XKNN_ERR_INVALID_ARGUMENT);      // knn_softmax.cpp:28-29
  if (total < m) {
    st->branch = kPad;
    st->need = m - total;
  } else if (total == m) {
    st->branch = kExact;
  } else {
    st->branch = kOverfull;
    st->take = m > nd ? m - nd : 0;
  }
  st->active_total = m;
}

// ---- padding: Lemire draws from the cached mt19937_64 stream
__global__ void k_picks(SelState* st, const uint64_t* __restrict__ mt, uint32_t* __restrict__ key) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kPad) return;
  const uint64_t need = st->need, csize = st->csize;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < need;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t range = csize - i;  // __uerange = (csize-1) - i + 1
    const uint64_t u = mt[i];
    const uint64_t lo = u * range;
    if (lo < range) {
      const uint64_t thr = (0ull - range) % range;
      if (lo < thr) atomicMin(&st->first_rej, (unsigned)i);
    }
    key[i] = (uint32_t)(i + __umul64hi(u, range));
  }
}

// Sequential replay from the first rejected draw (uniform_int_dist.h:268-272).  Taken with
// probability ~ need*csize/2^64 per step.
__global__ void k_picks_replay(SelState* st, const uint64_t* __restrict__ mt, uint64_t mt_len,
                               uint32_t* key, unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kPad || st->first_rej == kNone) return;
  const uint64_t need = st->need, csize = st->csize;
  uint64_t pos = st->first_rej;
  for (uint64_t i = st->first_rej; i < need; ++i) {
    const uint64_t range = csize - i;
    if (pos >= mt_len) { raise_error(err, XKNN_ERR_UNSUPPORTED); return; }
    uint64_t u = mt[pos++];
    uint64_t lo = u * range;
    if (lo < range) {
      const uint64_t thr = (0ull - range) % range;
      while (lo < thr) {
        if (pos >= mt_len) { raise_error(err, XKNN_ERR_UNSUPPORTED); return; }
        u = mt[pos++];
        lo = u * range;
      }
    }
    key[i] = (uint32_t)(i + __umul64hi(u, range));
  }
}

// Group the picks by complement position: a singly linked list per position (arbitrary order),
// heads in a dense u32[N] table that is all-kNone between steps.  Uniform picks collide rarely
// (~need^2 / 2|C| pairs), so groups have one or two members.
__global__ void k_link(const SelState* st, const uint32_t* __restrict__ key, uint32_t* head,
                       uint32_t* __restrict__ nxt, uint32_t* __restrict__ lw) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kPad) return;
  const uint32_t need = (uint32_t)st->need;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < need; i += gridDim.x * blockDim.x) {
    nxt[i] = atomicExch(&head[key[i]], i);
    lw[i] = kNone;
  }
}

// One thread per group (the current list head): within the group of position j,
//   pred[t] = largest member below t   (the swap that last wrote position j before step t)
//   lw[j]   = largest member below j   (the last value moved into position j before step j)
__global__ void k_resolve(const SelState* st, const uint32_t* __restrict__ key,
                          const uint32_t* __restrict__ head, const uint32_t* __restrict__ nxt,
                          uint32_t* __restrict__ pred, uint32_t* __restrict__ lw) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kPad) return;
  const uint32_t need = (uint32_t)st->need;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < need; i += gridDim.x * blockDim.x) {
    const uint32_t j = key[i];
    if (head[j] != i) continue;
    uint32_t lwj = kNone;
    for (uint32_t a = i; a != kNone; a = nxt[a]) {
      uint32_t p = kNone;
      for (uint32_t b = i; b != kNone; b = nxt[b])
        if (b < a && (p == kNone || b > p)) p = b;
      pred[a] = p;
      if (a < j && (lwj == kNone || a > lwj)) lwj = a;
    }
    if (j < need) lw[j] = lwj;
  }
}

// out[i] = C0[src(i)]; the shard owning complement position src marks the class
__global__ void k_pad_map(const SelState* st, const uint32_t* __restrict__ key,
                          const uint32_t* __restrict__ pred, const uint32_t* __restrict__ lw,
                          const uint32_t* __restrict__ pool_list,
                          const uint32_t* __restrict__ samp, uint64_t begin,
                          uint32_t* act_bits, uint32_t* head) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kPad) return;
  const uint64_t need = st->need, cbase = st->cbase, cl = st->compl_local;
  const uint32_t npool = st->pool_count;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < need;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t src;
    head[key[i]] = kNone;  // leave the group table clean for the next step
    uint32_t t = pred[i];
    if (t != kNone) {
      while (lw[t] != kNone) t = lw[t];
      src = t;
    } else {
      src = key[i];
    }
    if (src < cbase || src >= cbase + cl) continue;
    const uint64_t q = src - cbase;  // q-th class of [begin,end) outside the pool
    // first pool position p with g(p) = (pool_list[p] - begin) - p > q: over the every-64th
    // samples of g (small, cache-resident), then within one 64-entry stretch of pool_list
    const uint32_t nsamp = (npool + 63) / 64;
    uint32_t lo = 0, hi = nsamp;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((uint64_t)samp[mid] <= q) lo = mid + 1; else hi = mid;
    }
    hi = min(lo * 64, npool);
    lo = lo ? (lo - 1) * 64 : 0;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((uint64_t)(pool_list[mid] - begin) - mid <= q) lo = mid + 1; else hi = mid;
    }
    const uint64_t lc = q + lo;
    atomicOr(&act_bits[lc >> 5], 1u << (lc & 31));
  }
}

// ---- over-full ranking
__global__ void k_of_hist_rank(const SelState* st, const uint32_t* __restrict__ pool_list,
                               uint64_t begin, const uint32_t* __restrict__ lab_bits,
                               const uint32_t* __restrict__ best, uint32_t* hist) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kOverfull) return;
  const uint32_t np = st->pool_count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const uint32_t lc = pool_list[i] - (uint32_t)begin;
    if (lab_bits[lc >> 5] & (1u << (lc & 31))) continue;
    atomicAdd(&hist[best[lc]], 1u);
  }
}

__global__ void k_of_plan_rank(SelState* st, const uint32_t* hist, uint32_t nbins) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kOverfull) return;
  const unsigned long long t = st->take;
  unsigned long long cum = 0;
  uint32_t r = nbins;
  for (uint32_t b = 0; b < nbins; ++b) {
    if (cum + hist[b] >= t) { r = b; break; }
    cum += hist[b];
  }
  st->r_star = r;
  st->tie_quota = t - cum;  // still needed at rank r_star
}

__global__ void k_of_hist_occ(const SelState* st, const uint32_t* __restrict__ pool_list,
                              uint64_t begin, const uint32_t* __restrict__ lab_bits,
                              const uint32_t* __restrict__ best, const uint32_t* __restrict__ occ,
                              uint32_t* hist) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kOverfull) return;
  const uint32_t np = st->pool_count, rs = st->r_star;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const uint32_t lc = pool_list[i] - (uint32_t)begin;
    if (lab_bits[lc >> 5] & (1u << (lc & 31))) continue;
    if (best[lc] == rs) atomicAdd(&hist[occ[lc]], 1u);
  }
}

__global__ void k_of_plan_occ(SelState* st, const uint32_t* hist, uint32_t nbins) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kOverfull) return;
  const unsigned long long t = st->tie_quota;
  unsigned long long cum = 0;
  uint32_t o = 0;
  bool found = false;
  for (int b = (int)nbins - 1; b >= 0; --b) {  // occurrences descending
    if (cum + hist[b] >= t) { o = (uint32_t)b; found = true; break; }
    cum += hist[b];
  }
  st->o_star = found ? o : 0;
  st->tie_quota = found ? t - cum : 0;
}

__global__ void k_of_tie_count(SelState* st, const uint32_t* __restrict__ pool_list,
                               uint64_t begin, const uint32_t* __restrict__ lab_bits,
                               const uint32_t* __restrict__ best, const uint32_t* __restrict__ occ,
                               unsigned long long* tie_counts, int rank) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kOverfull) { if (threadIdx.x == 0 && blockIdx.x == 0) tie_counts[rank] = 0; return; }
  const uint32_t np = st->pool_count, rs = st->r_star, os = st->o_star;
  __shared__ unsigned int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
    const uint32_t lc = pool_list[i] - (uint32_t)begin;
    if (lab_bits[lc >> 5] & (1u << (lc & 31))) continue;
    if (best[lc] == rs && occ[lc] == os) atomicAdd(&cnt, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) tie_counts[rank] = cnt;
}

// single block: labels, strictly better candidates, and this shard's share of the ties (lowest
// class ids first; shards are ordered by class range so rank order == class order)
__global__ void k_of_select(SelState* st, const uint32_t* __restrict__ pool_list, uint64_t begin,
                            const uint32_t* __restrict__ lab_bits, const uint32_t* __restrict__ best,
                            const uint32_t* __restrict__ occ, const unsigned long long* tie_counts,
                            int rank, uint32_t nbins_rank, uint32_t* act_bits) {
  griddep_wait();
  griddep_launch();
  if (st->branch != kOverfull) return;
  using BS = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  unsigned long long before = 0;
  for (int s = 0; s < rank; ++s) before += tie_counts[s];
  const unsigned long long need = st->tie_quota;
  const unsigned long long quota = need > before ? min(need - before, tie_counts[rank]) : 0;
  const uint32_t np = st->pool_count, rs = st->r_star, os = st->o_star;
  const bool all = rs >= nbins_rank;  // fewer candidates than take: keep every candidate
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < np; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    uint32_t lc = 0, tie = 0;
    bool sel = false;
    if (i < np) {
      lc = pool_list[i] - (uint32_t)begin;
      if (!(lab_bits[lc >> 5] & (1u << (lc & 31)))) {
        const uint32_t b = best[lc], o = occ[lc];
        if (all || b < rs || (b == rs && o > os)) sel = true;
        else if (b == rs && o == os) tie = 1;
      }
    }
    uint32_t idx, total;
    BS(tmp).ExclusiveSum(tie, idx, total);
    if (tie && carry + idx < quota) sel = true;
    if (sel) atomicOr(&act_bits[lc >> 5], 1u << (lc & 31));
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

// label -> column in this shard's active list (-1 if another shard owns it or it is absent:
// the softmax then reports LabelOutOfRange as distributed_softmax_xent_cols does, :157-161)
__global__ void k_label_cols(const SelState* st, const uint32_t* __restrict__ labels,
                             uint32_t batch, const uint32_t* __restrict__ active,
                             const uint32_t* __restrict__ pos_of, uint64_t begin, uint64_t end,
                             int32_t* label_col, const uint32_t* __restrict__ pool_list,
                             uint32_t* best, uint32_t* occ, int track) {
  griddep_wait();
  griddep_launch();
  const uint32_t na = st->active_count, np = track ? st->pool_count : 0;
  // reset the candidate ranks of this step's pool (every touched class is in the pool)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const uint32_t lc = pool_list[i] - (uint32_t)begin;
    best[lc] = kNone;
    occ[lc] = 0;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < batch; i += gridDim.x * blockDim.x) {
    const uint32_t y = labels[i];
    int32_t col = -1;
    if (y >= begin && y < end) {
      const uint32_t p = pos_of[y - begin];
      if (p < na && active[p] == y) col = (int32_t)p;
    }
    label_col[i] = col;
  }
}

__global__ void k_zero_sel(SelState* st) {
  griddep_wait();
  griddep_launch();
  st->labels_local = 0;
  st->labels_found = 0;
  st->pool_count = 0;
  st->active_count = 0;
}

}  // namespace

// Compacts this shard's bitmap (mode 0: pool, mode 1: final active set) into sorted global ids.
static xknn_status_t compact_bits(Layer& L, int mode, uint32_t* out, uint32_t* pos_of) {
  const uint32_t nblocks = (uint32_t)((L.nwords + kCompactBlock - 1) / kCompactBlock);
  launch_pdl(k_bits_count, nblocks, kCompactBlock, 0, L.stream, mode, L.st, L.act_bits, L.pool_bits,
                                                        L.lab_bits, L.nwords, L.blk_counts);
  ++L.launches;
  // blk_counts[nblocks] is kept 0, so the exclusive scan's last entry is the total
  launch_pdl(k_scan_blocks, 1, 1024, 0, L.stream, L.blk_counts, nblocks + 1, L.blk_counts + nblocks + 1);
  ++L.launches;
  launch_pdl(k_bits_write, nblocks, kCompactBlock, 0, L.stream, 
      mode, L.st, L.act_bits, L.pool_bits, L.lab_bits, L.nwords, L.blk_counts + nblocks + 1,
      nblocks, (uint32_t)L.begin, out, pos_of, L.pool_counts, L.rank,
      mode == 0 ? L.pool_samp : nullptr, L.err, mode == 0 ? 0xffffffffu : (uint32_t)L.mw_cap);
  ++L.launches;
  return L.cuda_ok(cudaGetLastError(), __FILE__, __LINE__, "k_bits_write");
}

xknn_status_t Layer::run_selection(uint64_t batch) {
  const uint32_t B = (uint32_t)batch;
  const uint64_t m = cfg.m_active;
  XK_TRY(ensure_mt_cache());
  // pool_bits, act_bits, lab_bits are one allocation
  XK_CUDA(cudaMemsetAsync(pool_bits, 0, 3 * nwords * sizeof(uint32_t), stream));
  launch_pdl(k_zero_sel, 1, 1, 0, stream, st);
  XK_LAUNCH();

  // (1) pool of this shard: union of its slices for every batch label (knn_softmax.cpp:122-132),
  //     candidate best rank / occurrences, and the labels this shard owns
  // the over-full ranking (and its per-candidate rank/occurrence tracking) is only reachable
  // when the pool can exceed M; the default M = 10% N never lets it
  const bool overfull_possible = (uint64_t)B * g_kmax > m;
  launch_pdl(k_mark_pool, grid_for((uint64_t)B * 32, 256), 256, 0, stream, 
      labels_all, B, n, begin, nw, g_kpc, g_off, g_flat, (const uint32_t*)g_rank, pool_bits, lab_bits, sel_best, sel_occ,
      st, err, overfull_possible ? 1 : 0);
  XK_LAUNCH();
  // (2) sorted local pool; [pool size, distinct labels] exchanged between shards
  XK_TRY(compact_bits(*this, 0, pool_list, nullptr));
  if (world > 1)
    XK_NCCL(ncclAllGather(pool_counts + 2 * rank, pool_counts, 2, ncclUint64, comm, stream));
  launch_pdl(k_plan, 1, 1, 0, stream, st, pool_counts, world, rank, n, m, begin, nw, err);
  XK_LAUNCH();

  // (3a) padding branch (|pool| < M): picks from the cached stream, Fisher-Yates chains
  if (m > 0) {
    launch_pdl(k_picks, grid_for(m, 256), 256, 0, stream, st, mt_cache, pick_key);
    XK_LAUNCH();
    launch_pdl(k_picks_replay, 1, 1, 0, stream, st, mt_cache, mt_len, pick_key, err);
    XK_LAUNCH();
    launch_pdl(k_link, grid_for(m, 256), 256, 0, stream, st, pick_key, pick_head, pick_val, lw);
    XK_LAUNCH();
    launch_pdl(k_resolve, grid_for(m, 256), 256, 0, stream, st, pick_key, pick_head, pick_val, pred, lw);
    XK_LAUNCH();
    launch_pdl(k_pad_map, grid_for(m, 256), 256, 0, stream, st, pick_key, pred, lw, pool_list,
               pool_samp, begin, act_bits, pick_head);
    XK_LAUNCH();
  }
  // (3b) over-full branch: only reachable when B * k could exceed M
  if (overfull_possible) {
    const uint32_t nb_rank = g_kmax ? g_kmax : 1;
    const uint32_t nb_occ = B + 1;
    uint32_t* h_rank = hist;
    uint32_t* h_occ = hist + nb_rank;
    XK_CUDA(cudaMemsetAsync(hist, 0, (nb_rank + nb_occ) * sizeof(uint32_t), stream));
    launch_pdl(k_of_hist_rank, grid_for(nw, 256), 256, 0, stream, st, pool_list, begin, lab_bits,
                                                          sel_best, h_rank);
    XK_LAUNCH();
    if (world > 1) XK_NCCL(ncclAllReduce(h_rank, h_rank, nb_rank, ncclUint32, ncclSum, comm, stream));
    launch_pdl(k_of_plan_rank, 1, 1, 0, stream, st, h_rank, nb_rank);
    XK_LAUNCH();
    launch_pdl(k_of_hist_occ, grid_for(nw, 256), 256, 0, stream, st, pool_list, begin, lab_bits,
                                                         sel_best, sel_occ, h_occ);
    XK_LAUNCH();
    if (world > 1) XK_NCCL(ncclAllReduce(h_occ, h_occ, nb_occ, ncclUint32, ncclSum, comm, stream));
    launch_pdl(k_of_plan_occ, 1, 1, 0, stream, st, h_occ, nb_occ);
    XK_LAUNCH();
    launch_pdl(k_of_tie_count, 1, 1024, 0, stream, st, pool_list, begin, lab_bits, sel_best, sel_occ,
                                           tie_counts, rank);
    XK_LAUNCH();
    if (world > 1)
      XK_NCCL(ncclAllGather(tie_counts + rank, tie_counts, 1, ncclUint64, comm, stream));
    launch_pdl(k_of_select, 1, 1024, 0, stream, st, pool_list, begin, lab_bits, sel_best, sel_occ,
                                        tie_counts, rank, nb_rank, act_bits);
    XK_LAUNCH();
  }
  // (4) this shard's ActiveSet slice, sorted by construction; label -> column map
  XK_TRY(compact_bits(*this, 1, active, pos_of));
  launch_pdl(k_label_cols,
             grid_for(overfull_possible ? std::max<uint64_t>(B, (uint64_t)B * g_kmax) : B, 256),
             256, 0, stream, st, labels_all, B, active, pos_of, begin, end, label_col, pool_list,
             sel_best, sel_occ, overfull_possible ? 1 : 0);
  XK_LAUNCH();
  return XKNN_OK;
}

}  // namespace xknn
