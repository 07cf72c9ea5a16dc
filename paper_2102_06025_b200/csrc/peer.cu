// peer.cu -- the softmax statistics all-reduce (B x 3 doubles per step, latency-bound) as one
// kernel over NVLink peer memory instead of an NCCL call.  Every rank pushes its vector into its
// slot of every rank's receive buffer (CUDA IPC mappings of the peers' buffers), publishes an
// epoch flag with a system-scope release store, waits for all ranks' flags with acquire loads,
// then sums the world vectors in rank order -- the same order, hence the same bits, on every
// rank (all_reduce_sum's rank-order sum, parallel.cpp:51-64).  Two slots alternate by epoch, so
// a rank can run one all-reduce ahead of a slow peer without overwriting data it still reads.
#include <cstring>
#include <vector>

#include "kernels.cuh"
#include "layer.cuh"

namespace xknn {

namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(1024)
    k_peer_allreduce(double* __restrict__ data, uint64_t n, uint64_t cap, int rank, int world,
                     double* const* __restrict__ pbuf, uint64_t* const* __restrict__ pflag,
                     const double* __restrict__ mybuf, const uint64_t* __restrict__ myflag,
                     uint64_t* __restrict__ epoch, unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  const uint64_t e = *epoch + 1, slot = e & 1u;
  const uint32_t tid = threadIdx.x;
  for (int q = 0; q < world; ++q) {
    double* dst = pbuf[q] + (slot * (uint64_t)world + (uint64_t)rank) * cap;
    for (uint64_t i = tid; i < n; i += blockDim.x) dst[i] = data[i];
  }
  __threadfence_system();
  __syncthreads();
  if ((int)tid < world) {
    st_release_sys(pflag[tid] + rank, e);
    // a peer that never arrives (crashed process) must not hang the GPU: give up after ~10 s
    const long long t0 = clock64();
    while (ld_acquire_sys(myflag + tid) < e) {
      if (clock64() - t0 > 20000000000LL) {
        raise_error(err, XKNN_ERR_NCCL);
        break;
      }
    }
  }
  __syncthreads();
  __threadfence();
  for (uint64_t i = tid; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < world; ++q) s += mybuf[(slot * (uint64_t)world + (uint64_t)q) * cap + i];
    data[i] = s;
  }
  if (tid == 0) *epoch = e;
}

}  // namespace

// Collective (every rank, once): buffers, IPC handle exchange over `comm`, peer mappings.  Every
// rank takes part in both collectives whatever happens locally, and the ranks agree (MIN
// all-reduce) on whether all of them succeeded -- a partial setup is released everywhere.
xknn_status_t PeerAllreduce::setup(int rank_, int world_, uint64_t cap_, ncclComm_t comm,
                                   cudaStream_t s) {
  rank = rank_;
  world = world_;
  cap = cap_;
  auto cu = [](cudaError_t e) { return e == cudaSuccess; };
  bool ok = cu(cudaMalloc(&buf, 2 * (size_t)world * cap * sizeof(double))) &&
            cu(cudaMalloc(&flags, (size_t)world * sizeof(uint64_t))) &&
            cu(cudaMalloc(&epoch, sizeof(uint64_t))) &&
            cu(cudaMemsetAsync(flags, 0, (size_t)world * sizeof(uint64_t), s)) &&
            cu(cudaMemsetAsync(epoch, 0, sizeof(uint64_t), s));
  cudaIpcMemHandle_t hb{}, hf{};
  ok = ok && cu(cudaIpcGetMemHandle(&hb, buf)) && cu(cudaIpcGetMemHandle(&hf, flags));
  const size_t hs = sizeof(cudaIpcMemHandle_t);
  std::vector<uint8_t> hh(2 * hs * world, 0);
  std::memcpy(hh.data() + 2 * hs * rank, &hb, hs);
  std::memcpy(hh.data() + 2 * hs * rank + hs, &hf, hs);
  uint8_t* dh = nullptr;
  int* dok = nullptr;
  if (!cu(cudaMalloc(&dh, 2 * hs * world)) || !cu(cudaMalloc(&dok, sizeof(int))))
    return fail_msg(XKNN_ERR_CUDA, "peer all-reduce: scratch");  // (the collectives need it)
  bool coll = cu(cudaMemcpyAsync(dh + 2 * hs * rank, hh.data() + 2 * hs * rank, 2 * hs,
                                 cudaMemcpyHostToDevice, s)) &&
              ncclAllGather(dh + 2 * hs * rank, dh, 2 * hs, ncclUint8, comm, s) == ncclSuccess &&
              cu(cudaMemcpyAsync(hh.data(), dh, 2 * hs * world, cudaMemcpyDeviceToHost, s)) &&
              cu(cudaStreamSynchronize(s));
  std::vector<double*> pb(world, nullptr);
  std::vector<uint64_t*> pf(world, nullptr);
  for (int q = 0; q < world && ok && coll; ++q) {
    if (q == rank) {
      pb[q] = buf;
      pf[q] = flags;
      continue;
    }
    cudaIpcMemHandle_t qb, qf;
    std::memcpy(&qb, hh.data() + 2 * hs * q, hs);
    std::memcpy(&qf, hh.data() + 2 * hs * q + hs, hs);
    void *vb = nullptr, *vf = nullptr;
    if (!cu(cudaIpcOpenMemHandle(&vb, qb, cudaIpcMemLazyEnablePeerAccess))) { ok = false; break; }
    opened.push_back(vb);
    if (!cu(cudaIpcOpenMemHandle(&vf, qf, cudaIpcMemLazyEnablePeerAccess))) { ok = false; break; }
    opened.push_back(vf);
    pb[q] = static_cast<double*>(vb);
    pf[q] = static_cast<uint64_t*>(vf);
  }
  ok = ok && coll && cu(cudaMalloc(&peer_bufs, world * sizeof(double*))) &&
       cu(cudaMalloc(&peer_flags, world * sizeof(uint64_t*))) &&
       cu(cudaMemcpy(peer_bufs, pb.data(), world * sizeof(double*), cudaMemcpyHostToDevice)) &&
       cu(cudaMemcpy(peer_flags, pf.data(), world * sizeof(uint64_t*), cudaMemcpyHostToDevice));
  // every rank agrees: all set up, or nobody uses it
  int hok = ok ? 1 : 0;
  coll = coll && cu(cudaMemcpyAsync(dok, &hok, sizeof(int), cudaMemcpyHostToDevice, s)) &&
         ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm, s) == ncclSuccess &&
         cu(cudaMemcpyAsync(&hok, dok, sizeof(int), cudaMemcpyDeviceToHost, s)) &&
         cu(cudaStreamSynchronize(s));
  cudaFree(dh);
  cudaFree(dok);
  (void)cudaGetLastError();
  if (!coll || hok != 1) return fail_msg(XKNN_ERR_CUDA, "peer all-reduce: not available");
  ready = true;
  return XKNN_OK;
}

cudaError_t PeerAllreduce::launch(double* data, uint64_t n, unsigned long long* err,
                                  cudaStream_t s) const {
  if (!ready || n > cap) return cudaErrorInvalidValue;
  launch_pdl(k_peer_allreduce, 1, 1024, 0, s, data, n, cap, rank, world,
             (double* const*)peer_bufs, (uint64_t* const*)peer_flags, (const double*)buf,
             (const uint64_t*)flags, epoch, err);
  return cudaGetLastError();
}

void PeerAllreduce::release() {
  for (void* p : opened) cudaIpcCloseMemHandle(p);
  opened.clear();
  for (void* p : {(void*)buf, (void*)flags, (void*)epoch, (void*)peer_bufs, (void*)peer_flags})
    if (p) cudaFree(p);
  buf = nullptr;
  flags = epoch = nullptr;
  peer_bufs = nullptr;
  peer_flags = nullptr;
  ready = false;
}

}  // namespace xknn
