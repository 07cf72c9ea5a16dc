#!/usr/bin/env python
"""KNN-softmax fwd+bwd+update throughput on B200 (samples/s), driver contract of this repo.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3|c4|c4r|c1] [--precision fp32|bf16|fp32_exact]
                    [--no-bf16-line]

The headline runs XKNN_PREC_FP32 (fp32 accuracy, within 1e-5 of the fp32 reference, on tensor
cores: mixed tf32/bf16 logits GEMM, bf16x3 gradient GEMMs -- fast32.cu; XKNN_FP32_GEMM=3xtf32
selects 3xTF32 throughout); the same workload in the bf16 tensor-core mode is reported beside it
as `bf16_mode`.

One step = the fc half of HybridSim::train_step (parallel.cpp:455-572, :638-668) over one global
batch: feature/label all-gather, Algorithm-1 active-class selection, active-row gather +
normalize, logit GEMM + distributed softmax-CE, weight- and feature-gradient GEMMs, feature
normalize-backward, sparse momentum-SGD update of the active rows.

Workloads (BASELINE.json configs, D = 512, M = 10% N, s = 30, lr = 0.1, mu = 0.9):
    c1  N=100K  B=256   k=10    (the reference's CPU-runnable case; parity config)
    c2  N=1M    B=1024  k=50    the default at every N (configs[1]; strong-scaled over N GPUs)
    c3  N=10M   B=4096  k=100   class-sharded over 2/4/8 GPUs (--workload c3)
    c4  N=100M  B=8192  k=100   8 GPUs (paper headline scale); 25M classes/GPU on 4 GPUs
    c4r N=12.5M B=8192  k=100   one GPU: the per-rank work of C4 on 8 GPUs
Synthetic data: W ~ N(0, 0.05^2), features ~ N(0,1), labels uniform, a seeded self-first random
graph of k neighbours per class (random-init W makes the true KNN graph statistically random).
The per-step working set (weight shard, P~ of B x M_w bf16) exceeds the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
if os.environ.get("XKNN_PKG_DIR"):  # A/B runs against another build of the package
    sys.path.insert(0, os.environ["XKNN_PKG_DIR"])

WORKLOADS = {
    "c1": dict(n=100_000, b=256, k=10),
    "c2": dict(n=1_000_000, b=1024, k=50),
    "c3": dict(n=10_000_000, b=4096, k=100),
    "c4": dict(n=100_000_000, b=8192, k=100),
    # one rank of C4 on 8 GPUs, run on one GPU: its 12.5M-class shard, the global batch 8192,
    # k = 100, M_w = 1.25M active rows -- the GEMM/update work of a C4 rank (its selection differs:
    # the pool is drawn from 12.5M classes instead of 100M)
    "c4r": dict(n=12_500_000, b=8192, k=100),
}
D = 512
SCALE, LR, MOMENTUM, SEED = 30.0, 0.1, 0.9, 42
PHASES = ["allgather", "select", "gather_normalize", "gemm_logits_softmax", "softmax_stats",
          "gemm_dW", "gemm_dX", "dX_reduce_scatter", "update", "feature_backward"]


def peaks():
    """Roofline denominators.  HBM GB/s and bf16 TF/s (burst: best of 10; sustained: back to
    back for 4 s) from the driver-written MEASURED_PEAKS.json.  Fallbacks: B200_PROFILING.md's
    figures.  The XKNN_PREC_FP32 GEMMs' peaks derive from the bf16 one (fp32_gemm_peaks)."""
    out = {"hbm": 6650.0, "bf16_burst": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        out.update(hbm=p["hbm_gbs"], bf16_burst=p["bf16_tflops"],
                   bf16_sus=p["bf16_tflops_sustained"], src="MEASURED_PEAKS.json")
    except Exception:
        pass
    return out


FP32_GEMM = os.environ.get("XKNN_FP32_GEMM", "mixed")  # the library reads the same variable


def fp32_gemm_peaks(bf16_peak):
    """fp32-accuracy peaks (TF/s of fp32 flops) of the XKNN_PREC_FP32 GEMMs, from the tensor-pipe
    time each fp32 product costs with the arithmetic the library uses (fast32.cu), a kind::tf32
    MMA taking twice a kind::f16 one (dense TF32 = bf16 / 2, as B200_PROFILING.md's 1.1 vs 2.25
    PF/s; this repo's 3xTF32 GEMM-dX measured 835 TF/s of TF32 MMAs against bf16 / 2 = 832):
      mixed GEMM-F: one tf32 + two bf16 MMAs = 4 bf16-MMA times  -> bf16 / 4
      bf16x3 GEMM-dW / dX: three bf16 MMAs                        -> bf16 / 3
      3xTF32: three tf32 MMAs = 6 bf16-MMA times                  -> bf16 / 6"""
    f = {"mixed": 4.0, "f3": 6.0, "3xtf32": 6.0}.get(FP32_GEMM, 4.0)
    bw = 6.0 if FP32_GEMM == "3xtf32" else 3.0
    return {"gemm_logits_softmax": bf16_peak / f, "gemm_dW": bf16_peak / bw,
            "gemm_dX": bf16_peak / bw}


FP32_GEMM_SRC = ("MEASURED_PEAKS bf16 / (bf16-MMA times per fp32 product: mixed GEMM-F 4, "
                 "bf16x3 GEMM-dW/dX 3, 3xTF32 6; bench.fp32_gemm_peaks)")


def kernel_rooflines(phase_ms, precision, b, mw, splits, pk, burst):
    """Per-phase roofline of one step (SURVEY 8(d) units, stated per launch).  GEMMs: 2*B*M_w*D
    algorithmic flops each; HBM kernels: their algorithmic bytes (the update: 16*M_w*D = W and
    velocity read + written in fp32 -- the dW row it also reads is not credited; the gather: the
    M_w fp32 rows read + their tensor-core operand copy written).  Peak: burst when the clocks
    sat at max with no throttle reason, else sustained."""
    f32 = precision != "bf16"
    bf16_peak = pk["bf16_burst"] if burst else pk["bf16_sus"]
    tpeak = fp32_gemm_peaks(bf16_peak) if f32 else {}
    # bytes per element of the tensor-core operand copies written by the gather (W_sub) and the
    # fixup (X_hat'): bf16 | mixed: tf32 + 3 bf16 planes, bf16x3 planes | f3: hi + lo + 2 planes,
    # planes | 3xTF32: hi + lo, hi + lo
    opb, opx = {"mixed": (10, 4), "f3": (12, 4), "3xtf32": (8, 8)}.get(FP32_GEMM, (10, 4)) \
        if f32 else (2, 2)
    gemm = 2.0 * b * mw * D
    work = {
        "gemm_logits_softmax": ("tensor", gemm),
        "gemm_dW": ("tensor", gemm),
        "gemm_dX": ("tensor", gemm),
        "update": ("hbm", 16.0 * mw * D),
        "gather_normalize": ("hbm", (4.0 + opb) * mw * D + (4.0 + opb) * b * D),
        "softmax_stats": ("hbm", 2.0 * math.ceil(mw / 256) * b * 4 + (4.0 + opx) * b * D),
        "dX_reduce_scatter": ("hbm", (splits + 1) * 4.0 * b * D),
        "feature_backward": ("hbm", 3 * 4.0 * b * D),
    }
    rows, floor_ms = {}, 0.0
    for name, (bound, w) in work.items():
        ms = phase_ms.get(name)
        if not ms:
            continue
        if bound == "tensor":
            ach, peak, unit = w / (ms / 1e3) / 1e12, tpeak.get(name, bf16_peak), "TFLOP/s"
        else:
            ach, peak, unit = w / (ms / 1e3) / 1e9, pk["hbm"], "GB/s"
        floor_ms += (w / (peak * (1e12 if bound == "tensor" else 1e9))) * 1e3
        rows[name] = {"bound": bound, "ms": round(ms, 4), "work": w, "achieved": round(ach, 2),
                      "peak": round(peak, 1), "unit": unit, "frac": round(ach / peak, 4)}
    return rows, floor_ms


# ----------------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~10 ms in a thread."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.mask = 0
        self.maxclk = None
        self._stop = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.maxclk = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    self.mask |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    pass
                self._stop.wait(0.01)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.maxclk, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.maxclk,
                "reasons": sorted(k for k, v in self.REASONS.items() if self.mask & v),
                "samples": len(self.samples), "source": "nvml, 10 ms"}


# ----------------------------------------------------------------------------------------------
# synthetic inputs
# ----------------------------------------------------------------------------------------------
def install_shard_graph(torch, layer, n, k, p, rank, seed=7, chunk=1 << 20):
    """This shard's CompressedKnnGraph (compress_graph, knn_graph.cpp:235-266) of a seeded
    self-first random k-graph, generated chunk-wise on device identically on every rank and
    written straight into the layer's own graph arrays (xknn_layer_graph_buffers): a counting
    pass sizes the shard's entries, a second pass regenerates the chunks and fills them -- no
    staging copy (C4: ~10 GB of entries per GPU next to a 100 GB weight+velocity shard)."""
    import paper_2102_06025_b200 as X

    lo, hi = X.ShardLayout(n, p).class_range(rank)
    g = torch.Generator(device="cuda")

    def chunks():
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            g.manual_seed(seed * 1_000_003 + c0)
            nb = torch.randint(0, n, (c1 - c0, k), device="cuda", dtype=torch.int32, generator=g)
            nb[:, 0] = torch.arange(c0, c1, device="cuda", dtype=torch.int32)
            yield c0, c1, nb, (nb >= lo) & (nb < hi)

    kpc = torch.empty(n, dtype=torch.int32, device="cuda")
    for c0, c1, nb, mask in chunks():
        kpc[c0:c1] = mask.sum(1, dtype=torch.int32)
    flat_len = int(kpc.sum(dtype=torch.int64).item())
    kb, ob, fb = layer.graph_buffers(flat_len)
    kb.copy_(kpc)
    del kpc
    ob.copy_(torch.cumsum(kb, 0, dtype=torch.int64))
    ob.sub_(kb.to(torch.int64))
    for c0, c1, nb, mask in chunks():
        vals = nb[mask]
        start = int(ob[c0].item())
        fb[start:start + vals.numel()] = vals
    torch.cuda.synchronize()
    layer.commit_graph()


def make_batches(torch, n, b_local, rank, count=4):
    g = torch.Generator(device="cuda")
    out = []
    for i in range(count):
        g.manual_seed(1000 + 31 * rank + i)
        x = torch.randn(b_local, D, device="cuda", generator=g)
        y = torch.randint(0, n, (b_local,), device="cuda", dtype=torch.int32, generator=g)
        out.append((x, y))
    return out


# ----------------------------------------------------------------------------------------------
# the reference (CPU) arm
# ----------------------------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_cpu(wl, steps, warmup, budget_s=150.0, workers=None, max_n=1_000_000):
    """The reference's stock HybridSim::train_step (kKnn) from oracle/_ref (compiled from the
    unmodified reference sources) at the workload's FULL global batch, with `workers` simulated
    workers (SimOptions::worker_threads: one thread each, the reference's only multi-core
    mechanism; default nproc; 1 = one core).  Falls back to the oracle port (1 thread).
    Bounded sample: the warm-up step (which also allocates the velocity) is timed first, and only
    as many of the requested steps are timed as fit budget_s (at least one)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O

    n_full, b, k = wl["n"], wl["b"], wl["k"]
    # beyond 1M classes the reference's step is O(N*D) host work per step (whole-shard
    # normalization, a dense N/P x D gradient block) and tens of GB of host RAM, minutes per step
    # at 10M: it is timed at max_n classes with the workload's batch and k (its per-sample cost
    # grows with N, so this overstates its rate there)
    n = min(n_full, max_n)
    m = max(1, int(math.ceil(0.1 * n)))
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(SEED)
    w = (rng.standard_normal((n, D), dtype=np.float32) * np.float32(0.05)).astype(np.float32)
    g = O.random_graph(n, k, 7)
    kind = "reference" if O.ref_available() else "port"
    p = (workers or cores) if kind == "reference" else 1
    while b % p:
        p -= 1
    shards = [O.compress(g, p, s_) for s_ in range(p)]
    del g

    def batch(i):
        r = np.random.default_rng(100 + i)
        return (r.standard_normal((b, D), dtype=np.float32),
                r.integers(0, n, b).astype(np.uint32))

    if kind == "reference":
        sim = O.RefSim(w, p, threads=p > 1, scale=SCALE, momentum=MOMENTUM)
        sim.set_graphs(shards)

        def one(i):
            x, y = batch(i)
            t = time.perf_counter()
            rc, loss, _ = sim.step(x, y, m, SEED, LR, reset_fe=False)
            assert rc == 0, rc
            return time.perf_counter() - t
    else:
        vel = np.zeros_like(w)

        def one(i):
            x, y = batch(i)
            t = time.perf_counter()
            rc, *_ = O.fc_train_step(w, vel, x, y, shards, m, SEED, SCALE, LR, MOMENTUM, 0.0)
            assert rc == 0, rc
            return time.perf_counter() - t

    t0 = one(0)  # warm-up 1 (allocates the velocity); always run
    t_start = time.perf_counter()
    done_warm = 1
    while done_warm < warmup and (time.perf_counter() - t_start) + t0 < budget_s / 3:
        t0 = one(done_warm)
        done_warm += 1
    n_timed = max(1, min(steps, int(budget_s / max(t0, 1e-3))))
    times = [one(100 + i) for i in range(n_timed)]
    med = float(np.median(times))
    return dict(value=b / med, unit="samples/s", cores=p if kind == "reference" else 1,
                kind=kind, steps_timed=n_timed, warmup_steps=done_warm, cpu_model=cpu_model(),
                nproc=cores,
                sample=(f"{'HybridSim::train_step(kKnn)' if kind == 'reference' else 'oracle port'}"
                        f" at N={n}" + (f" (bounded sample of the N={n_full} workload: the "
                                        f"reference's per-sample cost grows with N, so this "
                                        f"overstates its rate there)" if n < n_full else "") +
                        f", k={k}, M={m}, D={D}, full batch {b}, P={p} worker thread(s), median of "
                        f"{n_timed} step(s) after {done_warm} warm-up, {cores} host cores ("
                        f"{cpu_model()})"),
                ms_per_step=med * 1e3, config_n=n)


# ----------------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------------
def run_ours(args, wl_name, wl, rank, world, local_rank, dist, precision=None):
    import torch

    import paper_2102_06025_b200 as X

    torch.cuda.set_device(local_rank)
    n, b, k = wl["n"], wl["b"], wl["k"]
    m = max(1, int(math.ceil(0.1 * n)))
    b_local = b // world
    comm = None
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(X.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = X.nccl_comm_init(bytes(uid.cpu().numpy().tobytes()), world, rank)
    precision = precision or args.precision
    prec = {"bf16": X.PREC_BF16, "fp32": X.PREC_FP32, "fp32_exact": X.PREC_FP32_EXACT}[precision]
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        # per-shard active capacity: uniform labels put ~M/P active classes on each shard; the
        # worst-case default min(shard, M) would size P~ at B x M (164 GB per GPU at C4 on 4)
        cap = 0 if world == 1 else int(math.ceil(m / world * 1.05)) + 4096
        layer = X.KnnSoftmaxLayer(n, D, rank=rank, world=world, m_active=m, max_batch=b,
                                  scale=SCALE, momentum=MOMENTUM, rng_seed=SEED, precision=prec,
                                  comm=comm, stream=stream, active_capacity=cap)
        gw = torch.Generator(device="cuda")
        gw.manual_seed(10 + rank)
        wv = layer.weights_view().tensor
        for r0 in range(0, wv.shape[0], 1 << 20):
            wv[r0:r0 + (1 << 20)].normal_(0.0, 0.05, generator=gw)
        install_shard_graph(torch, layer, n, k, world, rank)
        batches = make_batches(torch, n, b_local, rank)
        gfeat = torch.empty(b_local, D, device="cuda")
        loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # every step hands the next batch's labels to xknn_prepare right after it is enqueued, so
    # the next selection overlaps this step's tail (a training loop knows its next batch)
    nb = len(batches)
    it = {"i": 0}

    def step(_i=None):
        i = it["i"]
        it["i"] = i + 1
        x, y = batches[i % nb]
        with torch.cuda.stream(stream):
            layer.train_step(x, y, LR, grad_features_local=gfeat, loss_out=loss, sync=False)
            layer.prepare(batches[(i + 1) % nb][1])

    with torch.cuda.stream(stream):
        layer.prepare(batches[0][1])
    for i in range(args.warmup):
        step(i)
    layer.sync()
    barrier()
    clk = ClockSampler(local_rank)
    clk.__enter__()  # NVML sampling during the timed region

    # ---- timed region (device time, CUDA events on the layer stream) ----
    layer_launch0 = layer.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    for i in range(args.steps):
        step(i)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    clk.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1)
    launches = layer.kernel_launches - layer_launch0

    # ---- phase-profiled pass: the same steps again with CUDA events recorded inside the step
    #      at its phase boundaries (the events split the step's programmatic-launch chains, so
    #      this pass is a little slower; it yields the per-kernel times, not the headline) ----
    import ctypes as C

    X.lib().xknn_layer_profile(layer.h, 1)
    step(0)  # the step graph is re-captured with the event nodes
    layer.sync()
    X.lib().xknn_layer_profile(layer.h, 1)  # reset the accumulators
    pv0, pv1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    pv0.record(stream)
    for i in range(args.steps):
        step(i)
    pv1.record(stream)
    pv1.synchronize()
    barrier()
    ms_prof = pv0.elapsed_time(pv1)
    ph = (C.c_double * len(PHASES))()
    nsteps = C.c_uint64()
    X.lib().xknn_layer_phase_ms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int,
                                            C.POINTER(C.c_uint64)]
    X.lib().xknn_layer_phase_ms(layer.h, ph, len(PHASES), C.byref(nsteps))
    X.lib().xknn_layer_profile(layer.h, 0)
    phase_ms = {PHASES[i]: ph[i] / max(nsteps.value, 1) for i in range(len(PHASES))
                if PHASES[i] != "-"}
    layer.sync()
    active_total, active_local = layer.last_active()
    loss_v = float(loss.item())

    # ---- e2e: host buffers through the public API, copies inside the timed region ----
    # A pipelined training loop: every step's features and labels are copied from pinned host
    # memory on a copy stream (overlapping the previous step), the step runs on the layer
    # stream, and every step's loss is copied back to pinned host memory; the loop is timed by
    # the host wall clock until the last loss has arrived.
    hx = [bt[0].cpu().pin_memory() for bt in batches]
    hy = [bt[1].cpu().pin_memory() for bt in batches]
    dxs = [torch.empty(b_local, D, device="cuda") for _ in range(2)]
    dys = [torch.empty(b_local, dtype=torch.int32, device="cuda") for _ in range(2)]
    # at least 200 steps: a training loop's steady state, not its one-time start-up (first copy,
    # first launch) -- ~0.1 s of work at C2
    e2e_steps = max(args.steps, args.e2e_steps)
    hloss = torch.zeros(e2e_steps, dtype=torch.float64).pin_memory()
    copy_stream = torch.cuda.Stream()
    ev_copied = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    i0 = it["i"]  # the pending prepare holds batch i0's labels

    def copy_in(j):
        s_, i = j % 2, i0 + j
        with torch.cuda.stream(copy_stream):
            if j >= 2:
                copy_stream.wait_event(ev_used[s_])  # step j-2 is done reading this buffer
            dxs[s_].copy_(hx[i % len(hx)], non_blocking=True)
            dys[s_].copy_(hy[i % len(hy)], non_blocking=True)
            ev_copied[s_].record(copy_stream)

    barrier()
    clk_e2e = ClockSampler(local_rank)
    clk_e2e.__enter__()
    t0 = time.perf_counter()
    copy_in(0)
    for j in range(e2e_steps):
        s_ = j % 2
        stream.wait_event(ev_copied[s_])
        with torch.cuda.stream(stream):
            # the caller reads every step's loss: written straight into pinned host memory
            layer.train_step(dxs[s_], dys[s_], LR, grad_features_local=gfeat,
                             loss_out=hloss[j:j + 1], sync=False)
            ev_used[s_].record(stream)
        if j + 1 < e2e_steps:
            copy_in(j + 1)
            with torch.cuda.stream(stream):
                layer.prepare(dys[(j + 1) % 2], ready_stream=copy_stream)
    e2e_enqueue_ms = (time.perf_counter() - t0) * 1e3  # host time to issue every step
    stream.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    clk_e2e.__exit__(None, None, None)
    barrier()
    layer.sync()
    assert np.isfinite(hloss.numpy()).all()

    # ---- max over ranks ----
    if world > 1:
        t = torch.tensor([ms, e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), float(t[1])
        tg = torch.tensor([float(active_local)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        mw_max = int(tg.item())
    else:
        mw_max = active_local
    # every rank's clocks and its own GEMM-F / softmax-statistics phases: at N > 1 the step is the
    # slowest rank's, and the others wait for it at the softmax all-reduce (softmax_stats)
    per_rank = None
    if world > 1:
        cs = clk.summary()
        mine = {"rank": rank, "sm_mhz": cs.get("sm_mhz"), "reasons": cs.get("reasons"),
                "active_rows": int(active_local),
                "gemm_logits_softmax_ms": round(phase_ms.get("gemm_logits_softmax", 0.0), 4),
                "softmax_stats_ms": round(phase_ms.get("softmax_stats", 0.0), 4)}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)

    res = None
    if rank == 0:
        ms_step = ms / args.steps
        value = b / (ms_step / 1e3)
        pk = peaks()
        clocks = clk.summary()
        # burst peaks when the SMs ran at their max clock with no throttle reason in the timed
        # region (a short run that never reached the power limit), else the sustained ones
        burst = (clocks.get("sm_mhz") is not None and clocks.get("sm_max_mhz") is not None and
                 clocks["sm_mhz"] >= 0.98 * clocks["sm_max_mhz"] and not clocks["reasons"])
        splits = max(1, -(-148 // max(1, -(-b // 256))))  # dX split-K ranges (upper bound)
        kern, floor_ms = kernel_rooflines(phase_ms, precision, b, active_local, splits, pk,
                                          burst)
        dom = max(kern, key=lambda k_: kern[k_]["ms"])
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r02", f"traffic_{wl_name}_{precision}.json")
        if world == 1 and os.path.exists(tp):  # captured on one GPU: per-rank shapes differ at N > 1
            try:
                traffic = json.load(open(tp)).get(dom)
            except Exception:
                traffic = None
        kd = kern[dom]
        roof = {"bound": kd["bound"], "kernel": dom, "achieved": kd["achieved"],
                "peak": kd["peak"], "unit": kd["unit"], "frac": kd["frac"], "traffic": traffic,
                "work_per_launch": kd["work"], "launch_ms": kd["ms"],
                "peak_source": (FP32_GEMM_SRC + (" burst" if burst else " sustained")
                                if precision != "bf16" and kd["bound"] == "tensor" else
                                pk["src"] + (" burst" if burst else " sustained")),
                "how": "work per launch / the kernel's CUDA-event time on the layer stream "
                       "(phase_ms, second pass); dominant = the longest phase"}
        # whole-step floors: every kernel at its own roofline, serialized (the step's kernels
        # run back to back), and the SURVEY 8(d) overlap bound max(flops/peak, bytes/peak)
        bpk = pk["bf16_burst"] if burst else pk["bf16_sus"]
        gp = fp32_gemm_peaks(bpk) if precision != "bf16" else {
            "gemm_logits_softmax": bpk, "gemm_dW": bpk, "gemm_dX": bpk}
        t_roof = max(sum(2.0 * b * mw_max * D / (v * 1e12) for v in gp.values()),
                     16.0 * mw_max * D / (pk["hbm"] * 1e9))
        res = {
            "metric": "KNN-softmax fwd+bwd+update samples/sec @100M classes d=512, 1/2/4/8 "
                      "B200 vs roofline",
            "value": round(value, 1),
            "unit": "samples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None,
            "dtype": "bf16" if precision == "bf16" else "f32",
            "precision": {"bf16": "bf16 operands, fp32 accumulation (stated bound, DESIGN.md 2)",
                          "fp32": {"mixed": "fp32 accuracy (1e-5 of the reference) on tensor cores: "
                                            "GEMM-F tf32 + 2 bf16 cross terms, GEMM-dW/dX bf16x3",
                                   "f3": "fp32 accuracy: GEMM-F 3xTF32, GEMM-dW/dX bf16x3",
                                   "3xtf32": "fp32 accuracy: 3xTF32 GEMMs"}.get(FP32_GEMM, FP32_GEMM),
                          "fp32_exact": "CUDA-core fp32 in the reference's summation order"}[
                              precision],
            "data": "synthetic (W~N(0,0.05^2), X~N(0,1), uniform labels, seeded random "
                    "self-first k-NN graph)",
            "config": {"workload": wl_name, "num_classes": n, "dim": D, "global_batch": b,
                       "k": k, "m_active": m, "active_per_shard": active_local,
                       "scale": SCALE, "parallelism": f"class-sharded mp{world}",
                       "l2": "per-step working set > 126 MB L2 (weight shard, P~ bf16)"},
            "e2e": {"value": round(b / (e2e_ms / e2e_steps / 1e3), 1), "unit": "samples/s",
                    "steps": e2e_steps,
                    "host_issue_ms_per_step": round(e2e_enqueue_ms / e2e_steps, 4),
                    "h2d_bytes_per_step": int(b_local * D * 4 + b_local * 4),
                    "d2h_bytes_per_step": 8,
                    "how": "host wall clock over a pipelined loop: per step H2D of the rank's "
                           "features+labels from pinned memory on a copy stream, the next step's "
                           "selection prepared as soon as its labels land, the step, D2H of its "
                           "loss",
                    "clocks": clk_e2e.summary()},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernels": kern,
            "step_roofline": {"t_floor_serial_ms": round(floor_ms, 4),
                              "frac_serial": round(floor_ms / ms_step, 4),
                              "t_roof_overlap_ms": round(t_roof * 1e3, 4),
                              "frac_overlap": round(t_roof * 1e3 / ms_step, 4),
                              "how": "serial: sum over the step's kernels of work/peak; overlap: "
                                     "max(sum over the 3 GEMMs of 2*B*M_w*D/its peak, "
                                     "16*M_w*D/HBM peak)"},
            "phase_ms": {k_: round(v, 4) for k_, v in phase_ms.items()},
            **({"per_rank": per_rank} if per_rank else {}),
            "phase_profile": {"ms_per_step": round(ms_prof / args.steps, 4), "steps": args.steps,
                              "how": "second pass of the same steps with CUDA events at the "
                                     "step's phase boundaries (last step's graph replay)"},
            "clocks": clocks,
            "loss": loss_v,
            "active_classes": int(active_total),
        }
        if world > 1:
            # N = 1 runs C2 (the largest single-GPU config, BASELINE configs[1]); this line's
            # workload also runs on one GPU, measured separately -- the base of its strong scaling
            ref1 = os.path.join(ROOT, "profiles", "r02", f"bench_{wl_name}_1gpu_{precision}.json")
            if os.path.exists(ref1):
                try:
                    d1 = json.load(open(ref1))
                    res["same_workload_1gpu"] = {
                        "value": d1["value"], "ms_per_step": d1["ms_per_step"],
                        "strong_scaling_efficiency": round(value / (world * d1["value"]), 4),
                        "source": f"profiles/r02/bench_{wl_name}_1gpu_{precision}.json "
                                  f"(bench.py --workload {wl_name}, one B200, another box)"}
                except (OSError, KeyError, ValueError):
                    pass
    layer.close()
    if comm is not None:
        X.nccl_comm_destroy(comm)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


_JSON_OUT = None


def emit(obj) -> None:
    """The one JSON line of this run, on the process's original stdout."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def main():
    # stdout carries exactly one JSON line: everything else written to fd 1 -- NCCL's version
    # banner, library logs, prints -- is sent to stderr; emit() writes to the saved stdout
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=200,
                    help="minimum number of steps of the e2e (host-buffer) loop")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="fp32", choices=["bf16", "fp32", "fp32_exact"],
                    help="headline arithmetic: fp32 = 3xTF32 tensor cores at the reference's "
                         "fp32 accuracy (default); bf16 = bf16 operands, stated bound")
    ap.add_argument("--no-bf16-line", action="store_true",
                    help="skip the secondary bf16 measurement (bf16_mode) of the default run")
    ap.add_argument("--bf16-pause", type=float, default=15.0,
                    help="seconds idle between the fp32 run and the bf16 line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # the same workload at every N (strong scaling over the class shards), so the per-N lines
    # compare like for like; C3 / C4 run with --workload (their lines are in profiles/r02/)
    wl_name = args.workload or "c2"
    wl = WORKLOADS[wl_name]

    if args.impl == "reference":
        if rank != 0:
            return
        r = reference_cpu(wl, args.steps, args.warmup)
        same = r["config_n"] == wl["n"]
        emit({
            "impl": "reference",
            "metric": "KNN-softmax fwd+bwd+update samples/sec @100M classes d=512, 1/2/4/8 "
                      "B200 vs roofline",
            "value": round(r["value"], 3), "unit": "samples/s", "n_gpus": world,
            "steps": r["steps_timed"], "steps_requested": args.steps,
            "warmup": r["warmup_steps"], "ms_per_step": round(r["ms_per_step"], 2),
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl_name, "num_classes": wl["n"], "dim": D,
                       "global_batch": wl["b"], "k": wl["k"]},
            "same_config": same,
            "cpu_baseline": {k_: r[k_] for k_ in ("value", "unit", "cores", "kind", "sample",
                                                  "cpu_model", "nproc")},
            "e2e": {"value": round(r["value"], 3), "unit": "samples/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        })
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, wl_name, wl, rank, world, local_rank, dist)
    if args.precision == "fp32" and not args.no_bf16_line:
        # the same workload in the bf16 tensor-core mode (stated bound), same
        # process, after a pause that lets the power limiter recover from the fp32 run
        time.sleep(args.bf16_pause)
        r16 = run_ours(args, wl_name, wl, rank, world, local_rank, dist, precision="bf16")
        if rank == 0:
            res["bf16_mode"] = {k_: r16[k_] for k_ in ("value", "unit", "ms_per_step", "dtype",
                                                       "precision", "e2e", "roofline", "kernels",
                                                       "step_roofline", "phase_ms", "clocks",
                                                       "gpu_launches")}
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline and wl_name in ("c1", "c2"):
            # the reference on all host cores (P = nproc worker threads) and on one
            # core (P = 1), full batch, median after a warm-up step
            try:
                r = reference_cpu(wl, 3, 1, budget_s=40.0)
                res["cpu_baseline"] = {k_: r[k_] for k_ in ("value", "unit", "cores", "kind",
                                                            "sample", "cpu_model", "nproc")}
                res["cpu_baseline"]["value"] = round(res["cpu_baseline"]["value"], 3)
                r1 = reference_cpu(WORKLOADS["c1"], 3, 1, budget_s=30.0, workers=1)
                res["cpu_baseline"]["single_core_c1"] = {
                    "value": round(r1["value"], 3), "unit": "samples/s", "cores": 1,
                    "sample": r1["sample"]}
            except Exception as e:  # the baseline is reported, never required
                res["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        else:
            res["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": 0,
                                   "kind": "reference",
                                   "sample": "not run: reference needs >80 GB host RAM and "
                                             "~10 min/step beyond c2 (SURVEY 7.7)"}
        emit(res)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
