"""B200-native (sm_100a) model-parallel KNN-softmax layer -- Python host binding.

Mirrors the reference's C++ layer API (namespace ``xcls``, /root/reference/proj/include/xcls)
for the fc hot path over the C ABI in ``include/xknn.h`` (``libxknn.so``, built in-tree by
``make -C paper_2102_06025_b200``).  PyTorch is used only for device memory and streams.

There is no CPU fallback: importing this package without the built CUDA library raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libxknn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library with `make -C {_HERE}` "
        "(there is no CPU fallback)")

import torch as _torch  # noqa: F401  (plumbing; loads the NCCL build torch was linked against first)

_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

U64 = C.c_uint64
VP = C.c_void_p

PREC_BF16 = 0
PREC_FP32_EXACT = 1
PREC_FP32 = 2  # tensor cores at fp32 accuracy (split operands; include/xknn.h)
FLAG_NO_GRAPH = 1
FLAG_SELECT_ONLY = 2


class XknnConfig(C.Structure):
    """xknn_config_t (include/xknn.h) == SimOptions + SelectionConfig of the reference."""
    _fields_ = [("scale", C.c_float), ("momentum", C.c_float), ("weight_decay", C.c_float),
                ("m_active", U64), ("rng_seed", U64), ("max_batch", U64),
                ("precision", C.c_int32), ("flags", C.c_int32), ("active_capacity", U64)]


# ---- errors.hpp:10-54 -------------------------------------------------------------------------
class Error(RuntimeError):
    code = -1


class ShapeMismatch(Error): code = 1
class ZeroNormRow(Error):
    code = 2

    def __init__(self, msg, row=0):
        super().__init__(msg)
        self.row = row
class LabelOutOfRange(Error): code = 3
class KTooLarge(Error): code = 4
class EmptyShard(Error): code = 5
class MTooSmall(Error): code = 6
class LabelNotActive(Error): code = 7
class InvalidArgument(Error): code = 8
class IoError(Error): code = 9
class ConfigError(Error): code = 10
class CudaError(Error): code = 20
class NcclError(Error): code = 21
class OutOfMemory(Error): code = 22
class Unsupported(Error): code = 23


_ERRS = {c.code: c for c in (ShapeMismatch, ZeroNormRow, LabelOutOfRange, KTooLarge, EmptyShard,
                             MTooSmall, LabelNotActive, InvalidArgument, IoError, ConfigError,
                             CudaError, NcclError, OutOfMemory, Unsupported)}

_lib.xknn_last_error_message.restype = C.c_char_p
_lib.xknn_last_error_row.restype = U64
_lib.xknn_layer_kernel_launches.restype = U64
_lib.xknn_layer_kernel_launches.argtypes = [VP]


def _check(rc: int) -> None:
    if rc == 0:
        return
    cls = _ERRS.get(rc, Error)
    msg = _lib.xknn_last_error_message().decode()
    if cls is ZeroNormRow:
        raise ZeroNormRow(msg, int(_lib.xknn_last_error_row()))
    raise cls(msg)


for _name, _args in {
    "xknn_shard_range": [U64, U64, U64, C.POINTER(U64), C.POINTER(U64)],
    "xknn_nccl_unique_id": [C.c_char_p],
    "xknn_nccl_comm_init": [C.c_char_p, C.c_int, C.c_int, C.POINTER(VP)],
    "xknn_nccl_comm_destroy": [VP],
    "xknn_layer_create": [C.c_int, C.c_int, U64, U64, C.POINTER(XknnConfig), VP, VP, C.POINTER(VP)],
    "xknn_layer_destroy": [VP],
    "xknn_layer_shard": [VP, C.POINTER(U64), C.POINTER(U64)],
    "xknn_layer_set_config": [VP, C.POINTER(XknnConfig)],
    "xknn_layer_set_weights": [VP, VP, C.c_int],
    "xknn_layer_get_weights": [VP, VP, C.c_int],
    "xknn_layer_get_velocity": [VP, VP, C.c_int],
    "xknn_layer_weights_ptr": [VP, C.POINTER(VP)],
    "xknn_layer_set_graph_csr": [VP, VP, VP, VP, U64, C.c_int],
    "xknn_layer_set_graph_csr_ranked": [VP, VP, VP, VP, VP, U64, C.c_int],
    "xknn_layer_graph_buffers": [VP, U64, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)],
    "xknn_layer_graph_commit": [VP],
    "xknn_select_full_graph": [VP, U64, C.c_uint32, VP, U64, U64, U64, VP, C.POINTER(U64),
                               C.POINTER(C.c_int), VP],
    "xknn_knn_softmax_fwd_bwd": [VP, U64, VP, U64, U64, VP, VP, U64, C.c_float,
                                 C.POINTER(C.c_double), VP, VP, VP, VP],
    "xknn_select": [VP, VP, U64, VP, C.POINTER(U64), C.POINTER(C.c_int)],
    "xknn_step": [VP, VP, VP, U64, C.c_float, VP, VP],
    "xknn_step_micro": [VP, VP, VP, U64, C.c_float, C.c_uint32, VP, VP],
    "xknn_prepare": [VP, VP, U64, VP],
    "xknn_layer_sync": [VP],
    "xknn_layer_set_draw_stream": [VP, VP, U64],
    "xknn_layer_last_active": [VP, C.POINTER(U64), C.POINTER(U64)],
    "xknn_layer_last_logits": [VP, VP, U64],
    "xknn_graph_bruteforce": [VP, U64, U64, C.c_uint32, C.c_uint32, VP, VP, C.POINTER(U64)],
    "xknn_graph_release_cache": [],
    "xknn_graph_ring": [VP, U64, U64, C.c_uint32, C.c_uint32, C.c_int, C.c_int, VP, VP, VP,
                        C.POINTER(U64), C.POINTER(U64)],
    "xknn_layer_set_graph_rows": [VP, VP, C.c_uint32],
    "xknn_layer_rebuild_graph": [VP, C.c_uint32, C.c_uint32, VP, C.POINTER(U64)],
    "xknn_graph_save_rows": [C.c_char_p, U64, C.c_uint32, U64, U64, VP, C.c_int, C.c_int],
    "xknn_graph_load_rows": [C.c_char_p, U64, U64, U64, VP, U64, C.c_int,
                             C.POINTER(C.c_uint32)],
    "xknn_layer_get_graph": [VP, VP, VP, VP, U64, C.POINTER(U64), C.c_int],
    "xknn_layer_classify": [VP, VP, U64, VP, VP],
    "xknn_topk": [VP, U64, U64, VP, VP, VP],
    "xknn_dgc_create": [C.c_double, C.c_float, VP, C.POINTER(VP)],
    "xknn_dgc_set_sparsity": [VP, C.c_double],
    "xknn_dgc_compress": [VP, C.c_uint32, VP, U64, VP, VP, C.POINTER(U64)],
    "xknn_dgc_state": [VP, C.c_uint32, VP, VP, U64],
    "xknn_dgc_destroy": [VP],
}.items():
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = C.c_int


def lib() -> C.CDLL:
    return _lib


# ---- ShardLayout (knn_graph.hpp:30-41) -------------------------------------------------------
class ShardLayout:
    def __init__(self, num_classes: int, num_shards: int = 1):
        self.num_classes = num_classes
        self.num_shards = num_shards

    def class_range(self, shard: int) -> tuple[int, int]:
        b, e = U64(), U64()
        _check(_lib.xknn_shard_range(self.num_classes, self.num_shards, shard, C.byref(b),
                                     C.byref(e)))
        return b.value, e.value

    def shard_size(self, shard: int) -> int:
        b, e = self.class_range(shard)
        return e - b

    def shard_of(self, cls: int) -> int:
        base, rem = divmod(self.num_classes, self.num_shards)
        big = rem * (base + 1)
        return cls // (base + 1) if cls < big else rem + (cls - big) // base


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.xknn_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_init(uid: bytes, world: int, rank: int) -> int:
    comm = VP()
    _check(_lib.xknn_nccl_comm_init(uid, world, rank, C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm) -> None:
    _check(_lib.xknn_nccl_comm_destroy(comm))


def graph_bruteforce(w_norm, k: int, kprime: int = 0):
    """build_graph_bruteforce(w_norm, k) (knn_graph.cpp:124-145) on device, bit-exact.
    w_norm: (N, D) fp32 CUDA tensor of unit rows.  Returns ((N, k) int32 tensor, uncertified)."""
    import torch

    w = w_norm.contiguous()
    n, d = w.shape
    out = torch.empty(n, k, dtype=torch.int32, device=w.device)
    unc = U64()
    _check(_lib.xknn_graph_bruteforce(w.data_ptr(), n, d, k, kprime, out.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream, C.byref(unc)))
    return out, unc.value


def graph_ring(w_norm_local, num_classes: int, k: int, kprime: int, rank: int, world: int,
               comm=None):
    """build_graph_ring (knn_graph.cpp:147-233) with one process per GPU: this rank's normalized
    block of ShardLayout(num_classes, world) in, its rows of the exact graph out.  Collective.
    Returns ((rows, k) int32 tensor of global ids, uncertified rows, transfer steps)."""
    import torch

    w = w_norm_local.contiguous()
    rows, d = w.shape
    out = torch.empty(rows, k, dtype=torch.int32, device=w.device)
    unc, steps = U64(), U64()
    _check(_lib.xknn_graph_ring(w.data_ptr(), num_classes, d, k, kprime, rank, world, comm,
                                torch.cuda.current_stream().cuda_stream, out.data_ptr(),
                                C.byref(unc), C.byref(steps)))
    return out, unc.value, steps.value


def select_active_classes_full(graph, labels, m_active: int, seed: int):
    """select_active_classes(const KnnGraph&, labels, {m_active, seed}, N)
    (knn_softmax.cpp:100-115): graph is the uncompressed (N, k) int32/uint32 CUDA tensor; ranks
    are positions in the full lists.  Returns (sorted active classes int32 tensor,
    contains_all_labels)."""
    import torch

    g = graph.contiguous()
    n, k = g.shape
    lab = labels.to(torch.int32).contiguous()
    out = torch.empty(max(m_active, 1), dtype=torch.int32, device=g.device)
    cnt, ca = U64(), C.c_int()
    _check(_lib.xknn_select_full_graph(g.data_ptr(), n, k, lab.data_ptr(), lab.numel(), m_active,
                                       seed, out.data_ptr(), C.byref(cnt), C.byref(ca),
                                       torch.cuda.current_stream().cuda_stream))
    return out[: cnt.value], bool(ca.value)


def knn_softmax_forward_backward(x_norm, w_norm, labels, active, scale: float):
    """knn_softmax_forward_backward(x_norm, w_norm, labels, active, scale)
    (knn_softmax.cpp:136-186) on device (fp32, the reference's summation order).  Returns
    (loss, grad_logits (B, M), grad_features (B, D), grad_w_active (M, D) -- the active rows of
    the reference's dense grad_weights, zero elsewhere)."""
    import torch

    x = x_norm.contiguous()
    w = w_norm.contiguous()
    lab = labels.to(torch.int32).contiguous()
    act = active.to(torch.int32).contiguous()
    b, d = x.shape
    m = act.numel()
    gl = torch.empty(b, max(m, 1), device=x.device)
    gf = torch.empty(b, d, device=x.device)
    gw = torch.empty(max(m, 1), d, device=x.device)
    loss = C.c_double()
    _check(_lib.xknn_knn_softmax_fwd_bwd(x.data_ptr(), b, w.data_ptr(), w.shape[0], d,
                                         lab.data_ptr(), act.data_ptr(), m, float(scale),
                                         C.byref(loss), gl.data_ptr(), gf.data_ptr(),
                                         gw.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return loss.value, gl[:, :m], gf, gw[:m]


def release_graph_cache() -> None:
    """Return the graph builds' cached device scratch to the driver (xknn_graph_release_cache)."""
    _check(_lib.xknn_graph_release_cache())


def save_graph_rows(path: str, num_classes: int, begin: int, rows, create: bool) -> None:
    """save_graph (knn_graph.cpp:276-291) of classes [begin, begin + len(rows)): rows is a
    (n, k) uint32/int32 numpy array or CUDA tensor.  create: write the header (first writer)."""
    if hasattr(rows, "is_cuda") and rows.is_cuda:
        r = rows.contiguous()
        n, k = r.shape
        ptr, dev = r.data_ptr(), 1
    else:
        r = np.ascontiguousarray(rows).view(np.uint32)
        n, k = r.shape
        ptr, dev = r.ctypes.data, 0
    _check(_lib.xknn_graph_save_rows(path.encode(), num_classes, k, begin, begin + n, ptr, dev,
                                     int(create)))


def load_graph_rows(path: str, num_classes: int, begin: int = 0, end: int | None = None):
    """load_graph (knn_graph.cpp:293-311) of classes [begin, end): returns (k, rows u32 numpy)."""
    end = num_classes if end is None else end
    k = C.c_uint32()
    _check(_lib.xknn_graph_load_rows(path.encode(), num_classes, begin, end, None, 0, 0,
                                     C.byref(k)))
    rows = np.zeros((end - begin, k.value), np.uint32)
    _check(_lib.xknn_graph_load_rows(path.encode(), num_classes, begin, end, rows.ctypes.data,
                                     rows.size, 0, C.byref(k)))
    return k.value, rows


_lib.xknn_dgc_selected_count.restype = U64
_lib.xknn_dgc_selected_count.argtypes = [C.c_double, U64]


def selected_count(sparsity_ratio: float, length: int) -> int:
    """selected_count (sparsify.cpp:98-103)."""
    return int(_lib.xknn_dgc_selected_count(sparsity_ratio, length))


def topk(values, k: int):
    """topk_divide_conquer (sparsify.cpp:41-80) on device: (indices int64, values) of the k
    largest |values| (ties to the lower index) in selection order."""
    import torch

    t = values.contiguous()
    idx = torch.empty(k, dtype=torch.int64, device=t.device)
    val = torch.empty(k, dtype=torch.float32, device=t.device)
    _check(_lib.xknn_topk(t.data_ptr(), t.numel(), k, idx.data_ptr(), val.data_ptr(),
                          torch.cuda.current_stream().cuda_stream))
    return idx, val


class CompressionState:
    """CompressionState (sparsify.hpp:46-75): momentum-corrected top-k with residual
    accumulation and factor masking, state in HBM."""

    def __init__(self, sparsity_ratio: float, momentum: float):
        import torch

        self._torch = torch
        h = VP()
        _check(_lib.xknn_dgc_create(sparsity_ratio, momentum,
                                    torch.cuda.current_stream().cuda_stream, C.byref(h)))
        self.h = h.value
        self._len = {}

    def set_sparsity_ratio(self, r: float) -> None:
        _check(_lib.xknn_dgc_set_sparsity(self.h, r))

    def compress_step(self, layer_id: int, grad):
        """-> (indices int64 increasing, values) of the emitted entries."""
        torch = self._torch
        g = grad.contiguous()
        n = g.numel()
        cap = max(n, 1)
        idx = torch.empty(cap, dtype=torch.int64, device=g.device)
        val = torch.empty(cap, dtype=torch.float32, device=g.device)
        cnt = U64()
        torch.cuda.current_stream().synchronize()
        _check(_lib.xknn_dgc_compress(self.h, layer_id, g.data_ptr(), n, idx.data_ptr(),
                                      val.data_ptr(), C.byref(cnt)))
        self._len[layer_id] = n
        return idx[: cnt.value], val[: cnt.value]

    def state(self, layer_id: int, length: int):
        """(residual, velocity) of a layer."""
        torch = self._torch
        r = torch.empty(length, dtype=torch.float32, device="cuda")
        v = torch.empty(length, dtype=torch.float32, device="cuda")
        _check(_lib.xknn_dgc_state(self.h, layer_id, r.data_ptr(), v.data_ptr(), length))
        return r, v

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.xknn_dgc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


class KnnSoftmaxLayer:
    """One GPU's shard of the model-parallel KNN-softmax fc layer.

    The composite HybridSim fc half (parallel.cpp:433-677) restricted to one worker: owns the
    weight shard, the SgdMomentum velocity and the shard's CompressedKnnGraph on device.
    All tensor arguments are torch CUDA tensors on this layer's device.
    """

    def __init__(self, num_classes: int, dim: int, *, rank: int = 0, world: int = 1,
                 m_active: int, max_batch: int, scale: float = 30.0, momentum: float = 0.9,
                 weight_decay: float = 0.0, rng_seed: int = 0, precision: int = PREC_BF16,
                 comm=None, stream=None, use_graph: bool = True, select_only: bool = False,
                 active_capacity: int = 0):
        import torch  # plumbing only: device memory and streams

        self._torch = torch
        self.num_classes, self.dim, self.rank, self.world = num_classes, dim, rank, world
        self.cfg = XknnConfig(scale, momentum, weight_decay, m_active, rng_seed, max_batch,
                              precision, (0 if use_graph else FLAG_NO_GRAPH) |
                              (FLAG_SELECT_ONLY if select_only else 0), active_capacity)
        # the layer works on its own stream (capturable into a CUDA graph); every call is
        # ordered after the caller's current stream and the caller's stream after it
        self.stream = stream if stream is not None else torch.cuda.Stream()
        h = VP()
        _check(_lib.xknn_layer_create(rank, world, num_classes, dim, C.byref(self.cfg),
                                      comm, self.stream.cuda_stream, C.byref(h)))
        self.h = h.value
        b, e = U64(), U64()
        _check(_lib.xknn_layer_shard(self.h, C.byref(b), C.byref(e)))
        self.begin, self.end = b.value, e.value
        self._loss = torch.zeros(1, dtype=torch.float64, device="cuda")

    def _enter(self):
        cur = self._torch.cuda.current_stream()
        if cur != self.stream:
            self.stream.wait_stream(cur)

    def _leave(self):
        cur = self._torch.cuda.current_stream()
        if cur != self.stream:
            cur.wait_stream(self.stream)

    # -- state ----------------------------------------------------------------------------------
    @property
    def shard_rows(self) -> int:
        return self.end - self.begin

    def set_weights(self, w) -> None:
        """HybridSim::load_model for this shard: w is (shard_rows, dim) fp32."""
        assert w.shape == (self.shard_rows, self.dim) and w.dtype == self._torch.float32
        w = w.contiguous()
        self._enter()
        _check(_lib.xknn_layer_set_weights(self.h, w.data_ptr(), int(w.is_cuda)))

    def weights(self):
        out = self._torch.empty(self.shard_rows, self.dim, dtype=self._torch.float32,
                                device="cuda")
        self._enter()
        _check(_lib.xknn_layer_get_weights(self.h, out.data_ptr(), 1))
        self._leave()
        return out

    def velocity(self):
        out = self._torch.empty(self.shard_rows, self.dim, dtype=self._torch.float32,
                                device="cuda")
        self._enter()
        _check(_lib.xknn_layer_get_velocity(self.h, out.data_ptr(), 1))
        self._leave()
        return out

    def weights_view(self):
        """The resident weight shard as a torch tensor aliasing device memory (in-place init)."""
        p = VP()
        _check(_lib.xknn_layer_weights_ptr(self.h, C.byref(p)))
        return _DeviceView(p.value, (self.shard_rows, self.dim), self._torch)

    def set_shard_graph(self, k_per_class, offsets, flat) -> None:
        """HybridSim::set_shard_graphs for this shard (knn_graph.hpp:46-55 arrays)."""
        dev = int(k_per_class.is_cuda)
        kpc = k_per_class.contiguous()
        off = offsets.contiguous()
        fl = flat.contiguous()
        self._enter()
        _check(_lib.xknn_layer_set_graph_csr(self.h, kpc.data_ptr(), off.data_ptr(),
                                             fl.data_ptr() if fl.numel() else 0, fl.numel(), dev))

    def graph_buffers(self, flat_len: int):
        """In-place graph install: the layer-owned (k_per_class int32[N], offsets int64[N],
        flat int32[flat_len]) device arrays as torch tensors; fill them, synchronize, then
        commit_graph()."""
        torch = self._torch
        k, o, f = VP(), VP(), VP()
        self._enter()
        _check(_lib.xknn_layer_graph_buffers(self.h, flat_len, C.byref(k), C.byref(o), C.byref(f)))

        def view(ptr, n, typestr, dtype):
            class _V:
                __cuda_array_interface__ = {"data": (ptr, False), "shape": (n,),
                                            "typestr": typestr, "version": 2}
            return torch.as_tensor(_V(), device="cuda").view(dtype)

        return (view(k.value, self.num_classes, "<i4", torch.int32),
                view(o.value, self.num_classes, "<i8", torch.int64),
                view(f.value, max(flat_len, 1), "<i4", torch.int32)[:flat_len])

    def commit_graph(self) -> None:
        """Validate and install the arrays filled through graph_buffers (collective)."""
        self._enter()
        _check(_lib.xknn_layer_graph_commit(self.h))

    def set_shard_graph_ranked(self, k_per_class, offsets, flat, rank) -> None:
        """set_shard_graph with a per-entry rank (several shards' slices of a label merged into
        one list, each entry ranked within its own slice): xknn_layer_set_graph_csr_ranked."""
        dev = int(k_per_class.is_cuda)
        kpc, off, fl, rk = (t.contiguous() for t in (k_per_class, offsets, flat, rank))
        self._enter()
        _check(_lib.xknn_layer_set_graph_csr_ranked(self.h, kpc.data_ptr(), off.data_ptr(),
                                                    fl.data_ptr() if fl.numel() else 0,
                                                    rk.data_ptr() if rk.numel() else 0,
                                                    fl.numel(), dev))

    def set_graph_rows(self, rows, k: int) -> None:
        """compress_graph + set_shard_graphs from this rank's rows [begin, end) x k of the full
        graph (device int32/uint32, global ids).  Collective over the layer's ranks."""
        r = rows.contiguous()
        assert r.shape == (self.shard_rows, k) and r.is_cuda
        self._enter()
        _check(_lib.xknn_layer_set_graph_rows(self.h, r.data_ptr(), k))

    def rebuild_graph(self, k: int, kprime: int = 0, rows_out=None) -> int:
        """Exact KNN graph of the current (normalized) weights, sharded build + compression,
        installed as this shard's CompressedKnnGraph.  rows_out: optional (shard_rows, k) int32
        CUDA tensor receiving this rank's rows of the full graph.  Collective.  Returns the
        number of uncertified (exactly rescanned) rows."""
        unc = U64()
        self._enter()
        _check(_lib.xknn_layer_rebuild_graph(self.h, k, kprime, _ptr(rows_out), C.byref(unc)))
        self._leave()
        return unc.value

    def load_graph(self, path: str) -> int:
        """load_graph + compress_graph + set_shard_graphs from an XKNN file: this rank reads its
        rows [begin, end) and the shards exchange entries.  Collective.  Returns k."""
        k, rows = load_graph_rows(path, self.num_classes, self.begin, self.end)
        import torch

        self.set_graph_rows(torch.from_numpy(rows.view(np.int32)).cuda(), k)
        return k

    def graph(self):
        """The installed CompressedKnnGraph: (k_per_class u32[N], offsets u64[N], flat u32[])
        as numpy arrays."""
        import numpy as np

        n = U64()
        _check(_lib.xknn_layer_get_graph(self.h, None, None, None, 0, C.byref(n), 0))
        kpc = np.zeros(self.num_classes, np.uint32)
        off = np.zeros(self.num_classes, np.uint64)
        flat = np.zeros(max(n.value, 1), np.uint32)
        _check(_lib.xknn_layer_get_graph(self.h, kpc.ctypes.data, off.ctypes.data,
                                         flat.ctypes.data, flat.size, C.byref(n), 0))
        return kpc, off, flat[: n.value]

    def classify(self, queries):
        """classify_retrieval: nearest normalized class embedding of each query
        (n, dim) fp32 CUDA tensor.  Collective.  Returns (classes int32 tensor, cosines)."""
        torch = self._torch
        q = queries.contiguous()
        cls = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
        sc = torch.empty(q.shape[0], dtype=torch.float32, device="cuda")
        self._enter()
        _check(_lib.xknn_layer_classify(self.h, q.data_ptr(), q.shape[0], cls.data_ptr(),
                                        sc.data_ptr()))
        self._leave()
        return cls, sc

    # -- hot path ------------------------------------------------------------------------------
    def select_active_classes(self, labels):
        """This shard's slice of select_active_classes(span<CompressedKnnGraph>, ...)."""
        torch = self._torch
        cap = min(self.shard_rows, int(self.cfg.m_active)) + 32
        out = torch.empty(cap, dtype=torch.int32, device="cuda")
        cnt = U64()
        ca = C.c_int()
        lab = labels.to(torch.int32).contiguous()
        self._enter()
        _check(_lib.xknn_select(self.h, lab.data_ptr(), lab.numel(), out.data_ptr(), C.byref(cnt),
                                C.byref(ca)))
        self._leave()
        return out[: cnt.value].clone(), bool(ca.value)

    def prepare(self, labels_local, ready_stream=None) -> None:
        """Start the next train_step's selection now, overlapping the step in flight (the next
        train_step must get the same labels).  ready_stream: the torch stream on which
        labels_local becomes valid (None: it already is)."""
        torch = self._torch
        ready = ready_stream
        if labels_local.dtype != torch.int32 or not labels_local.is_contiguous():
            # converted on a stream of its own (not the current one, which may be the layer
            # stream with the step in flight: the selection must not wait for that), after the
            # labels are valid; the layer's side stream then waits for the converted buffer
            if getattr(self, "_conv_stream", None) is None:
                self._conv_stream = torch.cuda.Stream()
            conv = self._conv_stream
            conv.wait_stream(ready if ready is not None else torch.cuda.current_stream())
            with torch.cuda.stream(conv):
                lab = labels_local.to(torch.int32).contiguous()
            ready = conv
        else:
            lab = labels_local
        self._prep_keep = lab  # the buffer must outlive the asynchronous all-gather / copy
        _check(_lib.xknn_prepare(self.h, lab.data_ptr(), lab.numel(),
                                 ready.cuda_stream if ready is not None else None))

    def train_step(self, features_local, labels_local, lr: float, grad_features_local=None,
                   loss_out=None, sync: bool = True, micro_batches: int = 1):
        """The fc half of HybridSim::train_step (kKnn) for this rank's rows, with
        StepOptions::micro_batches = micro_batches (xknn_step_micro: grad_features rows of
        micro-batch c are the reference's micro-scaled mlp_backward input).
        Returns the mean loss (float) when sync, else None (loss in loss_out/self._loss)."""
        torch = self._torch
        assert features_local.dtype == torch.float32 and features_local.is_contiguous()
        lab = labels_local if labels_local.dtype == torch.int32 else labels_local.to(torch.int32)
        loss = self._loss if loss_out is None else loss_out
        self._enter()
        if micro_batches == 1:
            _check(_lib.xknn_step(self.h, features_local.data_ptr(), lab.data_ptr(),
                                  features_local.shape[0], float(lr), loss.data_ptr(),
                                  _ptr(grad_features_local)))
        else:
            _check(_lib.xknn_step_micro(self.h, features_local.data_ptr(), lab.data_ptr(),
                                        features_local.shape[0], float(lr), int(micro_batches),
                                        loss.data_ptr(), _ptr(grad_features_local)))
        self._leave()
        if sync:
            _check(_lib.xknn_layer_sync(self.h))
            return float(loss.item())
        return None

    def set_draw_stream(self, words=None) -> None:
        """Replace the padding draw's mt19937_64(rng_seed) word stream with `words` (uint64
        numpy array, >= m_active words), or restore it (None): xknn_layer_set_draw_stream."""
        if words is None:
            _check(_lib.xknn_layer_set_draw_stream(self.h, None, 0))
            return
        w = np.ascontiguousarray(words, dtype=np.uint64)
        self._enter()
        _check(_lib.xknn_layer_set_draw_stream(self.h, w.ctypes.data, w.size))

    def sync(self) -> None:
        _check(_lib.xknn_layer_sync(self.h))

    def last_active(self) -> tuple[int, int]:
        t, l = U64(), U64()
        _check(_lib.xknn_layer_last_active(self.h, C.byref(t), C.byref(l)))
        return t.value, l.value

    def last_logits(self, batch: int):
        import numpy as np

        _, loc = self.last_active()
        out = np.zeros((batch, loc), np.float32)
        _check(_lib.xknn_layer_last_logits(self.h, out.ctypes.data, out.size))
        return out

    @property
    def kernel_launches(self) -> int:
        return int(_lib.xknn_layer_kernel_launches(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.xknn_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DeviceView:
    """Minimal __cuda_array_interface__ wrapper so torch.as_tensor can alias library memory."""

    def __init__(self, ptr, shape, torch):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": "<f4",
                                         "version": 2}
        self.tensor = torch.as_tensor(self, device="cuda")
