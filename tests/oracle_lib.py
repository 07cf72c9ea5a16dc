"""ctypes access to the CPU checker (oracle/liboracle.so) and, when built, the compiled
reference (oracle/_ref/libxcls_ref.so).  Test infrastructure only: the product package never
imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libxcls_ref.so")

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
U64 = C.c_uint64


def _ensure_oracle() -> None:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True,
                       capture_output=True)


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        _ensure_oracle()
        _oracle = C.CDLL(ORACLE_SO)
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_SO)
        _ref.ref_sim_create.restype = C.c_void_p
        _ref.ref_sim_create.argtypes = [U64, U64, U64, C.c_int, C.c_float, C.c_float, C.c_float,
                                        f32p]
        _ref.ref_sim_step.argtypes = [C.c_void_p, f32p, u32p, U64, U64, U64, C.c_float,
                                      C.POINTER(C.c_double), C.POINTER(U64)]
        _ref.ref_sim_step_mb.argtypes = [C.c_void_p, f32p, u32p, U64, U64, U64, C.c_float, U64,
                                         C.POINTER(C.c_double), C.POINTER(U64)]
        _ref.ref_sim_get_weights.argtypes = [C.c_void_p, f32p]
        _ref.ref_sim_destroy.argtypes = [C.c_void_p]
        _ref.ref_sim_set_graphs.argtypes = [C.c_void_p, U64, C.c_void_p, C.c_void_p, C.c_void_p]
    return _ref


# ----------------------------------------------------------------------------------------------
# Graph helpers
# ----------------------------------------------------------------------------------------------
def shard_range(n: int, p: int, s: int) -> tuple[int, int]:
    """ShardLayout::class_range, knn_graph.cpp:102-115."""
    base, rem = divmod(n, p)
    if s < rem:
        b = s * (base + 1)
        return b, b + base + 1
    b = rem * (base + 1) + (s - rem) * base
    return b, b + base


def random_graph(n: int, k: int, seed: int) -> np.ndarray:
    """Self-first KNN-shaped graph of distinct neighbours (N×k u32).  Random-init class
    weights make the true graph statistically random, SURVEY.md 8(d)."""
    rng = np.random.default_rng(seed)
    g = np.empty((n, k), dtype=np.uint32)
    g[:, 0] = np.arange(n, dtype=np.uint32)
    if k > 1:
        # distinct non-self neighbours; only rows with a collision are redrawn
        cand = rng.integers(0, n - 1, size=(n, k - 1), dtype=np.int64)
        cand += cand >= np.arange(n)[:, None]  # skip self
        srt = np.sort(cand, axis=1)
        bad = np.nonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))[0] if k > 2 else []
        for i in bad:
            others = rng.permutation(n - 1)[: k - 1]
            cand[i] = others + (others >= i)
        g[:, 1:] = cand
    return g


def compress(g: np.ndarray, p: int, s: int):
    """compress_graph via the oracle: (k_per_class u32[n], offsets u64[n], flat u32[total])."""
    n, k = g.shape
    kpc = np.zeros(n, np.uint32)
    off = np.zeros(n, np.uint64)
    flat = np.zeros(max(n * k, 1), np.uint32)
    lib = oracle()
    lib.or_compress_graph.restype = U64
    lib.or_compress_graph.argtypes = [U64, U64, u32p, U64, U64, u32p, u64p, u32p]
    tot = lib.or_compress_graph(n, k, np.ascontiguousarray(g), p, s, kpc, off, flat)
    return kpc, off, flat[:tot].copy()


def _ptr_array(arrs, ctype):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data_as(C.c_void_p) for a in arrs])


def select_shards(lib_kind: str, n: int, shards, labels: np.ndarray, m: int, seed: int):
    """select_active_classes(span<CompressedKnnGraph>) via oracle ('oracle') or ref ('ref')."""
    p = len(shards)
    kpcs = [s[0] for s in shards]
    offs = [s[1] for s in shards]
    flats = [s[2] if s[2].size else np.zeros(1, np.uint32) for s in shards]
    out = np.zeros(max(m, 1), np.uint32)
    cnt = U64(0)
    ca = C.c_int(0)
    labels = np.ascontiguousarray(labels, dtype=np.uint32)
    if lib_kind == "oracle":
        fn = oracle().or_select_active_shards
    else:
        fn = ref().ref_select_active_shards
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, C.c_void_p, C.c_void_p, C.c_void_p, u32p, U64, U64, U64, u32p,
                   C.POINTER(U64), C.POINTER(C.c_int)]
    rc = fn(n, p, _ptr_array(kpcs, None), _ptr_array(offs, None), _ptr_array(flats, None),
            labels, labels.size, m, seed, out, C.byref(cnt), C.byref(ca))
    return rc, out[: cnt.value].copy(), bool(ca.value)


def select_shards_stream(n: int, shards, labels: np.ndarray, m: int, words: np.ndarray):
    """select_active_classes(span<CompressedKnnGraph>) with the padding draw's mt19937_64 words
    replaced by `words` (or_select_active_shards_stream: drives the Lemire rejection loop)."""
    p = len(shards)
    flats = [s[2] if s[2].size else np.zeros(1, np.uint32) for s in shards]
    out = np.zeros(max(m, 1), np.uint32)
    cnt = U64(0)
    ca = C.c_int(0)
    labels = np.ascontiguousarray(labels, dtype=np.uint32)
    words = np.ascontiguousarray(words, dtype=np.uint64)
    fn = oracle().or_select_active_shards_stream
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, C.c_void_p, C.c_void_p, C.c_void_p, u32p, U64, U64, u64p, U64, u32p,
                   C.POINTER(U64), C.POINTER(C.c_int)]
    rc = fn(n, p, _ptr_array([s[0] for s in shards], None), _ptr_array([s[1] for s in shards], None),
            _ptr_array(flats, None), labels, labels.size, m, words, words.size, out, C.byref(cnt),
            C.byref(ca))
    return rc, out[: cnt.value].copy(), bool(ca.value)


def select_full(lib_kind: str, g: np.ndarray, labels: np.ndarray, m: int, seed: int):
    n, k = g.shape
    out = np.zeros(max(m, 1), np.uint32)
    cnt = U64(0)
    ca = C.c_int(0)
    fn = oracle().or_select_active_full if lib_kind == "oracle" else ref().ref_select_active_full
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, u32p, u32p, U64, U64, U64, u32p, C.POINTER(U64), C.POINTER(C.c_int)]
    labels = np.ascontiguousarray(labels, dtype=np.uint32)
    rc = fn(n, k, np.ascontiguousarray(g), labels, labels.size, m, seed, out, C.byref(cnt),
            C.byref(ca))
    return rc, out[: cnt.value].copy(), bool(ca.value)


def mt64_stream(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    fn = oracle().or_mt64_stream
    fn.argtypes = [U64, U64, u64p]
    fn(seed, count, out)
    return out


def uniform_picks(seed: int, csize: int, need: int) -> np.ndarray:
    out = np.zeros(max(need, 1), np.uint64)
    fn = oracle().or_uniform_picks
    fn.argtypes = [U64, U64, U64, u64p]
    fn(seed, csize, need, out)
    return out[:need]


def fc_train_step(w: np.ndarray, vel: np.ndarray, x: np.ndarray, labels: np.ndarray, shards,
                  m: int, seed: int, scale=30.0, lr=0.1, momentum=0.9, wd=0.0, want_logits=False):
    """Oracle restatement of the fc half of HybridSim::train_step (one micro-batch).
    Updates w and vel in place; returns (rc, loss, active, grad_feat, logits|None)."""
    n, d = w.shape
    b = x.shape[0]
    p = len(shards)
    active = np.zeros(max(m, 1), np.uint32)
    cnt = U64(0)
    loss = C.c_double(0)
    gfeat = np.zeros((b, d), np.float32)
    logits = np.zeros((b, m), np.float32) if want_logits else None
    fn = oracle().or_fc_train_step
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, U64, f32p, f32p, f32p, u32p, U64, C.c_void_p, C.c_void_p,
                   C.c_void_p, U64, U64, C.c_float, C.c_float, C.c_float, C.c_float,
                   C.POINTER(C.c_double), u32p, C.POINTER(U64), f32p, C.c_void_p]
    flats = [s[2] if s[2].size else np.zeros(1, np.uint32) for s in shards]
    rc = fn(n, d, p, w, vel, np.ascontiguousarray(x, np.float32),
            np.ascontiguousarray(labels, np.uint32), b,
            _ptr_array([s[0] for s in shards], None), _ptr_array([s[1] for s in shards], None),
            _ptr_array(flats, None), m, seed, scale, lr, momentum, wd, C.byref(loss), active,
            C.byref(cnt), gfeat, logits.ctypes.data_as(C.c_void_p) if want_logits else None)
    act = active[: cnt.value].copy()
    if want_logits:
        logits = logits[:, : act.size].copy()
    return rc, loss.value, act, gfeat, logits


def fc_train_step_mb(w: np.ndarray, vel: np.ndarray, x: np.ndarray, labels: np.ndarray, shards,
                     m: int, seed: int, micro: int, scale=30.0, lr=0.1, momentum=0.9, wd=0.0):
    """Oracle fc half of HybridSim::train_step with `micro` micro-batches (or_fc_train_step_mb).
    Updates w and vel in place; returns (rc, loss, active, grad_feat)."""
    n, d = w.shape
    b = x.shape[0]
    p = len(shards)
    active = np.zeros(max(m, 1), np.uint32)
    cnt = U64(0)
    loss = C.c_double(0)
    gfeat = np.zeros((b, d), np.float32)
    fn = oracle().or_fc_train_step_mb
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, U64, f32p, f32p, f32p, u32p, U64, C.c_void_p, C.c_void_p,
                   C.c_void_p, U64, U64, C.c_float, C.c_float, C.c_float, C.c_float, U64,
                   C.POINTER(C.c_double), u32p, C.POINTER(U64), f32p]
    flats = [s[2] if s[2].size else np.zeros(1, np.uint32) for s in shards]
    rc = fn(n, d, p, w, vel, np.ascontiguousarray(x, np.float32),
            np.ascontiguousarray(labels, np.uint32), b,
            _ptr_array([s[0] for s in shards], None), _ptr_array([s[1] for s in shards], None),
            _ptr_array(flats, None), m, seed, scale, lr, momentum, wd, micro, C.byref(loss),
            active, C.byref(cnt), gfeat)
    return rc, loss.value, active[: cnt.value].copy(), gfeat


def bruteforce_graph(lib_kind: str, w_norm: np.ndarray, k: int):
    n, d = w_norm.shape
    out = np.zeros((n, k), np.uint32)
    fn = (oracle().or_build_graph_bruteforce if lib_kind == "oracle"
          else ref().ref_build_graph_bruteforce)
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, f32p, U64, u32p]
    rc = fn(n, d, np.ascontiguousarray(w_norm, np.float32), k, out)
    return rc, out


def graph_row(w_norm: np.ndarray, j: int, k: int) -> np.ndarray:
    n, d = w_norm.shape
    out = np.zeros(k, np.uint32)
    fn = oracle().or_graph_row
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, f32p, U64, U64, u32p]
    assert fn(n, d, np.ascontiguousarray(w_norm, np.float32), j, k, out) == 0
    return out


def knn_softmax_fwd_bwd(lib_kind: str, x_norm, w_norm, labels, active, scale=30.0):
    """knn_softmax_forward_backward (knn_softmax.cpp:136-186) via the oracle ('oracle'; grad
    weights compact, m_act x d) or the compiled reference ('ref'; dense n x d, the active rows
    gathered here).  Returns (rc, loss, grad_logits, grad_features, grad_w_active)."""
    x = np.ascontiguousarray(x_norm, np.float32)
    w = np.ascontiguousarray(w_norm, np.float32)
    lab = np.ascontiguousarray(labels, np.uint32)
    act = np.ascontiguousarray(active, np.uint32)
    b, d = x.shape
    n, m = w.shape[0], act.size
    loss = C.c_double(0)
    gl = np.zeros((b, max(m, 1)), np.float32)
    gf = np.zeros((b, d), np.float32)
    if lib_kind == "oracle":
        gw = np.zeros((max(m, 1), d), np.float32)
        fn = oracle().or_knn_softmax_forward_backward
    else:
        gw = np.zeros((n, d), np.float32)
        fn = ref().ref_knn_softmax_forward_backward
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, U64, f32p, f32p, u32p, u32p, U64, C.c_float, C.POINTER(C.c_double),
                   f32p, f32p, f32p]
    rc = fn(b, n, d, x, w, lab, act, m, scale, C.byref(loss), gl, gf, gw)
    if lib_kind != "oracle" and rc == 0:
        gw = gw[act.astype(np.int64)]
    return rc, loss.value, gl[:, :m], gf, gw[:m]


class GraphRowChecker:
    """Exact build_graph_bruteforce rows of a few query classes over a class matrix streamed in
    chunks (or_graph_rows_update): feed every chunk once, in any order; rows() then equals
    graph_row() on the whole matrix."""

    def __init__(self, qid, q: np.ndarray, k: int):
        self.qid = np.ascontiguousarray(qid, np.uint64)
        self.q = np.ascontiguousarray(q, np.float32)
        self.k = k
        nq = self.qid.size
        self.sc = np.zeros((nq, k), np.float32)
        self.ix = np.zeros((nq, k), np.uint32)
        self.sz = np.zeros(nq, np.uint64)
        fn = oracle().or_graph_rows_update
        fn.restype = None
        fn.argtypes = [U64, U64, f32p, u64p, U64, f32p, U64, U64, f32p, u32p, u64p]

    def update(self, chunk: np.ndarray, base: int) -> None:
        chunk = np.ascontiguousarray(chunk, np.float32)
        oracle().or_graph_rows_update(self.qid.size, self.q.shape[1], self.q, self.qid, self.k,
                                      chunk, chunk.shape[0], base, self.sc, self.ix, self.sz)

    def rows(self) -> np.ndarray:
        assert (self.sz == self.k).all()
        return self.ix.copy()


def l2_normalize(x: np.ndarray):
    x = np.ascontiguousarray(x, np.float32)
    r, c = x.shape
    out = np.zeros_like(x)
    norms = np.zeros(r, np.float32)
    bad = U64(0)
    fn = oracle().or_l2_normalize_rows
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, f32p, C.c_float, f32p, f32p, C.POINTER(U64)]
    rc = fn(r, c, x, 1e-12, out, norms, C.byref(bad))
    return rc, out, norms, bad.value


def softmax_xent(lib_kind: str, logits: np.ndarray, labels: np.ndarray):
    logits = np.ascontiguousarray(logits, np.float32)
    m, c = logits.shape
    grad = np.zeros_like(logits)
    loss = C.c_double(0)
    fn = oracle().or_softmax_xent if lib_kind == "oracle" else ref().ref_softmax_xent
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, f32p, u32p, C.POINTER(C.c_double), f32p]
    rc = fn(m, c, logits, np.ascontiguousarray(labels, np.uint32), C.byref(loss), grad)
    return rc, loss.value, grad


class RefSim:
    """The reference's stock HybridSim (identity feature extractor) -- oracle/_ref."""

    def __init__(self, w: np.ndarray, p: int, threads: bool = False, scale=30.0, momentum=0.9,
                 wd=0.0):
        self.n, self.d = w.shape
        self.p = p
        self.h = ref().ref_sim_create(self.n, self.d, p, int(threads), scale, momentum, wd,
                                      np.ascontiguousarray(w, np.float32))
        assert self.h

    def set_graphs(self, shards):
        self._keep = shards
        flats = [s[2] if s[2].size else np.zeros(1, np.uint32) for s in shards]
        rc = ref().ref_sim_set_graphs(self.h, len(shards), _ptr_array([s[0] for s in shards], None),
                                      _ptr_array([s[1] for s in shards], None),
                                      _ptr_array(flats, None))
        assert rc == 0

    def step_mb(self, x, labels, m, seed, micro, lr=0.1, reset_fe=True):
        """train_step with StepOptions::micro_batches = micro (parallel.cpp:444)."""
        if reset_fe:
            assert ref().ref_sim_reset_fe(C.c_void_p(self.h)) == 0
        loss = C.c_double(0)
        na = U64(0)
        rc = ref().ref_sim_step_mb(self.h, np.ascontiguousarray(x, np.float32),
                                   np.ascontiguousarray(labels, np.uint32), x.shape[0], m, seed,
                                   lr, micro, C.byref(loss), C.byref(na))
        return rc, loss.value, na.value

    def step(self, x, labels, m, seed, lr=0.1, reset_fe=True):
        if reset_fe:
            assert ref().ref_sim_reset_fe(C.c_void_p(self.h)) == 0
        loss = C.c_double(0)
        na = U64(0)
        rc = ref().ref_sim_step(self.h, np.ascontiguousarray(x, np.float32),
                                np.ascontiguousarray(labels, np.uint32), x.shape[0], m, seed, lr,
                                C.byref(loss), C.byref(na))
        return rc, loss.value, na.value

    def weights(self) -> np.ndarray:
        w = np.zeros((self.n, self.d), np.float32)
        ref().ref_sim_get_weights(self.h, w)
        return w

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_sim_destroy(self.h)
            self.h = None


def ref_feature_grad(w, x, labels, active, p, scale=30.0):
    n, d = w.shape
    b = x.shape[0]
    g = np.zeros((b, d), np.float32)
    loss = C.c_double(0)
    fn = ref().ref_fc_feature_grad
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, U64, f32p, f32p, u32p, U64, u32p, U64, C.c_float,
                   C.POINTER(C.c_double), f32p]
    rc = fn(n, d, p, np.ascontiguousarray(w, np.float32), np.ascontiguousarray(x, np.float32),
            np.ascontiguousarray(labels, np.uint32), b, np.ascontiguousarray(active, np.uint32),
            active.size, scale, C.byref(loss), g)
    return rc, loss.value, g


def ref_save_graph(path: str, g: np.ndarray) -> int:
    """The reference's save_graph (through oracle/_ref)."""
    g = np.ascontiguousarray(g, np.uint32)
    fn = ref().ref_save_graph
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, U64, U64, u32p]
    return fn(path.encode(), g.shape[0], g.shape[1], g)


def ref_load_graph(path: str):
    """The reference's load_graph: (rc, graph ndarray or None)."""
    fn = ref().ref_load_graph
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.POINTER(U64), C.POINTER(U64), C.c_void_p]
    n, k = U64(), U64()
    rc = fn(path.encode(), C.byref(n), C.byref(k), None)
    if rc:
        return rc, None
    out = np.zeros((n.value, k.value), np.uint32)
    rc = fn(path.encode(), C.byref(n), C.byref(k), out.ctypes.data)
    return rc, out


def classify_retrieval(q: np.ndarray, w: np.ndarray):
    """classify_retrieval restated in oracle/: (rc, classes u32, cosines)."""
    q = np.ascontiguousarray(q, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    out = np.zeros(q.shape[0], np.uint32)
    sc = np.zeros(q.shape[0], np.float32)
    fn = oracle().or_classify_retrieval
    fn.restype = C.c_int
    fn.argtypes = [U64, U64, U64, f32p, f32p, u32p, f32p]
    rc = fn(q.shape[0], w.shape[0], q.shape[1], q, w, out, sc)
    return rc, out, sc


def topk(lib_kind: str, t: np.ndarray, k: int, m_chunks: int = 0):
    """topk_divide_conquer: (rc, indices u64, values) from the oracle or the reference."""
    t = np.ascontiguousarray(t, np.float32)
    idx = np.zeros(max(k, 1), np.uint64)
    val = np.zeros(max(k, 1), np.float32)
    if lib_kind == "ref":
        fn = ref().ref_topk
        fn.restype = C.c_int
        fn.argtypes = [U64, f32p, U64, U64, u64p, f32p]
        rc = fn(t.size, t, k, m_chunks, idx, val)
    else:
        fn = oracle().or_topk
        fn.restype = C.c_int
        fn.argtypes = [U64, f32p, U64, u64p, f32p]
        rc = fn(t.size, t, k, idx, val)
    return rc, idx[:k], val[:k]


class OracleDgc:
    """CompressionState restated in oracle/ (or_dgc_step), one state per layer."""

    def __init__(self, ratio: float, momentum: float):
        self.ratio, self.momentum, self.state = ratio, momentum, {}

    def step(self, layer: int, g: np.ndarray):
        g = np.ascontiguousarray(g, np.float32)
        vel, res = self.state.setdefault(layer, (np.zeros(g.size, np.float32),
                                                 np.zeros(g.size, np.float32)))
        idx = np.zeros(g.size, np.uint64)
        val = np.zeros(g.size, np.float32)
        cnt = U64()
        fn = oracle().or_dgc_step
        fn.restype = C.c_int
        fn.argtypes = [U64, f32p, f32p, f32p, C.c_double, C.c_float, u64p, f32p, C.POINTER(U64)]
        rc = fn(g.size, g, vel, res, self.ratio, self.momentum, idx, val, C.byref(cnt))
        assert rc == 0
        return idx[: cnt.value], val[: cnt.value]


class RefDgc:
    """The reference's CompressionState through oracle/_ref."""

    def __init__(self, ratio: float, momentum: float):
        lib = ref()
        lib.ref_dgc_create.restype = C.c_void_p
        lib.ref_dgc_create.argtypes = [C.c_double, C.c_float]
        lib.ref_dgc_step.restype = C.c_int
        lib.ref_dgc_step.argtypes = [C.c_void_p, C.c_uint32, U64, f32p, U64, u64p, f32p,
                                     C.POINTER(U64)]
        lib.ref_dgc_residual.restype = C.c_int
        lib.ref_dgc_residual.argtypes = [C.c_void_p, C.c_uint32, U64, f32p]
        lib.ref_dgc_set_sparsity.restype = C.c_int
        lib.ref_dgc_set_sparsity.argtypes = [C.c_void_p, C.c_double]
        lib.ref_dgc_destroy.argtypes = [C.c_void_p]
        self.lib, self.h = lib, lib.ref_dgc_create(ratio, momentum)

    def set_sparsity(self, r: float) -> int:
        return self.lib.ref_dgc_set_sparsity(self.h, r)

    def step(self, layer: int, g: np.ndarray, m_chunks: int = 0):
        g = np.ascontiguousarray(g, np.float32)
        idx = np.zeros(g.size, np.uint64)
        val = np.zeros(g.size, np.float32)
        cnt = U64()
        rc = self.lib.ref_dgc_step(self.h, layer, g.size, g, m_chunks, idx, val, C.byref(cnt))
        return rc, idx[: cnt.value], val[: cnt.value]

    def residual(self, layer: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        assert self.lib.ref_dgc_residual(self.h, layer, n, out) == 0
        return out

    def __del__(self):
        try:
            self.lib.ref_dgc_destroy(self.h)
        except Exception:
            pass
