"""The C-ABI library loads without a GPU and exports every entry point include/xknn.h declares;
host-only entry points agree with the reference layout (no GPU compute here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xknn.h")
LIB = os.path.join(ROOT, "paper_2102_06025_b200", "libxknn.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xknn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("xknn_layer_create", "xknn_step", "xknn_select", "xknn_layer_set_graph_csr"):
        assert s in syms


def test_library_exports_every_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libxknn.so not built")
    lib = C.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_package_import_and_shard_layout():
    if not os.path.exists(LIB):
        pytest.skip("libxknn.so not built")
    import paper_2102_06025_b200 as X

    for n, p in [(10, 3), (100_000, 8), (7, 7), (1_000_003, 4)]:
        lay = X.ShardLayout(n, p)
        for s in range(p):
            assert lay.class_range(s) == O.shard_range(n, p, s)
        for c in np.random.default_rng(0).integers(0, n, 50):
            b, e = lay.class_range(lay.shard_of(int(c)))
            assert b <= c < e
    with pytest.raises(X.InvalidArgument):
        X.ShardLayout(10, 3).class_range(3)
