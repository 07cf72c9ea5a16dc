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


SHIM_LIB = os.path.join(ROOT, "paper_2102_06025_b200", "libxcls_gpu.so")


def compile_shim_caller(out_path):
    """g++ -std=c++20 of tests/cpp/shim_caller.cpp against include/xcls_gpu.hpp, linked with
    libxcls_gpu.so + libxknn.so (no GPU needed to compile and link)."""
    import subprocess

    pkg = os.path.join(ROOT, "paper_2102_06025_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-o", out_path, os.path.join(ROOT, "tests", "cpp", "shim_caller.cpp"), "-L", pkg,
           "-lxcls_gpu", "-lxknn", f"-Wl,-rpath,{pkg}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_cpp_shim_caller_compiles_and_links(tmp_path):
    """A C++ caller written against the reference's xcls:: API (namespace xcls = xcls_gpu)
    compiles against include/xcls_gpu.hpp and links the shim and the C-ABI library."""
    if not os.path.exists(SHIM_LIB):
        pytest.skip("libxcls_gpu.so not built")
    compile_shim_caller(str(tmp_path / "shim_caller"))
    assert os.path.exists(tmp_path / "shim_caller")


def test_c_caller_compiles_and_links(tmp_path):
    """A plain C11 caller of include/xknn.h (the cgo/FFI view of the boundary) compiles and
    links against libxknn.so; it runs the host-only entry points."""
    import subprocess

    if not os.path.exists(LIB):
        pytest.skip("libxknn.so not built")
    src = tmp_path / "c_caller.c"
    src.write_text(r'''
#include <stdio.h>
#include "xknn.h"
int main(void) {
  uint64_t b = 0, e = 0;
  if (xknn_shard_range(1000003, 4, 3, &b, &e) != XKNN_OK) return 1;
  if (xknn_shard_range(10, 3, 3, &b, &e) != XKNN_ERR_INVALID_ARGUMENT) return 2;
  printf("%llu %llu %s %llu\n", (unsigned long long)b, (unsigned long long)e,
         xknn_status_string(XKNN_ERR_LABEL_NOT_ACTIVE),
         (unsigned long long)xknn_dgc_selected_count(0.99, 1000));
  return 0;
}
''')
    pkg = os.path.join(ROOT, "paper_2102_06025_b200")
    exe = str(tmp_path / "c_caller")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", exe,
                        str(src), "-L", pkg, "-lxknn", f"-Wl,-rpath,{pkg}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    b, e = O.shard_range(1000003, 4, 3)
    fn = O.oracle().or_selected_count
    fn.restype, fn.argtypes = C.c_uint64, [C.c_double, C.c_uint64]
    assert r.stdout.split() == [str(b), str(e), "LabelNotActive", str(fn(0.99, 1000))]
