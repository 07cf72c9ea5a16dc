import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs the compiled reference oracle/_ref")


def pytest_collection_modifyitems(config, items):
    import oracle_lib

    skip_ref = pytest.mark.skip(reason="oracle/_ref/libxcls_ref.so not built (no /root/reference)")
    for it in items:
        if "ref" in it.keywords and not oracle_lib.ref_available():
            it.add_marker(skip_ref)
