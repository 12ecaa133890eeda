"""The C-ABI library loads, exports every symbol include/egonet.h declares, and its
host-only helpers behave (-m "not gpu": no compute calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "egonet.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^EG_API[^(]*?\b(eg_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2112_15345_b200 import egonet
    L = egonet.lib()
    declared = _declared()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(egonet.ABI_SYMBOLS)
    assert egonet.version().startswith("egonet")


def test_library_is_sm100a_sass():
    import subprocess
    from paper_2112_15345_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_range_bounds_policy():
    from paper_2112_15345_b200 import egonet
    assert list(egonet.range_bounds(10, 4)) == [0, 2, 5, 7, 10]
    assert list(egonet.range_bounds(0, 3)) == [0, 0, 0, 0]
    n = 244_160_499
    b = egonet.range_bounds(n, 8)
    assert b[0] == 0 and b[-1] == n and all(b[p] == p * n // 8 for p in range(9))


def test_batch_caps_closed_form():
    from paper_2112_15345_b200 import egonet
    # homogeneous, 3 hops of [15,10,5], batch 1024: 1024 -> 1024*16 -> *11 -> *6 (capped by N)
    cn, ce = egonet.batch_caps([10**8], [0], [0], [10**9], [1000], 1024, [[15], [10], [5]])
    assert list(ce[:, 0]) == [1024 * 15, 1024 * 16 * 10, 1024 * 16 * 11 * 5]
    assert cn[0] == 1024 * 16 * 11 * 6
    # fanout -1 uses the max in-degree; caps never exceed |E_r| or N_t
    cn, ce = egonet.batch_caps([50, 20], [0], [1], [300], [40], 10, [[-1]])
    assert ce[0, 0] == 300 and cn[0] == 50 and cn[1] == 10
    cn, ce = egonet.batch_caps([50, 20], [0], [1], [300], [40], 10, [[0]])
    assert ce[0, 0] == 0 and cn[0] == 10 and cn[1] == 10   # seeds of either type, no edges


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2112_15345_b200 import egonet
    h = ctypes.c_void_p()
    rc = egonet.lib().eg_create(0, 1, 0, None, ctypes.byref(h))
    assert rc == -4 and not h.value          # EG_ECUDA, no context, no CPU fallback


def test_bad_arguments_rejected_on_host():
    from paper_2112_15345_b200 import egonet
    L = egonet.lib()
    h = ctypes.c_void_p()
    assert L.eg_create(2, 2, 0, None, ctypes.byref(h)) == -1      # rank >= world
    assert L.eg_create(0, 9, 0, None, ctypes.byref(h)) == -1      # world > EG_MAX_RANKS
    assert L.eg_range_bounds(5, 0, None) == -1
    assert L.eg_sample_blocks(None, None, 0, 1, None, 0, ctypes.byref(h)) == -1


def test_product_package_does_not_touch_the_oracle():
    """The product path never imports, includes, links or loads oracle/."""
    pkg = os.path.join(ROOT, "paper_2112_15345_b200")
    bad = re.compile(r"(import\s+oracle|from\s+oracle|#include\s*[<\"][^>\"]*oracle|liboracle|og_sample|og_gather)")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c", ".cc")):
                with open(os.path.join(dirpath, f)) as fh:
                    assert not bad.search(fh.read()), f
