"""Host-only checks of the C ABI (no GPU needed): the library loads, exports every symbol that
include/cr.h declares, and its host-side functions/validation behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cr():
    from paper_2005_12692_b200 import build
    build.build()
    import paper_2005_12692_b200 as m
    return m


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cr_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(cr):
    names = declared_functions()
    assert "cr_barcodes" in names and "cr_pairing" in names and "cr_barcodes_batched" in names
    lib = ctypes.CDLL(cr.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(cr.EXPORTED)


def test_no_oracle_in_product(cr):
    import subprocess
    out = subprocess.run(["ldd", cr.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out
    pkg = os.path.join(ROOT, "paper_2005_12692_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "cr_oracle" not in txt, f


def test_max_pairs_and_num_cells(cr):
    import oracle
    for shape in [(7,), (1,), (5, 6), (3, 4, 5), (128, 128), (1, 1, 9)]:
        for md in range(4):
            assert cr.max_pairs(shape, md) == oracle.max_pairs(shape, min(md, 3))
        K = 1
        for s in shape:
            K *= 2 * s - 1
        assert cr.num_cells(shape) == K
    with pytest.raises(cr.CrError):
        cr.max_pairs((0, 3), 1)
    with pytest.raises(cr.CrError):
        cr.num_cells((1 << 17, 1 << 17))  # Khalimsky size >= 2^32


def test_validation_before_any_cuda_call(cr):
    lib = ctypes.CDLL(cr.LIB_PATH)
    lib.cr_barcodes.restype = ctypes.c_int
    shape = (ctypes.c_int64 * 2)(4, 4)
    n = ctypes.c_int64(0)
    # null image
    assert lib.cr_barcodes(None, shape, 2, 1, None, None, ctypes.c_int64(0), ctypes.byref(n), None) == cr.CR_EINVAL
    # bad ndim / maxdim / shape
    dummy = ctypes.c_void_p(16)
    assert lib.cr_barcodes(dummy, shape, 4, 1, None, None, ctypes.c_int64(0), ctypes.byref(n), None) == cr.CR_EINVAL
    assert lib.cr_barcodes(dummy, shape, 2, -1, None, None, ctypes.c_int64(0), ctypes.byref(n), None) == cr.CR_EINVAL
    bad = (ctypes.c_int64 * 2)(4, 0)
    assert lib.cr_barcodes(dummy, bad, 2, 1, None, None, ctypes.c_int64(0), ctypes.byref(n), None) == cr.CR_EINVAL
    # pairing with null partner
    lib.cr_pairing.restype = ctypes.c_int
    assert lib.cr_pairing(dummy, shape, 2, None, None) == cr.CR_EINVAL
    lib.cr_status_string.restype = ctypes.c_char_p
    assert b"invalid" in lib.cr_status_string(cr.CR_EINVAL)
