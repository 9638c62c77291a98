"""Runtime properties of the library on the GPU: workspace release (the boundary of
include/cr.h) and run-to-run determinism of the schedule-dependent parallel stages (the K5
reduction commits columns asynchronously and the H0 merge rounds use atomics; their results must
not depend on timing -- SURVEY §4 T5)."""
import hashlib

import numpy as np
import pytest

from workloads import generators as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cr():
    import torch
    import paper_2005_12692_b200 as m
    torch.cuda.init()
    return m


def test_release_workspace_returns_memory(cr):
    import torch
    torch.cuda.synchronize()
    cr.release_workspace()
    torch.cuda.empty_cache()
    free0 = torch.cuda.mem_get_info()[0]
    v, md = gen.config("c4")
    t = torch.from_numpy(v).cuda()
    cr.barcodes(t, md)
    held = cr.workspace_bytes()
    assert held > 100 * 2 ** 20  # births, tags, owner table, pools of a 128^3 volume are cached
    free_mid = torch.cuda.mem_get_info()[0]
    assert free_mid < free0 - held // 2
    del t
    torch.cuda.empty_cache()
    cr.release_workspace()
    assert cr.workspace_bytes() == 0
    free1 = torch.cuda.mem_get_info()[0]
    assert free1 >= free0 - 64 * 2 ** 20, (free0, free_mid, free1)
    # and the library still works after a release
    check = cr.barcodes(torch.from_numpy(gen.iid_uniform((40, 44), 5)).cuda(), 1)
    assert len(check.pairs) > 0


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["c4", "c5crop96"])
def test_repeated_calls_bit_identical(cr, name):
    """10 repeated calls give byte-identical bars (with birth cells) and pairings."""
    import torch
    if name == "c4":
        v, md = gen.config("c4")
    else:
        v = gen.masked_grf((384, 384, 384), 3.0, 180.0, 5)[144:240, 144:240, 144:240].copy()
        md = 2
    t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    seen = set()
    for _ in range(10):
        bc = cr.barcodes(t, md, cells=True)
        p = cr.pairing(t)
        seen.add(_digest(bc.pairs.cpu().numpy(), bc.cells.cpu().numpy(), p.cpu().numpy()))
    assert len(seen) == 1
