"""End-to-end entry with host buffers (cr_barcodes_batched_host, include/cr.h): the stacked 3D /
large-2D path copies the host batch in pieces straight into the stacked layout while the
filtration of the arrived planes runs; the small-2D and 1D paths copy it whole.
Every case must equal the device-resident cr_barcodes_batched call byte for byte."""
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


def _both(cr, imgs, md):
    import torch
    imgs = np.ascontiguousarray(imgs, dtype=np.float32)
    dbc, doff = cr.barcodes_batched(torch.from_numpy(imgs).cuda(), md, cells=True)
    hbc, hoff = cr.barcodes_batched_host(imgs, md, cells=True)
    return (dbc.pairs.cpu().numpy(), dbc.cells.cpu().numpy(), doff.cpu().numpy(),
            np.asarray(hbc.pairs), np.asarray(hbc.cells), np.asarray(hoff))


@pytest.mark.parametrize("case", ["3d_12", "3d_9_ragged_pieces", "3d_1", "2d_large", "2d_small_k7"])
def test_host_batch_equals_device_batch(cr, case):
    rng = np.random.default_rng(77)
    if case == "3d_12":
        imgs, md = np.stack([gen.masked_grf((40, 40, 40), 3.0, 19.0, rng) for _ in range(12)]), 2
    elif case == "3d_9_ragged_pieces":  # 9 volumes: pieces of 2 (8 pieces, the last one short)
        imgs, md = np.stack([gen.masked_grf((23, 31, 37), 2.0, 15.0, rng) for _ in range(9)]), 2
    elif case == "3d_1":
        imgs, md = gen.masked_grf((30, 30, 30), 3.0, 14.0, rng)[None], 2
    elif case == "2d_large":
        imgs, md = np.stack([gen.iid_uniform((150, 170), 90 + i) for i in range(5)]), 1
    else:
        imgs, md = gen.blobs(64, 5), 1
    dp, dc, do, hp, hc, ho = _both(cr, imgs, md)
    assert np.array_equal(do, ho), case
    assert np.array_equal(dp.view(np.uint32), hp.view(np.uint32)), case
    assert np.array_equal(dc.view(np.uint32), hc.view(np.uint32)), case
    assert len(dp) > 0
