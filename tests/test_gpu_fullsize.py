"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C2, C3 and C4 are compared element by element with the oracle (bars, birth cells, and for C4
the full pairing).  C5 (451 M cells) is beyond the oracle's memory/time budget, so it is checked
by properties that hold at any size: the Euler-characteristic curve (an exact integer identity
between cell counts computed here from the image with numpy and the bars alive at each
threshold), one essential class for the contractible ball domain, and births/deaths drawn from
the image's values; its cropped version is compared element by element in test_gpu_parity.py.
"""
import os
from multiprocessing import Pool

import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def cr():
    import torch
    import paper_2005_12692_b200 as m
    torch.cuda.init()
    return m


def _bars(cr, img, maxdim, batched=False):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    if batched:
        bc, off = cr.barcodes_batched(t, maxdim, cells=True)
        return bc.numpy(), off.cpu().numpy()
    return cr.barcodes(t, maxdim, cells=True).numpy()


def _eq(g, o, ctx):
    d, b, e, c = g
    assert len(d) == len(o.dim), ctx
    assert np.array_equal(d, o.dim), ctx
    assert np.array_equal(c, o.cell), ctx
    assert np.array_equal(b.view(np.uint32), o.birth.view(np.uint32)), ctx
    assert np.array_equal(e.view(np.uint32), o.death.view(np.uint32)), ctx


def test_c2_full(cr):
    x, md = gen.config("c2")
    _eq(_bars(cr, x, md), oracle.ph(x, md), "c2")


def _oracle_one(args):
    img, md = args
    r = oracle.ph(img, md)
    return r.dim, r.birth, r.death, r.cell


def test_c3_full(cr):
    imgs, md = gen.config("c3")
    (d, b, e, c), off = _bars(cr, imgs, md, batched=True)
    with Pool(min(32, os.cpu_count() or 1)) as pool:
        res = pool.map(_oracle_one, [(im, md) for im in imgs], chunksize=256)
    for i, (od, ob, oe, oc) in enumerate(res):
        s = slice(off[i], off[i + 1])
        assert np.array_equal(d[s], od), i
        assert np.array_equal(c[s], oc), i
        assert np.array_equal(b[s].view(np.uint32), ob.view(np.uint32)), i
        assert np.array_equal(e[s].view(np.uint32), oe.view(np.uint32)), i


def test_c4_full_with_pairing(cr):
    import torch
    v, md = gen.config("c4")
    o = oracle.ph(v, md, partner=True)
    _eq(_bars(cr, v, md), o, "c4")
    p = cr.pairing(torch.from_numpy(v).cuda()).cpu().numpy().view(np.uint32)
    assert np.array_equal(p, o.partner)


def _cell_births_3d(v):
    """Births of every cell type of the 3D V-construction, from the image (numpy)."""
    out = {}
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                b = v[: v.shape[0] - dz, : v.shape[1] - dy, : v.shape[2] - dx]
                for sz in range(dz + 1):
                    for sy in range(dy + 1):
                        for sx in range(dx + 1):
                            b = np.maximum(b, v[sz: v.shape[0] - dz + sz, sy: v.shape[1] - dy + sy,
                                                sx: v.shape[2] - dx + sx])
                out[(dz, dy, dx)] = b
    return out


def test_c5_properties(cr):
    v, md = gen.config("c5")
    d, b, e, c = _bars(cr, v, md)
    # births and finite deaths are values of the image
    vals = np.unique(v[np.isfinite(v)])
    assert np.all(np.isin(b, vals))
    assert np.all(np.isin(e[np.isfinite(e)], vals))
    assert np.all(e > b)
    # the ball is contractible: exactly one essential class, in dimension 0
    ess = np.isinf(e)
    assert ess.sum() == 1 and d[ess][0] == 0
    # Euler curve: sum_d (-1)^d #{d-cells born <= t} == sum_d (-1)^d #{bars alive at t}
    births = _cell_births_3d(v.astype(np.float32))
    sorted_by_dim = {k: np.sort(a[np.isfinite(a)], axis=None) for k, a in births.items()}
    ts = np.quantile(vals, np.linspace(0, 1, 48))
    for t in ts:
        lhs = 0
        for (dz, dy, dx), a in sorted_by_dim.items():
            lhs += (-1) ** (dz + dy + dx) * int(np.searchsorted(a, t, side="right"))
        alive = (b <= t) & (t < e)
        rhs = int(np.sum(np.where(d[alive] % 2 == 0, 1, -1)))
        assert lhs == rhs, t


def _eq64(cr, img, md, ctx):
    import torch
    o = oracle.ph(img, md, dtype=np.float64)
    d, b, e, c = cr.barcodes_f64(torch.from_numpy(img).cuda(), md, cells=True).numpy()
    assert len(d) == len(o.dim), ctx
    assert np.array_equal(d, o.dim), ctx
    assert np.array_equal(c, o.cell), ctx
    assert np.array_equal(b.view(np.uint64), o.birth.view(np.uint64)), ctx
    assert np.array_equal(e.view(np.uint64), o.death.view(np.uint64)), ctx


def test_c2_full_f64(cr):
    """C2's random walk kept in float64 (rank path: 2^24 distinct doubles)."""
    x = gen.random_walk(1 << 24, 2, dtype=np.float64)
    _eq64(cr, x, 0, "c2_f64")


def test_c1_and_c4_crop_f64(cr):
    rng = np.random.default_rng(11)
    _eq64(cr, rng.random((128, 128)), 1, "c1_f64")
    _eq64(cr, gen.grf((48, 48, 48), 2.0, 4).astype(np.float64) + rng.random((48, 48, 48)) * 1e-12,
          2, "c4crop_f64")
