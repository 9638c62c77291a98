"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C2, C3 and C4 are compared element by element with the oracle run live (bars, birth cells, and
for C4 the full pairing).  C5 (384^3, 451 M cells: ~3 min and ~20 GB for the oracle on one core)
and C5b (64 x 128^3) are compared with SHA-256 digests of the oracle's own outputs, written once
by ``tools/oracle_digest.py`` (which calls only ``oracle/``) into
``tests/golden/fullsize_oracle.json``: the bars (dim, birth, death, birth cell, in output order)
and the full partner array over every Khalimsky cell -- bit-exact, element for element, through a
hash.  The same file pins the full-size partner arrays of C1, C2, C4 and of the first 1024 C3
images.  C5 is additionally checked by properties that hold at any size (Euler curve, one
essential class), which localise a failure that the digest only detects.
"""
import hashlib
import json
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


_GOLD = os.path.join(os.path.dirname(__file__), "golden", "fullsize_oracle.json")


@pytest.fixture(scope="module")
def gold():
    with open(_GOLD) as f:
        return json.load(f)


def _bars_digest(d, b, e, c):
    h = hashlib.sha256()
    for a, t in ((d, np.int32), (b, np.float32), (e, np.float32), (c, np.uint32)):
        h.update(np.ascontiguousarray(a).view(t).tobytes())
    return h.hexdigest()


def _partner_digest(cr, img):
    import torch
    p = cr.pairing(torch.from_numpy(np.ascontiguousarray(img)).cuda()).cpu().numpy().view(np.uint32)
    return hashlib.sha256(p.tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_full_partner_digest(cr, gold, name):
    """The full cell pairing (every Khalimsky cell) at BASELINE size equals the oracle's."""
    img, md = gen.config(name)
    assert _bars_digest(*_bars(cr, img, md)) == gold[name]["bars"], name
    assert _partner_digest(cr, img) == gold[name]["partner"], name


def test_c3_partner_first1024(cr, gold):
    imgs = gen.config("c3")[0][:1024]
    want = gold["c3"]["partner_first1024"]
    for i in range(1024):
        assert _partner_digest(cr, imgs[i]) == want[i], i


def test_c5_full_digest(cr, gold):
    """C5 (384^3 GRF in a ball, H0-H2): bars and the full 451 M-cell pairing vs the oracle."""
    v, md = gen.config("c5")
    bars = _bars(cr, v, md)
    assert len(bars[0]) == gold["c5"]["n_bars"]
    assert _bars_digest(*bars) == gold["c5"]["bars"]
    assert _partner_digest(cr, v) == gold["c5"]["partner"]


def test_c5b_full_digest(cr, gold):
    """C5b (64 x 128^3, batched call as bench.py times it): per-volume bars vs the oracle, and
    every volume's full pairing."""
    vols, md = gen.config("c5b")
    (d, b, e, c), off = _bars(cr, vols, md, batched=True)
    recs = gold["c5b"]["volumes"]
    assert len(off) == len(recs) + 1
    for i, r in enumerate(recs):
        s = slice(off[i], off[i + 1])
        assert off[i + 1] - off[i] == r["n_bars"], i
        assert _bars_digest(d[s], b[s], e[s], c[s]) == r["bars"], i
    for i, r in enumerate(recs):
        assert _partner_digest(cr, vols[i]) == r["partner"], i


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
