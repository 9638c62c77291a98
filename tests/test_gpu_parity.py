"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar: bit-exact.  Every birth and death is an input value, so the (dim, birth, death) arrays --
ordered by (dim, birth cell kidx) on both sides -- must be byte-identical, and so must the full
cell pairing (partner array), whose tie-break both sides share (reading R1).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def cr():
    import torch
    import paper_2005_12692_b200 as m
    torch.cuda.init()
    return m


def gpu_bars(cr, img, maxdim):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img, np.float32)).cuda()
    bc = cr.barcodes(t, maxdim, cells=True)
    d, b, e, c = bc.numpy()
    return d, b, e, c


def assert_bars_equal(g, o, ctx=""):
    d, b, e, c = g
    assert len(d) == len(o.dim), (ctx, len(d), len(o.dim))
    assert np.array_equal(d, o.dim), ctx
    assert np.array_equal(c, o.cell), ctx
    assert np.array_equal(b.view(np.uint32), o.birth.view(np.uint32)), ctx
    assert np.array_equal(e.view(np.uint32), o.death.view(np.uint32)), ctx


def check_image(cr, img, maxdim, partner=True, ctx=""):
    o = oracle.ph(img, maxdim, partner=partner)
    assert_bars_equal(gpu_bars(cr, img, maxdim), o, ctx)
    if partner:
        import torch
        p = cr.pairing(torch.from_numpy(np.ascontiguousarray(img, np.float32)).cuda())
        gp = p.cpu().numpy().view(np.uint32)
        assert np.array_equal(gp, o.partner), (ctx, np.flatnonzero(gp != o.partner)[:10])


# ---------------------------------------------------------------- paper examples

def test_golden_examples(cr):
    for name in ["ttk_3x3.json", "fig2_h0.json"]:
        g = json.load(open(os.path.join(GOLDEN, name)))
        img = np.array(g["image"], np.float32)
        d, b, e, _ = gpu_bars(cr, img, g["maxdim"])
        got = sorted(zip(d.tolist(), b.tolist(), e.tolist()))
        exp = sorted((int(x), float(y), float("inf") if z == "inf" else float(z)) for x, y, z in g["expected"])
        assert got == exp, name
        check_image(cr, img, g["maxdim"], ctx=name)


def test_sin_example(cr):
    x = np.linspace(0, 4 * np.pi, 100)
    check_image(cr, (np.sin(x) + 0.1 * x).astype(np.float32), 1)


# ---------------------------------------------------------------- exhaustive tiny sets

def test_exhaustive_2x2_and_2x2x2(cr):
    for vals in itertools.product([0, 1, 2], repeat=4):
        check_image(cr, np.array(vals, np.float32).reshape(2, 2), 1, ctx=vals)
    for vals in itertools.product([0, 1], repeat=8):
        check_image(cr, np.array(vals, np.float32).reshape(2, 2, 2), 2, ctx=vals)


def test_exhaustive_3x3_binary(cr):
    for vals in itertools.product([0, 1], repeat=9):
        check_image(cr, np.array(vals, np.float32).reshape(3, 3), 1, partner=False, ctx=vals)


def test_fuzz_small_with_inf(cr):
    rng = np.random.default_rng(777)
    for t in range(300):
        nd = int(rng.integers(1, 4))
        shape = tuple(int(s) for s in rng.integers(1, 7 if nd < 3 else 5, size=nd))
        img = gen.small_int_image(shape, 5, seed=int(rng.integers(1 << 30)),
                                  inf_frac=0.2 if t % 2 else 0.0)
        check_image(cr, img, 2, ctx=(t, shape))


def test_general_path_on_1d(cr):
    """The general (K1/K2/H0) path and the 1D path agree with the oracle on 1D inputs."""
    x = gen.random_walk(5000, seed=3)
    x[[100, 101, 2500]] = np.inf
    check_image(cr, x, 0, ctx="1d-path")
    with cr.options(force_general=1):
        check_image(cr, x, 0, ctx="general-path")
        check_image(cr, x.reshape(1, -1), 1, ctx="general-path 1xN")


def test_filtration_tiles_ragged(cr):
    """K1+K2 (one fused kernel) on shapes whose extents are not multiples of its tiles (30
    columns x 6 rows x z-chunks; two rows per warp, so odd row counts leave a half-used warp): the
    pairing is the oracle's and the cell / apparent-pair counts equal their numpy definitions
    (tests/apparent.py) -- a missed apparent pair would still be paired by the reduction, so the
    counts are compared too."""
    import torch
    import apparent as ap
    imgs = [gen.masked_grf((33, 37, 41), 2.0, 17.0, 21),
            gen.small_int_image((9, 70, 13), 3, seed=22, inf_frac=0.1),
            gen.small_int_image((67, 35), 4, seed=23, inf_frac=0.05),
            gen.small_int_image((20, 45, 61), 3, seed=24, inf_frac=0.05),
            gen.masked_grf((70, 31, 29), 1.5, 12.0, 25),
            gen.small_int_image((11, 7, 31), 3, seed=26, inf_frac=0.05),   # 7 rows: 6 + 1
            gen.small_int_image((5, 12, 60), 4, seed=27),                 # 12 rows: 2 tiles exactly
            gen.small_int_image((13, 1, 17), 3, seed=28),                 # a single row
            gen.small_int_image((6, 5), 3, seed=29)]                      # 2D, 5 rows
    for k, img in enumerate(imgs):
        o = oracle.ph(img, img.ndim - 1, partner=True)
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        p = cr.pairing(t).cpu().numpy().view(np.uint32)
        assert np.array_equal(p, o.partner), (k, np.flatnonzero(p != o.partner)[:10])
        cr.barcodes(t, img.ndim - 1)
        st = cr.last_stats()
        exp = ap.counts(img)
        assert list(st["cells"]) == exp["cells"], k
        assert list(st["apparent"])[:3] == exp["apparent"][:3], k


def test_filtration_tma_ring(cr):
    """The TMA voxel ring (option kf_tma; nx % 4 == 0: one cp.async.bulk.tensor box per CTA and
    plane from a 16-B aligned column, out-of-image voxels zero-filled by TMA and read as +inf)
    against the oracle and against the per-thread cp.async ring (the product path) on the same
    images: box edges past the image in x (nx < 36,
    nx not a multiple of 30) and y (2D images of few rows), +inf masks, -0.0, planes that are +inf
    over a CTA's footprint (the all-absent fast steps), a 3D batch read unstacked (separator
    planes never loaded) and NaN detection."""
    import torch
    import apparent as ap
    ball = gen.masked_grf((23, 40, 44), 2.0, 12.0, 31)
    ball[:6] = np.inf                                              # all-+inf planes first
    imgs = [gen.small_int_image((4, 4), 3, seed=40),
            gen.small_int_image((3, 8), 3, seed=41, inf_frac=0.2),
            gen.small_int_image((67, 36), 4, seed=42, inf_frac=0.05),
            gen.small_int_image((9, 13, 32), 3, seed=43, inf_frac=0.05),
            gen.masked_grf((17, 31, 64), 1.5, 10.0, 44),
            gen.small_int_image((11, 7, 100), 3, seed=45),
            gen.small_int_image((2, 3, 4), 2, seed=46),
            ball,
            np.array([[0.0, -0.0, 1.0, -0.0], [-0.0, 2.0, 0.0, 1.0]], np.float32)]
    for k, img in enumerate(imgs):
        o = oracle.ph(img, img.ndim - 1, partner=True)
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        for tma in (0, 1):
            with cr.options(kf_tma=tma):
                p = cr.pairing(t).cpu().numpy().view(np.uint32)
                assert np.array_equal(p, o.partner), (k, tma, np.flatnonzero(p != o.partner)[:10])
                assert_bars_equal(gpu_bars(cr, img, img.ndim - 1), o, ctx=(k, tma))
                st = cr.last_stats()
                assert st["kf_tma"] == tma, (k, tma)
                exp = ap.counts(img)
                assert list(st["cells"]) == exp["cells"], k
                assert list(st["apparent"])[:3] == exp["apparent"][:3], k
    vs = np.stack([gen.masked_grf((12, 10, 8), 1.5, 4.5, 60 + s) for s in range(7)])
    with cr.options(kf_tma=1):
        bc, off = cr.barcodes_batched(torch.from_numpy(vs).cuda(), 2, cells=True)
        assert cr.last_stats()["kf_tma"] == 1
    d, b, e, c = bc.numpy()
    off = off.cpu().numpy()
    for i in range(len(vs)):
        s = slice(off[i], off[i + 1])
        assert_bars_equal((d[s], b[s], e[s], c[s]), oracle.ph(vs[i], 2), ctx=("batch", i))
    for shape in ((8, 12), (5, 6, 40)):
        img = gen.small_int_image(shape, 3, seed=70)
        img.flat[img.size // 2] = np.nan
        with cr.options(kf_tma=1), pytest.raises(cr.CrError) as ei:
            cr.barcodes(torch.from_numpy(img).cuda(), len(shape) - 1)
        assert ei.value.status == cr.CR_EINVAL


def test_residual_edge_list_overflow(cr):
    """The filtration lists the residual edges (H0's candidates and, uncleared, the dim-1
    columns), staged per CTA in shared memory; past the stage's capacity (option kf_rcap = 1, 3)
    entries go straight to the global list.  Same pairing and bars as the oracle either way, on
    tie-heavy and iid images (many residual edges per CTA), a masked GRF and a 3D batch."""
    import torch
    imgs = [gen.small_int_image((14, 33, 40), 3, seed=80, inf_frac=0.05),
            gen.iid_uniform((9, 20, 64), 81),
            gen.masked_grf((21, 22, 23), 1.5, 9.0, 82),
            gen.iid_uniform((70, 90), 83)]
    for k, img in enumerate(imgs):
        o = oracle.ph(img, img.ndim - 1, partner=True)
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        for cap in (0, 1, 3):
            with cr.options(kf_rcap=cap):
                p = cr.pairing(t).cpu().numpy().view(np.uint32)
                assert np.array_equal(p, o.partner), (k, cap, np.flatnonzero(p != o.partner)[:10])
                assert_bars_equal(gpu_bars(cr, img, img.ndim - 1), o, ctx=(k, cap))
    vs = np.stack([gen.iid_uniform((6, 7, 8), 90 + s) for s in range(9)])
    with cr.options(kf_rcap=2):
        bc, off = cr.barcodes_batched(torch.from_numpy(vs).cuda(), 2, cells=True)
    d, b, e, c = bc.numpy()
    off = off.cpu().numpy()
    for i in range(len(vs)):
        s = slice(off[i], off[i + 1])
        assert_bars_equal((d[s], b[s], e[s], c[s]), oracle.ph(vs[i], 2), ctx=("batch", i))


def _cavity_cases():
    rng = np.random.default_rng(50)
    a = rng.random((20, 22)).astype(np.float32)
    a[8:12, 9:13] = np.inf                      # enclosed hole: an essential H1 bar
    b = rng.integers(0, 4, (19, 23)).astype(np.float32)
    b[3:6, 3:6] = np.inf                        # two holes and one touching the border
    b[12:15, 15:18] = np.inf
    b[0:4, 20:23] = np.inf
    c = gen.grf((12, 13, 14), 1.5, 51)
    c[5:8, 5:8, 5:9] = np.inf                   # enclosed void: an essential H2 bar
    d = gen.small_int_image((10, 11, 9), 3, seed=52)
    d[4:7, 4:7, :] = np.inf                     # a tunnel through the volume: essential H1
    e = gen.small_int_image((9, 8, 10), 3, seed=53, inf_frac=0.15)
    f = gen.small_int_image((31, 29), 3, seed=54, inf_frac=0.2)
    return {"hole2d": a, "holes2d": b, "void3d": c, "tunnel3d": d, "fuzz3d": e, "fuzz2d": f}


def test_dim1_cavities_and_batches(cr):
    """3D dimension 1 (the coboundary reduction) gives the oracle's bars and pairing incl.
    essential H1 bars (tunnels through +inf) and H1-only requests (maxdim=1); a batch of volumes
    (per-image segments of one reduction) gives each image's oracle bars."""
    import torch
    cases = _cavity_cases()
    imgs = [cases["tunnel3d"], cases["void3d"], cases["fuzz3d"],
            gen.masked_grf((26, 30, 28), 2.0, 13.0, 61),
            gen.small_int_image((12, 14, 11), 3, seed=62, inf_frac=0.08)]
    for k, img in enumerate(imgs):
        for md in (1, 2):
            check_image(cr, img, md, partner=(md == 2), ctx=(k, md))
    vols = np.stack([gen.masked_grf((14, 15, 13), 1.5, 6.5, 70 + i) for i in range(5)])
    bc, offs = cr.barcodes_batched(torch.from_numpy(vols).cuda(), 2, cells=True)
    d, bi, de, c = bc.numpy()
    offs = offs.cpu().numpy()
    for i in range(len(vols)):  # each image's bars are the oracle's
        o = oracle.ph(vols[i], 2)
        a, b = int(offs[i]), int(offs[i + 1])
        assert_bars_equal((d[a:b], bi[a:b], de[a:b], c[a:b]), o, i)


@pytest.mark.parametrize("name", sorted(_cavity_cases()))
def test_topdim_duality(cr, name):
    """The top dimension by Alexander duality gives the oracle's bars and the
    same full pairing as the coboundary reduction (option top_reduce), incl. essential bars of
    enclosed +inf cavities."""
    import torch
    img = _cavity_cases()[name]
    md = img.ndim - 1
    check_image(cr, img, md, ctx=name)
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    p_dual = cr.pairing(t).cpu().numpy()
    with cr.options(top_reduce=1):
        p_red = cr.pairing(t).cpu().numpy()
    assert np.array_equal(p_dual, p_red)


def test_batched_small_2d_dual(cr):
    """The one-CTA-per-image path (K7) with dimension 1 by duality equals the oracle and its own
    reduction variant, on blob images with +inf holes (enclosed and touching the border)."""
    import torch
    imgs = gen.blobs(96, 7)
    rng = np.random.default_rng(8)
    for i in range(0, 96, 3):
        y, x = rng.integers(3, 22, 2)
        imgs[i, y:y + 3, x:x + 4] = np.inf
    imgs[1, 0:3, 10:14] = np.inf
    t = torch.from_numpy(imgs).cuda()
    ba, offa = cr.barcodes_batched(t, 1, cells=True)
    assert cr.last_stats()["path"] == 5
    with cr.options(top_reduce=1):
        bb, offb = cr.barcodes_batched(t, 1, cells=True)
    pa, pb = ba.pairs.cpu().numpy(), bb.pairs.cpu().numpy()
    assert np.array_equal(pa, pb) and np.array_equal(ba.cells.cpu().numpy(), bb.cells.cpu().numpy())
    off = offa.cpu().numpy()
    assert np.array_equal(off, offb.cpu().numpy())
    for i in range(0, 96, 5):
        o = oracle.ph(imgs[i], 1)
        seg = pa[off[i]:off[i + 1]]
        assert np.array_equal(seg[:, 0], o.dim), i
        assert np.array_equal(seg[:, 1].view(np.uint32), o.birth.view(np.uint32)), i
        assert np.array_equal(seg[:, 2].view(np.uint32), o.death.view(np.uint32)), i


def test_barcodes_topdim(cr):
    """cr_barcodes_topdim (the paper's --top_dim) returns exactly the oracle's dim-(D-1) bars,
    birth cells included, with no H0 or lower-dimensional reduction."""
    import torch
    cases = dict(_cavity_cases())
    cases["c1"] = gen.config("c1")[0]
    cases["c4crop"] = gen.grf((40, 36, 44), 2.0, 4)
    for name, img in cases.items():
        D = sum(1 for v in img.shape if v > 1)
        o = oracle.ph(img, D - 1)
        sel = o.dim == D - 1
        bc = cr.barcodes_topdim(torch.from_numpy(np.ascontiguousarray(img)).cuda(), cells=True)
        d, b, e, c = bc.numpy()
        assert np.all(d == D - 1), name
        assert np.array_equal(c, o.cell[sel]), name
        assert np.array_equal(b.view(np.uint32), o.birth[sel].view(np.uint32)), name
        assert np.array_equal(e.view(np.uint32), o.death[sel].view(np.uint32)), name
        assert cr.last_stats()["path"] == 6


def test_h0_many_basins(cr):
    """H0 with more basins than one CTA's shared memory (the device-wide merge rounds, incl. the
    one-sided commit of a younger component's minimum edge) on iid noise and on integer levels."""
    rng = np.random.default_rng(60)
    for img in [rng.random((600, 640), dtype=np.float32),
                rng.integers(0, 6, (700, 560)).astype(np.float32)]:
        check_image(cr, img, 1, partner=False, ctx="many basins")
        st = cr.last_stats()
        assert st["columns"][0] > 56000, st["columns"][0]


# ---------------------------------------------------------------- configs (cropped / full)

def test_c1_full(cr):
    img, md = gen.config("c1")
    check_image(cr, img, md, ctx="c1")


def test_c2_cropped(cr):
    for n in [1 << 12, (1 << 16) + 37]:
        check_image(cr, gen.random_walk(n, seed=2), 0, ctx=n)


def test_c3_subset_batched(cr):
    import torch
    imgs = gen.blobs(64, seed=3)
    bc, off = cr.barcodes_batched(torch.from_numpy(imgs).cuda(), 1, cells=True)
    d, b, e, c = bc.numpy()
    off = off.cpu().numpy()
    for i in range(len(imgs)):
        o = oracle.ph(imgs[i], 1)
        s = slice(off[i], off[i + 1])
        assert_bars_equal((d[s], b[s], e[s], c[s]), o, ctx=i)
        if i < 8:
            check_image(cr, imgs[i], 1, ctx=("c3", i))


def test_c4_cropped(cr):
    v = gen.grf((40, 44, 36), 2.0, 4)
    check_image(cr, v, 2, ctx="c4-crop")


def test_c5_cropped_ball(cr):
    v = gen.masked_grf((48, 48, 48), 3.0, 22.0, 5)
    check_image(cr, v, 2, ctx="c5-crop")


def test_batched_1d_and_3d(cr):
    import torch
    xs = np.stack([gen.small_int_image((9,), 3, seed=s) for s in range(50)])
    bc, off = cr.barcodes_batched(torch.from_numpy(xs).cuda(), 0, cells=True)
    d, b, e, c = bc.numpy()
    off = off.cpu().numpy()
    for i in range(len(xs)):
        s = slice(off[i], off[i + 1])
        assert_bars_equal((d[s], b[s], e[s], c[s]), oracle.ph(xs[i], 0), ctx=i)
    vs = np.stack([gen.small_int_image((3, 4, 5), 4, seed=100 + s, inf_frac=0.1) for s in range(10)])
    bc, off = cr.barcodes_batched(torch.from_numpy(vs).cuda(), 2, cells=True)
    d, b, e, c = bc.numpy()
    off = off.cpu().numpy()
    for i in range(len(vs)):
        s = slice(off[i], off[i + 1])
        assert_bars_equal((d[s], b[s], e[s], c[s]), oracle.ph(vs[i], 2), ctx=i)


def test_edge_cases(cr):
    import torch
    # single voxel, all +inf, -0.0, -inf, FLT_MAX
    check_image(cr, np.array([[[5.0]]], np.float32), 2)
    check_image(cr, np.full((3, 4), np.inf, np.float32), 1)
    check_image(cr, np.array([[0.0, -0.0], [-0.0, 1.0]], np.float32), 1)
    check_image(cr, np.array([[-np.inf, 1, 3.4e38], [2, -np.inf, 0]], np.float32), 1)
    # NaN -> EINVAL
    with pytest.raises(cr.CrError) as ei:
        cr.barcodes(torch.tensor([1.0, float("nan")], device="cuda"), 0)
    assert ei.value.status == cr.CR_EINVAL
    with pytest.raises(cr.CrError) as ei:
        cr.barcodes(torch.tensor([[1.0, float("nan")], [0.0, 2.0]], device="cuda"), 1)
    assert ei.value.status == cr.CR_EINVAL
    # capacity too small -> ERANGE with the needed count
    t = torch.from_numpy(gen.iid_uniform((16, 16), 1)).cuda()
    need = len(cr.barcodes(t, 1).pairs)
    with pytest.raises(cr.CrError) as ei:
        cr.barcodes(t, 1, capacity=need - 1)
    assert ei.value.status == cr.CR_ERANGE


def test_host_entry_point(cr):
    img = gen.iid_uniform((40, 30), 9)
    bc = cr.barcodes_host(img, 1, cells=True)
    d, b, e, c = bc.numpy()
    assert_bars_equal((d, b, e, c), oracle.ph(img, 1))


# ---------------------------------------------------------------- 1D tile path edge cases

def _series_cases():
    rng = np.random.default_rng(99)
    n = 3 * 4096 + 17
    cases = {
        "walk": gen.random_walk(5 * 4096 + 3, seed=11),
        "stairs_up": (np.arange(n) // 2 + (np.arange(n) % 2) * 7.5).astype(np.float32),
        "stairs_down": (-(np.arange(n) // 2) + (np.arange(n) % 2) * 7.5).astype(np.float32),
        "monotone": np.arange(n, dtype=np.float32),
        "monotone_down": -np.arange(n, dtype=np.float32),
        "constant": np.zeros(n, np.float32),
        "levels3": rng.integers(0, 3, n).astype(np.float32),
        "plateaus": np.repeat(rng.integers(0, 6, n // 37 + 1), 37)[:n].astype(np.float32),
        "one": np.array([4.0], np.float32),
        "two": np.array([4.0, 1.0], np.float32),
        "tile": gen.random_walk(4096, seed=3),
        "tile_plus1": gen.random_walk(4097, seed=3),
        # adversarial for tile contraction: minima getting older while barriers rise (every
        # merge needs the far left), and minima getting younger while barriers rise
        "adv_desc_min_asc_bar": np.where(np.arange(n) % 2 == 0, -np.arange(n),
                                         np.arange(n)).astype(np.float32),
        "adv_asc_min_asc_bar": np.where(np.arange(n) % 2 == 0, np.arange(n),
                                        np.arange(n) + 100000).astype(np.float32),
        # long plateau across tile boundaries: a basin undecided in its tile dies at zero
        # persistence later (a hole in the staged output)
        "plateau_across_tiles": np.concatenate([[5.0], np.full(9000, 3.0), [1.0], np.full(5000, 3.0),
                                                [0.5]]).astype(np.float32),
        "vee": np.abs(np.arange(n) - n // 2).astype(np.float32),
        "peak": -np.abs(np.arange(n) - n // 2).astype(np.float32),
    }
    g = gen.random_walk(4 * 4096, seed=5)
    g[[0, 4095, 4096, 8191, 8192, 9000, 9001, 9002, 16383]] = np.inf
    cases["inf_at_tile_edges"] = g
    g = gen.random_walk(3 * 4096 + 5, seed=7)  # +inf at warp-region (512) and float4 edges
    g[[1, 511, 512, 513, 1023, 1024, 1536, 2047, 2048, 4094, 4095, 4096, 4100, 6143]] = np.inf
    cases["inf_at_warp_edges"] = g
    cases["walk_unaligned"] = gen.random_walk(2 * 4096 + 1, seed=12)[1:]
    h = gen.random_walk(20000, seed=6)
    h[rng.random(20000) < 0.3] = np.inf
    cases["inf_30pct"] = h
    cases["all_inf"] = np.full(5000, np.inf, np.float32)
    return cases


@pytest.mark.parametrize("name", sorted(_series_cases()))
def test_1d_tile_path_cases(cr, name):
    x = _series_cases()[name]
    check_image(cr, x, 0, partner=(len(x) < 20000), ctx=name)


def test_1d_tile_vs_tree_large(cr):
    import torch
    x = gen.random_walk(1 << 20, seed=8)
    t = torch.from_numpy(x).cuda()
    a = cr.barcodes(t, 0, cells=True).numpy()
    assert cr.last_stats()["path"] == 1
    with cr.options(**{"1d_tree": 1}):
        b = cr.barcodes(t, 0, cells=True).numpy()
    for u, v in zip(a, b):
        assert np.array_equal(np.asarray(u).view(np.uint32), np.asarray(v).view(np.uint32))
    assert_bars_equal(a, oracle.ph(x, 0))


def test_batched_small_2d_vs_oracle_and_stacked(cr):
    """One-CTA-per-image kernel (K7) = oracle = stacked device-wide path, with ties and +inf."""
    import torch
    imgs = gen.blobs(300, seed=31)
    rng = np.random.default_rng(5)
    imgs[rng.random(imgs.shape) < 0.02] = np.inf
    imgs[:10] = np.floor(imgs[:10] / 64)  # heavy ties
    t = torch.from_numpy(imgs).cuda()
    bc, off = cr.barcodes_batched(t, 1, cells=True)
    assert cr.last_stats()["path"] == 5
    a = bc.numpy()
    offa = off.cpu().numpy()
    for i in range(len(imgs)):
        s = slice(offa[i], offa[i + 1])
        assert_bars_equal(tuple(x[s] for x in a), oracle.ph(imgs[i], 1), ctx=i)
    with cr.options(force_general=1):
        bc2, off2 = cr.barcodes_batched(t, 1, cells=True)
        assert cr.last_stats()["path"] == 3
    assert np.array_equal(off2.cpu().numpy(), offa)
    for u, v in zip(a, bc2.numpy()):
        assert np.array_equal(np.asarray(u).view(np.uint32), np.asarray(v).view(np.uint32))
    # maxdim 0 and 1xN / Nx1 shapes
    for shp in [(5, 1, 9), (5, 9, 1), (7, 6, 5)]:
        x = gen.small_int_image(shp, 4, seed=sum(shp))
        bc3, off3 = cr.barcodes_batched(torch.from_numpy(x).cuda(), 0, cells=True)
        d3 = bc3.numpy()
        o3 = off3.cpu().numpy()
        for i in range(shp[0]):
            s = slice(o3[i], o3[i + 1])
            assert_bars_equal(tuple(y[s] for y in d3), oracle.ph(x[i], 0), ctx=(shp, i))


# ---------------------------------------------------------------- NEXT-2 / NEXT-4

def test_death_cells_and_coords(cr):
    """Death locations (location="death") equal the oracle's partner of each
    bar's birth cell; cell_coords decodes kidx."""
    import torch
    for img, md in [(gen.small_int_image((13, 17), 4, seed=31, inf_frac=0.05), 1),
                    (gen.masked_grf((12, 14, 16), 2.0, 7.0, 32), 2),
                    (gen.random_walk(9000, seed=33), 0)]:
        o = oracle.ph(img, md, partner=True)
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        bc = cr.barcodes(t, md, cells=True)
        births = bc.cells.cpu().numpy().view(np.uint32)
        deaths = cr.death_cells(t, bc.cells).cpu().numpy().view(np.uint32)
        assert np.array_equal(deaths, o.partner[births])
        ess = deaths == 0xFFFFFFFF
        assert np.array_equal(ess, np.isinf(bc.numpy()[2]))
        K, v = cr.cell_coords(births, img.shape)
        s = [1] * (3 - img.ndim) + list(img.shape)
        KX, KY = 2 * s[2] - 1, 2 * s[1] - 1
        assert np.array_equal((K[:, 2] * KY + K[:, 1]) * KX + K[:, 0], births.astype(np.int64))
        assert np.array_equal(v, K // 2)


def test_lifetime_image(cr):
    """Lifetime-enhanced image equals a numpy scatter-max of the oracle's bars
    at their birth cells' base voxels; the TTK 3x3 example puts lifetime 9 in channel 2."""
    import torch
    g = json.load(open(os.path.join(GOLDEN, "ttk_3x3.json")))
    img = np.array(g["image"], np.float32)
    li = cr.lifetime_image(torch.from_numpy(img).cuda(), 1, inf_value=9.0).cpu().numpy()
    assert li.shape == (3, 3, 3) and np.array_equal(li[0], img)
    assert li[2].max() == 9.0 and li[1].max() == 9.0  # H1 bar [0, 9); essential H0 [0, inf->9)
    imgs = np.stack([gen.small_int_image((11, 9), 5, seed=40 + i, inf_frac=0.05) for i in range(6)])
    out = cr.lifetime_image(torch.from_numpy(imgs).cuda(), 1, inf_value=10.0, batched=True)
    out = out.cpu().numpy()
    for b in range(len(imgs)):
        o = oracle.ph(imgs[b], 1)
        ref = np.zeros((3,) + imgs[b].shape, np.float32)
        ref[0] = imgs[b]
        KX = 2 * imgs[b].shape[1] - 1
        for d, bi, de, c in zip(o.dim, o.birth, o.death, o.cell):
            life = (10.0 if np.isinf(de) else de) - bi
            y, x = (int(c) // KX) // 2, (int(c) % KX) // 2
            ref[1 + d, y, x] = max(ref[1 + d, y, x], life)
        assert np.array_equal(out[b], ref), b


# ---------------------------------------------------------------- float64 images

def _check_f64(cr, img, maxdim, ctx=""):
    import torch
    img = np.ascontiguousarray(img, np.float64)
    o = oracle.ph(img, maxdim, dtype=np.float64)
    bc = cr.barcodes_f64(torch.from_numpy(img).cuda(), maxdim, cells=True)
    d, b, e, c = bc.numpy()
    assert len(d) == len(o.dim), (ctx, len(d), len(o.dim))
    assert np.array_equal(d, o.dim), ctx
    assert np.array_equal(c, o.cell), ctx
    assert np.array_equal(b.view(np.uint64), o.birth.view(np.uint64)), ctx
    assert np.array_equal(e.view(np.uint64), o.death.view(np.uint64)), ctx
    return o


def test_barcodes_f64_rank_path(cr):
    """Values that differ below float32 resolution (all round to the same float32) -> rank path."""
    step = 2.0 ** -40
    cases = [
        ("1d_small", (257,)), ("1d_tiles", (20011,)), ("2d", (61, 47)), ("2d_wide", (7, 3001)),
        ("3d", (13, 17, 19)),
    ]
    for s, (name, shape) in enumerate(cases):
        k = gen.small_int_image(shape, 50, seed=1200 + s, inf_frac=0.1 if s % 2 else 0.0)
        img = 1.0 + k.astype(np.float64) * step
        o = _check_f64(cr, img, 2, ctx=name)
        if s % 2 == 0:
            assert len(o.dim) > 1, name  # the sub-float32 structure is really there


def test_f64_rank_sort_tile_boundaries(cr):
    """The ranking's radix sort (64-bit keys, 32-bit indices, 8 passes; tiles of 3072 keys, see
    DESIGN.md §K3; one tile takes the single-tile path) at tile boundaries and with long runs of
    equal values: sub-float32 distinct doubles with ties, 1D (the tiles path) and 2D, against the
    oracle."""
    step = 2.0 ** -38
    for s, n in enumerate([3071, 3072, 3073, 6145, 3 * 3072 + 17, 4097]):
        k = gen.small_int_image((n,), 700, seed=1300 + s, inf_frac=0.05 if s % 2 else 0.0)
        _check_f64(cr, 1.0 + k.astype(np.float64) * step, 1, ctx=("1d", n))
    k = gen.small_int_image((67, 129), 3000, seed=1310)
    _check_f64(cr, -2.0 - k.astype(np.float64) * step, 1, ctx="2d negative")


def test_barcodes_f64_iid_and_specials(cr):
    rng = np.random.default_rng(4242)
    for shape in [(5000,), (90, 110), (16, 18, 20)]:
        _check_f64(cr, rng.random(shape), 2, ctx=shape)            # distinct doubles
        _check_f64(cr, rng.standard_normal(shape) * 1e300, 2, ctx=shape)
    img = rng.random((40, 41))
    img[3, 4], img[5, 6], img[7, 8] = -np.inf, -0.0, 0.0
    img[10:14, 10:14] = np.inf
    _check_f64(cr, img, 1, ctx="specials")
    # the exact (cast) path: float32-representable values
    f = gen.iid_uniform((33, 35), seed=3).astype(np.float64)
    o = _check_f64(cr, f, 1, ctx="exact")
    g = oracle.ph(f.astype(np.float32), 1)
    assert np.array_equal(o.birth, g.birth.astype(np.float64))
    import torch
    with pytest.raises(cr.CrError):
        cr.barcodes_f64(torch.tensor([1.0, float("nan")], dtype=torch.float64).cuda(), 0)
    with pytest.raises(TypeError):
        cr.barcodes_f64(torch.zeros(4, device="cuda"), 0)


def test_stats_counters_match_definitions(cr):
    """The pairing-determined counters of cr_stats equal their definitions:
    finite cells and apparent (UP) cells per dimension and the H0 basins from tests/apparent.py,
    bars per dimension from the oracle -- for the fused K1+K2 kernel and the former pair."""
    import torch
    import apparent as ap
    imgs = [gen.masked_grf((23, 27, 31), 2.0, 11.0, 81),
            gen.small_int_image((9, 40, 33), 3, seed=82, inf_frac=0.1),
            gen.iid_uniform((61, 47), seed=83),
            gen.small_int_image((50, 45), 5, seed=84, inf_frac=0.05)]
    for k, img in enumerate(imgs):
        exp = ap.counts(img)
        o = oracle.ph(img, img.ndim - 1, partner=True)
        # K5 columns of dimension d (cohomology, d < D-1): d-cells that are neither apparent nor
        # the death cell of a (d-1)-pair -- from the oracle's pairing and the definition
        up, dims, finite = ap.apparent_up(img)
        part = o.partner.astype(np.int64)
        flat_dims = dims.ravel()
        app_any = up.ravel().copy()
        for s_, t_ in ap.pairs_up(img):
            app_any[t_] = True
        is_cell = finite.ravel()
        paired = (part < len(part))
        partner_dim = np.where(paired, flat_dims[np.minimum(part, len(part) - 1)], -1)
        cols_exp = [int(np.count_nonzero(is_cell & (flat_dims == d) & ~app_any &
                                         ~(paired & (partner_dim == d - 1))))
                    for d in range(4)]
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        for var in ("",):
            cr.barcodes(t, img.ndim - 1)
            st = cr.last_stats()
            assert list(st["cells"]) == exp["cells"], (k, var, st["cells"], exp["cells"])
            assert list(st["apparent"])[:3] == exp["apparent"][:3], (k, var, st["apparent"], exp)
            assert st["columns"][0] == exp["basins"], (k, var, st["columns"][0], exp["basins"])
            nb = [int(np.count_nonzero(o.dim == d)) for d in range(img.ndim)]
            assert list(st["pairs"])[:img.ndim] == nb, (k, var, st["pairs"], nb)
            for d in range(1, img.ndim - 1):  # the top dimension runs by duality (roots)
                assert st["columns"][d] == cols_exp[d], (k, var, d, st["columns"], cols_exp)


def test_k5_schedule_independence(cr):
    """The dims >= 1 reduction's pairing does not depend on its schedule (the commit rule of
    DESIGN.md §6): one resident block per SM (fewer columns in flight), and pseudo-random delays
    of up to 2 / 50 us injected before commits, all give the oracle's pairing."""
    import torch
    imgs = [gen.masked_grf((20, 22, 24), 2.0, 10.0, 91),
            gen.small_int_image((9, 16, 13), 3, seed=92, inf_frac=0.1),
            gen.grf((18, 17, 19), 1.5, 93),
            gen.grf((40, 44, 36), 2.0, 94)]
    knobs = [{}, {"k5_blocks_per_sm": 1}, {"k5_jitter_ns": 2000},
             {"k5_jitter_ns": 50000, "k5_blocks_per_sm": 2}]
    for k, img in enumerate(imgs):
        o = oracle.ph(img, 2, partner=True)
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        for kn in knobs:
            with cr.options(top_reduce=1, **kn):  # both dims by the reduction
                p = cr.pairing(t).cpu().numpy().view(np.uint32)
            assert np.array_equal(p, o.partner), (k, kn, np.flatnonzero(p != o.partner)[:10])


def test_k7_fuzz_shapes(cr):
    """Batches of small 2D images through the one-CTA-per-image path (K7) on random shapes from
    1-wide to 32 x 32 (the last takes the reduction variant), with and without +inf masks: each
    image's bars equal the oracle's."""
    import torch
    rng = np.random.default_rng(2024)
    for t in range(40):
        ny, nx = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        if t == 0:
            ny = nx = 32
        B = int(rng.integers(1, 30))
        imgs = np.stack([gen.small_int_image((ny, nx), int(rng.integers(2, 9)),
                                             seed=int(rng.integers(1 << 30)),
                                             inf_frac=[0.0, 0.05, 0.3][t % 3]) for _ in range(B)])
        bc, off = cr.barcodes_batched(torch.from_numpy(imgs).cuda(), 1)
        d, b, e, _ = bc.numpy()
        off = off.cpu().numpy()
        for i in range(B):
            o = oracle.ph(imgs[i], 1)
            s = slice(off[i], off[i + 1])
            got = sorted(zip(d[s].tolist(), b[s].tolist(), e[s].tolist()))
            exp = sorted(zip(o.dim.tolist(), o.birth.tolist(), o.death.tolist()))
            assert got == exp, (t, (ny, nx), i)
