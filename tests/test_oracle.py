"""Pins for the CPU oracle (``-m "not gpu"``).

The oracle (oracle/cr_oracle.cpp) is checked against things other than itself:
the paper's worked examples (tests/golden/, cited), closed forms, brute-force persistent
Betti numbers from GF(2) ranks, an independent cohomology reduction, the elder-rule
union-find, the 1D closed form and the Euler-characteristic identity (tests/bruteforce.py).
A plausible mistake (dropped facet, wrong tie-break, wrong sign of a birth comparison,
transposed axis) fails at least one of them.
"""
import itertools
import json
import math
import os
from collections import Counter

import numpy as np
import pytest

import oracle
import bruteforce as bf
from workloads import generators as gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
INF = math.inf


def _multiset(res, maxdim=3):
    return Counter((int(d), float(b), float(e)) for d, b, e in
                   zip(res.dim, res.birth, res.death) if d <= maxdim)


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        g = json.load(f)
    exp = Counter((int(d), float(b), INF if e == "inf" else float(e)) for d, b, e in g["expected"])
    return g, exp


# ---------------------------------------------------------------- paper's worked examples

def test_ttk_counterexample_golden():
    g, exp = _load("ttk_3x3.json")
    res = oracle.ph(np.array(g["image"], np.float32), g["maxdim"])
    assert _multiset(res) == exp
    assert bf.barcode_by_ranks(np.array(g["image"], np.float32), 1) == exp


def test_fig2_h0_golden():
    g, exp = _load("fig2_h0.json")
    res = oracle.ph(np.array(g["image"], np.float32), g["maxdim"])
    assert _multiset(res) == exp


def test_sin_example_counts():
    with open(os.path.join(GOLDEN, "sin_1d.json")) as f:
        g = json.load(f)
    x = np.linspace(0, 4 * np.pi, g["n"])
    img = (np.sin(x) + 0.1 * x).astype(np.float32)
    res = oracle.ph(img, 1)
    ess = int(np.sum(np.isinf(res.death)))
    fin = int(np.sum(~np.isinf(res.death)))
    assert (ess, fin) == (g["expected_essential"], g["expected_finite"])
    assert float(res.birth[np.isinf(res.death)][0]) == float(img.min())
    assert _multiset(res) == bf.barcode_by_ranks(img, 1)


# ---------------------------------------------------------------- closed forms

def test_constant_and_two_voxels():
    assert _multiset(oracle.ph(np.full((4, 5), 2.5, np.float32), 1)) == Counter({(0, 2.5, INF): 1})
    assert _multiset(oracle.ph(np.array([3, 7], np.float32), 0)) == Counter({(0, 3.0, INF): 1})
    assert _multiset(oracle.ph(np.array([[[5.0]]], np.float32), 2)) == Counter({(0, 5.0, INF): 1})


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_checkerboard(n):
    img = (np.add.outer(np.arange(n), np.arange(n)) % 2).astype(np.float32)
    exp = Counter({(0, 0.0, INF): 1})
    k = (n * n + 1) // 2 - 1
    if k:
        exp[(0, 0.0, 1.0)] = k
    assert _multiset(oracle.ph(img, 1)) == exp


def test_void_and_tunnel_3d():
    v = np.zeros((3, 3, 3), np.float32)
    v[1, 1, 1] = 9
    assert _multiset(oracle.ph(v, 2)) == Counter({(0, 0.0, INF): 1, (2, 0.0, 9.0): 1})
    t = np.zeros((3, 3, 3), np.float32)
    t[:, 1, 1] = 9  # a tunnel along z through the cube
    assert _multiset(oracle.ph(t, 2)) == Counter({(0, 0.0, INF): 1, (1, 0.0, 9.0): 1})


def test_annulus():
    img = np.full((5, 5), 2.0, np.float32)  # outside o = 2
    img[1:4, 1:4] = 0.0                      # ring a = 0
    img[2, 2] = 5.0                          # hole h = 5
    assert _multiset(oracle.ph(img, 1)) == Counter({(0, 0.0, INF): 1, (1, 0.0, 5.0): 1})


def test_inf_outside_domain_absent():
    # +inf voxels are outside the domain: two components, each essential (reading R5)
    img = np.array([1, 4, np.inf, 2, 0], np.float32)
    assert _multiset(oracle.ph(img, 0)) == Counter({(0, 1.0, INF): 1, (0, 0.0, INF): 1})
    allinf = np.full((3, 3), np.inf, np.float32)
    r = oracle.ph(allinf, 1, partner=True)
    assert len(r.dim) == 0 and np.all(r.partner == oracle.PARTNER_ABSENT)


def test_negative_zero_canonicalised():
    a = np.array([[0.0, 1.0], [1.0, -0.0]], np.float32)
    b = np.array([[0.0, 1.0], [1.0, 0.0]], np.float32)
    ra, rb = oracle.ph(a, 1, partner=True), oracle.ph(b, 1, partner=True)
    assert np.array_equal(ra.partner, rb.partner)
    assert np.array_equal(ra.birth.view(np.uint32), rb.birth.view(np.uint32))


def test_invalid_inputs():
    with pytest.raises(ValueError):
        oracle.ph(np.array([1.0, np.nan], np.float32), 0)
    with pytest.raises(ValueError):
        oracle.ph(np.zeros((2, 2), np.float32), -1)


# ---------------------------------------------------------------- births

def test_births_match_definition():
    img = gen.small_int_image((3, 4, 5), 7, seed=11, inf_frac=0.1)
    B = oracle.births(img)
    KZ, KY, KX = B.shape
    cells = bf.enumerate_cells(img)
    seen = set()
    for c in cells:
        z, y, x = divmod(c["kidx"], KY * KX)[0], (c["kidx"] // KX) % KY, c["kidx"] % KX
        assert B[z, y, x] == np.float32(c["birth"])
        seen.add(c["kidx"])
    flat = B.reshape(-1)
    absent = [k for k in range(flat.size) if k not in seen]
    assert all(flat[k] == np.inf for k in absent)


def test_cell_counts_closed_form():
    img = np.zeros((3, 4, 5), np.float32)
    cells = bf.enumerate_cells(img)
    cnt = Counter(c["dim"] for c in cells)
    nx, ny, nz = 5, 4, 3
    assert cnt[0] == nx * ny * nz
    assert cnt[1] == (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
    assert cnt[2] == (nx - 1) * (ny - 1) * nz + (nx - 1) * ny * (nz - 1) + nx * (ny - 1) * (nz - 1)
    assert cnt[3] == (nx - 1) * (ny - 1) * (nz - 1)
    assert oracle.max_pairs((3, 4, 5), 3) == sum(cnt.values())


# ---------------------------------------------------------------- exhaustive and fuzz

def _check_against_bruteforce(img, maxdim=3, pairing=True):
    r_tw = oracle.ph(img, maxdim, twist=True, partner=True)
    assert _multiset(r_tw) == bf.barcode_by_ranks(img, maxdim), img
    if pairing:
        r_nt = oracle.ph(img, maxdim, twist=False, partner=True)
        assert np.array_equal(r_tw.partner, r_nt.partner)
        coh = bf.cohomology_pairing(img)
        P = r_tw.partner
        for k, p in coh.items():
            assert P[k] == (oracle.PARTNER_ESSENTIAL if p is None else p), (img, k)
    return r_tw


def test_exhaustive_2x2_levels3():
    for vals in itertools.product([0, 1, 2], repeat=4):
        _check_against_bruteforce(np.array(vals, np.float32).reshape(2, 2), 1)


def test_exhaustive_3x3_binary():
    for vals in itertools.product([0, 1], repeat=9):
        _check_against_bruteforce(np.array(vals, np.float32).reshape(3, 3), 1,
                                  pairing=(sum(vals) % 5 == 0))


def test_exhaustive_2x2x2_binary():
    for vals in itertools.product([0, 1], repeat=8):
        _check_against_bruteforce(np.array(vals, np.float32).reshape(2, 2, 2), 2)


def test_exhaustive_1d_len8_levels3():
    for i, vals in enumerate(itertools.product([0, 1, 2], repeat=8)):
        img = np.array(vals, np.float32)
        r = oracle.ph(img, 0, partner=True)
        # elder-rule closed form on the full pairing of vertices
        ref = bf.elder_1d(img)
        for v, e in ref.items():
            exp = oracle.PARTNER_ESSENTIAL if e is None else 2 * e + 1
            assert r.partner[2 * v] == exp, (vals, v)
        if i % 37 == 0:
            assert _multiset(r) == bf.barcode_by_ranks(img, 0)


def test_fuzz_random_small():
    """>= 1000 random images up to 5x5x5, values {0..4}, some with +inf masks."""
    rng = np.random.default_rng(12345)
    n_done = 0
    for t in range(1000):
        nd = int(rng.integers(1, 4))
        if nd == 3:
            shape = tuple(int(s) for s in rng.integers(1, 4, size=3))
        elif nd == 2:
            shape = tuple(int(s) for s in rng.integers(1, 6, size=2))
        else:
            shape = (int(rng.integers(1, 13)),)
        img = gen.small_int_image(shape, 5, seed=int(rng.integers(1 << 30)),
                                  inf_frac=0.15 if t % 3 == 0 else 0.0)
        _check_against_bruteforce(img, 2, pairing=(t % 4 == 0))
        n_done += 1
    assert n_done == 1000


def test_fuzz_larger_3d_pairing():
    for s in range(6):
        img = gen.small_int_image((4, 5, 5), 5, seed=100 + s, inf_frac=0.1 if s % 2 else 0.0)
        _check_against_bruteforce(img, 2)


# ---------------------------------------------------------------- invariants

def test_h0_pairing_union_find():
    for s in range(20):
        shape = [(6, 7), (3, 4, 5), (17,)][s % 3]
        img = gen.small_int_image(shape, 6, seed=200 + s, inf_frac=0.1 if s % 2 else 0.0)
        r = oracle.ph(img, 0, partner=True)
        for v, e in bf.union_find_h0(img).items():
            assert r.partner[v] == (oracle.PARTNER_ESSENTIAL if e is None else e)


def test_elder_1d_random_walk():
    x = gen.random_walk(3000, seed=7)
    r = oracle.ph(x, 0, partner=True)
    ref = bf.elder_1d(x)
    got = np.array([r.partner[2 * i] for i in range(len(x))], np.int64)
    exp = np.array([oracle.PARTNER_ESSENTIAL if e is None else 2 * e + 1 for e in
                    (ref[i] for i in range(len(x)))], np.int64)
    assert np.array_equal(got, exp)


def test_euler_and_betti_curves():
    for s in range(12):
        shape = [(5, 5), (3, 3, 4), (11,)][s % 3]
        img = gen.small_int_image(shape, 5, seed=300 + s, inf_frac=0.2 if s % 2 else 0.0)
        r = oracle.ph(img, 3)
        assert bf.euler_curve_ok(img, r.dim, r.birth, r.death)
        for t, betti in bf.betti_curve(img).items():
            alive = [sum(1 for d, b, e in zip(r.dim, r.birth, r.death) if d == dd and b <= t < e)
                     for dd in range(3)]
            assert tuple(alive) == betti


def test_metamorphic_monotone_map_keeps_pairing():
    img = gen.iid_uniform((9, 11), seed=5)
    r1 = oracle.ph(img, 1, partner=True)
    r2 = oracle.ph(img * np.float32(2.0), 1, partner=True)
    assert np.array_equal(r1.partner, r2.partner)
    assert np.array_equal(r1.birth * 2, r2.birth)
    k = gen.small_int_image((6, 6), 9, seed=9)
    a, b = oracle.ph(k, 1), oracle.ph(k + np.float32(3), 1)
    assert Counter((d, x + 3, y + 3) for d, x, y in zip(a.dim, a.birth, a.death)) == _multiset(b)


def test_contractible_domain_one_essential():
    for shape in [(7,), (6, 5), (4, 3, 5)]:
        r = oracle.ph(gen.iid_uniform(shape, seed=3), 2)
        assert int(np.sum(np.isinf(r.death))) == 1
        assert int(r.dim[np.isinf(r.death)][0]) == 0


# ---------------------------------------------------------------- float64
#
# The paper's implementation stores pixel values as doubles.  oracle_ph_f64 runs
# the same steps in double precision; these pins use values that differ BELOW float32
# resolution (1 + k*2^-40 all round to 1.0f), so a float64 path that rounded through float32
# anywhere would collapse them and fail.

def _tiny(k, base=1.0, step=2.0 ** -40):
    return base + np.asarray(k, np.float64) * step


def test_f64_values_below_f32_resolution():
    k = np.arange(6, dtype=np.float64)
    assert np.all(_tiny(k).astype(np.float32) == np.float32(1.0))
    img = _tiny(np.array([3, 0, 2, 1, 5, 4]))
    r = oracle.ph(img, 0, dtype=np.float64)
    assert r.birth.dtype == np.float64
    # f32 collapses everything to one constant component; f64 sees three minima
    assert len(oracle.ph(img, 0).dim) == 1
    exp = Counter([(0, _tiny(0), INF), (0, _tiny(1), _tiny(2)), (0, _tiny(4), _tiny(5))])
    assert _multiset(r) == exp


def test_f64_exhaustive_2x2_levels3():
    for vals in itertools.product([0, 1, 2], repeat=4):
        img = _tiny(np.array(vals).reshape(2, 2))
        r = oracle.ph(img, 1, partner=True, dtype=np.float64)
        assert _multiset(r) == bf.barcode_by_ranks(img, 1), vals


def test_f64_fuzz_against_bruteforce():
    rng = np.random.default_rng(777)
    for t in range(150):
        nd = int(rng.integers(1, 4))
        shape = {1: (int(rng.integers(1, 12)),),
                 2: tuple(int(s) for s in rng.integers(1, 5, size=2)),
                 3: tuple(int(s) for s in rng.integers(1, 4, size=3))}[nd]
        img = _tiny(rng.integers(0, 5, size=shape))
        if t % 3 == 0:
            img[rng.random(shape) < 0.15] = np.inf
        r = oracle.ph(img, 2, partner=(t % 4 == 0), dtype=np.float64)
        assert _multiset(r) == bf.barcode_by_ranks(img, 2), (t, img)
        if t % 4 == 0:
            for kk, p in bf.cohomology_pairing(img).items():
                assert r.partner[kk] == (oracle.PARTNER_ESSENTIAL if p is None else p)


def test_f64_pairing_equals_integer_levels():
    """Strictly increasing g: pairing of g(k) in float64 == pairing of k (exact in float32)."""
    for s, shape in enumerate([(6, 7), (3, 4, 5), (40,)]):
        k = gen.small_int_image(shape, 9, seed=900 + s, inf_frac=0.1 if s % 2 else 0.0)
        r32 = oracle.ph(k, 2, partner=True)
        r64 = oracle.ph(_tiny(k.astype(np.float64)), 2, partner=True, dtype=np.float64)
        assert np.array_equal(r32.partner, r64.partner)
        fin = np.isfinite(r32.death)
        assert np.array_equal(_tiny(r32.birth.astype(np.float64)), r64.birth)
        assert np.array_equal(_tiny(r32.death[fin].astype(np.float64)), r64.death[fin])


def test_f64_elder_1d_and_union_find():
    x = gen.random_walk(2000, seed=8).astype(np.float64) * 2.0 ** -30 + 1.0
    r = oracle.ph(x, 0, partner=True, dtype=np.float64)
    ref = bf.elder_1d(x)
    for i in range(len(x)):
        assert r.partner[2 * i] == (oracle.PARTNER_ESSENTIAL if ref[i] is None else 2 * ref[i] + 1)
    img = _tiny(gen.small_int_image((5, 6), 7, seed=4))
    r = oracle.ph(img, 0, partner=True, dtype=np.float64)
    for v, e in bf.union_find_h0(img).items():
        assert r.partner[v] == (oracle.PARTNER_ESSENTIAL if e is None else e)


def test_f64_births_and_invalid():
    img = _tiny(gen.small_int_image((3, 4, 5), 7, seed=12))
    B = oracle.births(img, dtype=np.float64)
    assert B.dtype == np.float64
    KZ, KY, KX = B.shape
    for c in bf.enumerate_cells(img):
        assert B.reshape(-1)[c["kidx"]] == c["birth"]
    with pytest.raises(ValueError):
        oracle.ph(np.array([1.0, np.nan]), 0, dtype=np.float64)
    a = oracle.ph(np.array([-0.0, 1.0, 0.0]), 0, partner=True, dtype=np.float64)
    b = oracle.ph(np.array([0.0, 1.0, 0.0]), 0, partner=True, dtype=np.float64)
    assert np.array_equal(a.partner, b.partner)


# ---------------------------------------------------------------- apparent pairs

def test_apparent_pairs_in_oracle_pairing():
    """Every apparent pair by its definition (tests/apparent.py) is a pair of the
    oracle's full pairing with death == birth (App. A.4), on random 1D/2D/3D images with +inf
    masks and ties; the per-dimension finite-cell counts match the closed-form grid counts."""
    import apparent as ap
    rng = np.random.default_rng(4545)
    for t in range(120):
        nd = int(rng.integers(1, 4))
        shape = tuple(int(s) for s in rng.integers(1, 8 if nd < 3 else 5, size=nd))
        img = gen.small_int_image(shape, 4, seed=int(rng.integers(1 << 30)),
                                  inf_frac=0.15 if t % 3 == 0 else 0.0)
        o = oracle.ph(img, 2, partner=True)
        b = ap.khalimsky_births(img).ravel()
        for s, u in ap.pairs_up(img):
            assert o.partner[s] == u and o.partner[u] == s, (t, shape, s, u)
            assert b[s] == b[u], (t, s, u)
        if not np.isinf(img).any():
            c = ap.counts(img)["cells"]
            full = [1, 1, 1]
            full[3 - nd:] = shape
            nz, ny, nx = full
            exp = [nz * ny * nx,
                   (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1),
                   (nx - 1) * (ny - 1) * nz + (nx - 1) * ny * (nz - 1) + nx * (ny - 1) * (nz - 1),
                   (nx - 1) * (ny - 1) * (nz - 1)]
            assert c == exp, (shape, c, exp)
