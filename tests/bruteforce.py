"""Independent checkers that pin the oracle (test-only, pure Python, tiny inputs).

None of this shares code with ``oracle/cr_oracle.cpp`` or the CUDA path.  Cells are
enumerated here the way the paper describes them -- an anchor voxel plus the set of
spanned axes, i.e. the tuple (x, y, z, m, d) of PAPER.md:90-107 -- and only mapped to
the Khalimsky index kidx (reading R1) where a total order or a pairing is compared.

* ``barcode_by_ranks``  -- the barcode as a multiset from persistent Betti numbers
  beta^{i,j} = dim Z(K_i) - dim(Z(K_i) & B(K_j)) computed by GF(2) ranks at every pair of
  thresholds; independent of any reduction and of any tie-break.
* ``betti_curve``       -- beta_d(t) = n_d - rk d_d - rk d_{d+1} at every threshold.
* ``cohomology_pairing`` -- the cell pairing from reducing the COboundary matrix in
  reverse filtration order with pivot = earliest coface, a different
  algorithm from the oracle's homology reduction.
* ``union_find_h0``     -- dimension-0 pairing by union-find with the elder rule
  (PAPER.md:121-128).
* ``elder_1d``          -- 1D closed form: a local minimum dies at the lower of the two
  bottleneck edges to the nearest older vertex on either side.
"""
from __future__ import annotations

import itertools
import math
from collections import Counter

import numpy as np

INF = math.inf


def _canon(img):
    a = np.asarray(img)
    # float64 images keep their precision; everything else is read as float32
    a = a.astype(np.float64) if a.dtype == np.float64 else a.astype(np.float32).astype(np.float64)
    a = np.where(a == 0.0, 0.0, a)  # -0.0 -> +0.0
    s = [1] * (3 - a.ndim) + list(a.shape)
    return a.reshape(s)  # (nz, ny, nx)


def enumerate_cells(img):
    """All finite cells: dict with 'birth', 'dim', 'verts', 'kidx', 'axes', 'anchor'."""
    a = _canon(img)
    nz, ny, nx = a.shape
    sizes = (nx, ny, nz)
    KX, KY = 2 * nx - 1, 2 * ny - 1
    cells = []
    for d in range(4):
        for axes in itertools.combinations(range(3), d):
            ext = [sizes[ax] - (1 if ax in axes else 0) for ax in range(3)]
            if min(ext) <= 0:
                continue
            for z in range(ext[2]):
                for y in range(ext[1]):
                    for x in range(ext[0]):
                        anchor = (x, y, z)
                        verts = []
                        for off in itertools.product((0, 1), repeat=d):
                            v = list(anchor)
                            for ax, o in zip(axes, off):
                                v[ax] += o
                            verts.append(tuple(v))
                        b = max(a[v[2], v[1], v[0]] for v in verts)
                        if b == INF:
                            continue  # outside the domain: absent (reading R5)
                        X = 2 * x + (1 if 0 in axes else 0)
                        Y = 2 * y + (1 if 1 in axes else 0)
                        Z = 2 * z + (1 if 2 in axes else 0)
                        cells.append(dict(birth=float(b), dim=d, verts=frozenset(verts),
                                          kidx=(Z * KY + Y) * KX + X, axes=axes, anchor=anchor))
    return cells


def _faces(cell, index_of):
    """Faces of a cell as keys into index_of: drop one spanned axis at offset 0 or 1."""
    out = []
    for ax in cell["axes"]:
        rest = tuple(a for a in cell["axes"] if a != ax)
        for o in (0, 1):
            anc = list(cell["anchor"])
            anc[ax] += o
            out.append(index_of[(tuple(anc), rest)])
    return out


def _index(cells):
    return {(c["anchor"], c["axes"]): i for i, c in enumerate(cells)}


class _Basis:
    """Incremental GF(2) row-echelon basis of int bitsets."""

    def __init__(self):
        self.piv = {}

    def add(self, v: int) -> bool:
        while v:
            h = v.bit_length() - 1
            if h in self.piv:
                v ^= self.piv[h]
            else:
                self.piv[h] = v
                return True
        return False

    def __len__(self):
        return len(self.piv)


def _rank(vectors):
    b = _Basis()
    for v in vectors:
        b.add(v)
    return len(b)


def _kernel(cols):
    """Kernel basis of the map given by `cols` (list of (combination_bit, image_bitset))."""
    piv = {}
    ker = []
    for comb, img in cols:
        while img:
            h = img.bit_length() - 1
            if h in piv:
                pc, pi = piv[h]
                img ^= pi
                comb ^= pc
            else:
                piv[h] = (comb, img)
                break
        if not img:
            ker.append(comb)
    return ker


def barcode_by_ranks(img, maxdim=3):
    """Counter of (dim, birth, death) over bars with death > birth, death = inf if essential."""
    cells = enumerate_cells(img)
    idx = _index(cells)
    by_dim = {d: [i for i, c in enumerate(cells) if c["dim"] == d] for d in range(4)}
    pos_in_dim = {}
    for d in range(4):
        for p, i in enumerate(by_dim[d]):
            pos_in_dim[i] = p
    bd = {}
    for i, c in enumerate(cells):
        v = 0
        for f in _faces(c, idx) if c["dim"] > 0 else []:
            v ^= 1 << pos_in_dim[f]
        bd[i] = v
    ts = sorted({c["birth"] for c in cells})
    m = len(ts)
    out = Counter()
    for d in range(min(maxdim, 3) + 1):
        cur = by_dim[d]
        if not cur:
            continue
        # kernel of boundary_d restricted to K_i, as bitsets over d-cells
        Z = [None] * (m + 1)
        for i in range(m + 1):
            t = ts[i - 1] if i > 0 else -INF
            cols = [(1 << pos_in_dim[c], bd[c] if d > 0 else 0) for c in cur if cells[c]["birth"] <= t]
            Z[i] = _kernel(cols)
        B = [None] * (m + 1)
        for j in range(m + 1):
            t = ts[j - 1] if j > 0 else -INF
            B[j] = [bd[c] for c in by_dim.get(d + 1, []) if cells[c]["birth"] <= t]
        rB = [_rank(B[j]) for j in range(m + 1)]

        def beta(i, j):
            if i == 0:
                return 0
            z = len(Z[i])
            return z - (z + rB[j] - _rank(Z[i] + B[j]))

        for i in range(1, m + 1):
            for j in range(i + 1, m + 1):
                mu = beta(i, j - 1) - beta(i, j) - beta(i - 1, j - 1) + beta(i - 1, j)
                assert mu >= 0
                if mu:
                    out[(d, ts[i - 1], ts[j - 1])] += mu
            mu = beta(i, m) - beta(i - 1, m)
            assert mu >= 0
            if mu:
                out[(d, ts[i - 1], INF)] += mu
    return out


def betti_curve(img):
    """{t: (beta_0, beta_1, beta_2)} at every distinct finite value t."""
    cells = enumerate_cells(img)
    idx = _index(cells)
    ts = sorted({c["birth"] for c in cells})
    res = {}
    for t in ts:
        live = [i for i, c in enumerate(cells) if c["birth"] <= t]
        live_set = set(live)
        pos = {}
        for d in range(4):
            for p, i in enumerate([i for i in live if cells[i]["dim"] == d]):
                pos[i] = p
        n = [sum(1 for i in live if cells[i]["dim"] == d) for d in range(4)]
        rk = [0] * 5
        for d in range(1, 4):
            vecs = []
            for i in live:
                if cells[i]["dim"] == d:
                    v = 0
                    for f in _faces(cells[i], idx):
                        assert f in live_set
                        v ^= 1 << pos[f]
                    vecs.append(v)
            rk[d] = _rank(vecs)
        res[t] = tuple(n[d] - rk[d] - rk[d + 1] for d in range(3))
    return res


def _order(cells):
    """Filtration order (birth, dim, kidx) ascending (reading R1)."""
    return sorted(range(len(cells)), key=lambda i: (cells[i]["birth"], cells[i]["dim"], cells[i]["kidx"]))


def cohomology_pairing(img):
    """{kidx: partner kidx or None (essential)} via coboundary reduction (A.2 of SURVEY)."""
    cells = enumerate_cells(img)
    idx = _index(cells)
    order = _order(cells)
    rank = {i: r for r, i in enumerate(order)}
    cof = {i: [] for i in range(len(cells))}
    for i, c in enumerate(cells):
        if c["dim"] > 0:
            for f in _faces(c, idx):
                cof[f].append(i)
    owner = {}
    partner = {c["kidx"]: None for c in cells}
    reduced = {}
    for i in reversed(order):  # columns in decreasing filtration order
        col = set(rank[j] for j in cof[i])
        while col:
            p = min(col)  # pivot = earliest coface
            if p in owner:
                col ^= reduced[owner[p]]
            else:
                owner[p] = i
                reduced[i] = set(col)
                k1, k2 = cells[i]["kidx"], cells[order[p]]["kidx"]
                partner[k1], partner[k2] = k2, k1
                break
    return partner


def union_find_h0(img):
    """{vertex kidx: edge kidx or None}: H0 pairing by the elder rule."""
    cells = enumerate_cells(img)
    verts = {c["anchor"]: c for c in cells if c["dim"] == 0}
    edges = sorted([c for c in cells if c["dim"] == 1], key=lambda c: (c["birth"], c["kidx"]))
    parent = {v: v for v in verts}

    def find(v):
        while parent[v] != v:
            parent[v] = parent[parent[v]]
            v = parent[v]
        return v

    def key(v):
        return (verts[v]["birth"], verts[v]["kidx"])

    out = {c["kidx"]: None for c in verts.values()}
    for e in edges:
        a, b = sorted(e["verts"])
        ra, rb = find(a), find(b)
        if ra == rb:
            continue
        young, old = (ra, rb) if key(ra) > key(rb) else (rb, ra)
        out[verts[young]["kidx"]] = e["kidx"]
        parent[young] = old
    return out


def elder_1d(x):
    """1D closed form (finite inputs): {vertex index: dying edge index or None}.

    Vertex i is older than j iff (x_i, i) < (x_j, j).  A vertex that is not older than both
    neighbours dies at its lower incident edge (zero persistence).  A local minimum dies at
    min(left bottleneck, right bottleneck), where a bottleneck is the highest edge key between
    the vertex and its nearest older vertex on that side (edge key = (max endpoint value, 2j+1)).
    """
    x = [float(v) for v in x]
    n = len(x)
    vk = [(x[i], 2 * i) for i in range(n)]
    ek = [(max(x[j], x[j + 1]), 2 * j + 1) for j in range(n - 1)]
    out = {}
    for i in range(n):
        best = None
        # left
        m = None
        for j in range(i - 1, -1, -1):
            m = ek[j] if m is None or ek[j] > m else m
            if vk[j] < vk[i]:
                best = m if best is None or m < best else best
                break
        m = None
        for j in range(i + 1, n):
            m = ek[j - 1] if m is None or ek[j - 1] > m else m
            if vk[j] < vk[i]:
                best = m if best is None or m < best else best
                break
        out[i] = None if best is None else (best[1] - 1) // 2
    return out


def euler_curve_ok(img, dims, births, deaths):
    """Sum_d (-1)^d #{finite d-cells with birth <= t} == Sum_d (-1)^d #{bars alive at t}."""
    cells = enumerate_cells(img)
    ts = sorted({c["birth"] for c in cells})
    for t in ts:
        lhs = sum((-1) ** c["dim"] for c in cells if c["birth"] <= t)
        rhs = sum((-1) ** int(d) for d, b, e in zip(dims, births, deaths) if b <= t < e)
        if lhs != rhs:
            return False
    return True
