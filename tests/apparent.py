"""Apparent pairs by their definition (Ripser's shortcut inherited by the paper),
vectorised numpy over the Khalimsky grid -- test infrastructure, independent of oracle/ and of the
CUDA path.

A finite cell s (key = (birth, kidx), reading R1) is UP when t = its min-key cofacet exists and
s is t's max-key facet; then (s, t) is an apparent pair.  Cells outside the grid or with a +inf
vertex are absent (reading R5).  Also the per-dimension counts the GPU path reports in cr_stats
(SURVEY.md §8(d.8)): finite cells, UP cells, and the basins (finite vertices that are not UP)."""
import numpy as np


def khalimsky_births(img: np.ndarray) -> np.ndarray:
    """float64 births over the (2n-1)^3 grid (1D/2D images padded to 3D), +inf = absent."""
    a = np.asarray(img, np.float64)
    while a.ndim < 3:
        a = a[None]
    nz, ny, nx = a.shape
    b = np.full((2 * nz - 1, 2 * ny - 1, 2 * nx - 1), -np.inf)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                # cell (2z+i, 2y+j, 2x+k) takes the max over voxel offsets <= (i, j, k)
                for i in range(dz + 1):
                    for j in range(dy + 1):
                        for k in range(dx + 1):
                            v = a[i:nz - dz + i, j:ny - dy + j, k:nx - dx + k]
                            sl = b[dz::2, dy::2, dx::2]
                            np.maximum(sl, v, out=sl)
    return b


def apparent_up(img: np.ndarray):
    """(up mask over the Khalimsky grid, dims array, finite mask)."""
    b = khalimsky_births(img)
    KZ, KY, KX = b.shape
    kidx = np.arange(b.size, dtype=np.int64).reshape(b.shape)
    finite = np.isfinite(b)
    Z, Y, X = np.meshgrid(np.arange(KZ), np.arange(KY), np.arange(KX), indexing="ij")
    odd = [Z & 1, Y & 1, X & 1]
    dims = odd[0] + odd[1] + odd[2]
    INF = np.inf

    def shifted(arr, axis, sgn, fill):
        out = np.full_like(arr, fill)
        src = [slice(None)] * 3
        dst = [slice(None)] * 3
        if sgn > 0:
            src[axis], dst[axis] = slice(1, None), slice(None, -1)
        else:
            src[axis], dst[axis] = slice(None, -1), slice(1, None)
        out[tuple(dst)] = arr[tuple(src)]
        return out

    # neighbours in increasing kidx order: -Z, -Y, -X, +X, +Y, +Z
    order = [(0, -1), (1, -1), (2, -1), (2, 1), (1, 1), (0, 1)]
    # min-key cofacet (even axis of s): strict < over births in kidx order
    mcb = np.full(b.shape, INF)
    mc = np.full(b.shape, -1)
    mfb = np.full(b.shape, -INF)
    mf = np.full(b.shape, -1)
    for q, (ax, sg) in enumerate(order):
        nb = shifted(b, ax, sg, INF)
        nbf = shifted(finite, ax, sg, False)
        cof = (odd[ax] == 0) & nbf
        take = cof & (nb < mcb)
        mcb = np.where(take, nb, mcb)
        mc = np.where(take, q, mc)
        fac = (odd[ax] == 1)
        takef = fac & (nb >= mfb)
        mfb = np.where(takef, nb, mfb)
        mf = np.where(takef, q, mf)
    up = np.zeros(b.shape, bool)
    for q, (ax, sg) in enumerate(order):
        # t = s + sg e_ax; s is t's max facet iff mf(t) points back (opposite direction)
        back = order.index((ax, -sg))
        mf_t = shifted(mf, ax, sg, -2)
        up |= finite & (mc == q) & (mf_t == back)
    return up, dims, finite


def counts(img: np.ndarray) -> dict:
    up, dims, finite = apparent_up(img)
    cells = [int(np.count_nonzero(finite & (dims == d))) for d in range(4)]
    app = [int(np.count_nonzero(up & (dims == d))) for d in range(4)]
    basins = int(np.count_nonzero(finite & (dims == 0) & ~up))
    return {"cells": cells, "apparent": app, "basins": basins}


def pairs_up(img: np.ndarray):
    """[(s, t)] kidx of the apparent pairs (lower cell s, upper cell t)."""
    up, _, _ = apparent_up(img)
    b = khalimsky_births(img)
    KZ, KY, KX = b.shape
    st = {0: KY * KX, 1: KX, 2: 1}
    out = []
    for s in np.flatnonzero(up.ravel()):
        z, r = divmod(int(s), KY * KX)
        y, x = divmod(r, KX)
        c = (z, y, x)
        best, bt = None, None
        for ax, sg in [(0, -1), (1, -1), (2, -1), (2, 1), (1, 1), (0, 1)]:
            if c[ax] & 1:
                continue
            cc = list(c)
            cc[ax] += sg
            if not (0 <= cc[ax] < b.shape[ax]):
                continue
            bb = b[tuple(cc)]
            if np.isfinite(bb) and (best is None or bb < best):
                best, bt = bb, int(s) + sg * st[ax]
        out.append((int(s), bt))
    return out
