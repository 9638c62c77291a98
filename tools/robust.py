"""Robustness sweep (not a unit test: minutes of oracle time): larger / differently distributed
inputs than the parity tests, GPU vs oracle (bars, birth cells) and GPU path cross-checks."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_12692_b200 as cr
import oracle
from workloads import generators as gen

def gpu(img, md, **opts):
    with cr.options(**opts):
        t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        t0 = time.time()
        d, b, e, c = cr.barcodes(t, md, cells=True).numpy()
        torch.cuda.synchronize()
        return (d, b, e, c), time.time() - t0, cr.last_stats()

def same(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint32) if np.asarray(x).dtype == np.float32 else x,
                              np.asarray(y).view(np.uint32) if np.asarray(y).dtype == np.float32 else y)
               for x, y in zip(a, b))

rng = np.random.default_rng(123)
cases = [
    ("1d walk 2^26", np.cumsum(rng.standard_normal(1 << 26)).astype(np.float32), 0, "tree"),
    ("1d iid 2^24", rng.random(1 << 24, dtype=np.float32), 0, "oracle"),
    ("1d int levels 2^22", rng.integers(0, 50, 1 << 22).astype(np.float32), 0, "oracle"),
    ("1d walk+inf 2^23", np.where(rng.random(1 << 23) < 0.01, np.inf, np.cumsum(rng.standard_normal(1 << 23))).astype(np.float32), 0, "tree"),
    ("2d iid 1024^2", rng.random((1024, 1024), dtype=np.float32), 1, "oracle"),
    ("2d grf 2048^2", gen.grf((2048, 2048), 4.0, 7), 1, "reduce"),
    ("2d int8 512x700", rng.integers(0, 8, (512, 700)).astype(np.float32), 1, "oracle"),
    ("3d iid 48^3", rng.random((48, 48, 48), dtype=np.float32), 2, "oracle"),
]
for name, img, md, ref in cases:
    g, dt, st = gpu(img, md)
    msg = f"{name}: gpu {dt*1e3:.1f} ms path {st['path']} bars {len(g[0])}"
    if ref == "oracle":
        t0 = time.time()
        o = oracle.ph(img, md)
        ok = same(g, (o.dim, o.birth, o.death, o.cell))
        msg += f" | oracle {time.time()-t0:.1f} s equal={ok}"
    elif ref == "tree":
        h, _, st2 = gpu(img, md, **{"1d_tree": 1})
        msg += f" | tree path {st2['path']} equal={same(g, h)}"
    elif ref == "reduce":
        h, dt2, _ = gpu(img, md, top_reduce=1)
        msg += f" | top by reduction ({dt2*1e3:.1f} ms) equal={same(g, h)}"
    print(msg, flush=True)
