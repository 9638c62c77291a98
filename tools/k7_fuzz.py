"""K7 fuzz: random batch shapes (incl. 1-wide, 32x32 = the reduction variant) with +inf masks,
each image's bars vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_12692_b200 as cr, oracle
from workloads import generators as gen
rng = np.random.default_rng(2024)
bad = 0
for t in range(60):
    ny, nx = int(rng.integers(1, 33)), int(rng.integers(1, 33))
    B = int(rng.integers(1, 40))
    imgs = np.stack([gen.small_int_image((ny, nx), int(rng.integers(2, 9)), seed=int(rng.integers(1 << 30)),
                                         inf_frac=[0.0, 0.05, 0.3][t % 3]) for _ in range(B)])
    bc, off = cr.barcodes_batched(torch.from_numpy(imgs).cuda(), 1)
    d, b, e, _ = bc.numpy()
    off = off.cpu().numpy()
    for i in range(B):
        o = oracle.ph(imgs[i], 1)
        s = slice(off[i], off[i + 1])
        got = sorted(zip(d[s].tolist(), b[s].tolist(), e[s].tolist()))
        exp = sorted(zip(o.dim.tolist(), o.birth.tolist(), o.death.tolist()))
        if got != exp:
            bad += 1
            print("MISMATCH", t, (ny, nx), i, len(got), len(exp))
            break
print("k7 fuzz done, bad =", bad, "path", cr.last_stats()["path"])
