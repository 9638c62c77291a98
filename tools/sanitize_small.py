"""Small end-to-end calls for compute-sanitizer (memcheck / racecheck / synccheck): every path
(1D tiles, 1D tree, general 2D/3D with duality and reduction, batched K7, pairing, death cells,
lifetime image, top dimension, host-buffer entries, K5 with schedule jitter)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen

dev = torch.device("cuda", 0)
x = torch.from_numpy(gen.random_walk(3 * 4096 + 5, 1)).to(dev)
cr.barcodes(x, 0, cells=True)
with cr.options(**{"1d_tree": 1}):
    cr.barcodes(x, 0)
cr.pairing(x)
a = gen.small_int_image((23, 19), 4, seed=2, inf_frac=0.05); a[8:11, 6:9] = np.inf
ta = torch.from_numpy(a).to(dev)
bc = cr.barcodes(ta, 1, cells=True); cr.death_cells(ta, bc.cells); cr.pairing(ta)
cr.barcodes_topdim(ta); cr.lifetime_image(ta, 1)
v = gen.masked_grf((14, 15, 16), 2.0, 6.5, 3)
tv = torch.from_numpy(v).to(dev)
cr.barcodes(tv, 2); cr.pairing(tv)
with cr.options(top_reduce=1, k5_jitter_ns=3000):
    cr.barcodes(tv, 2)
vols = torch.from_numpy(np.stack([gen.masked_grf((12, 13, 11), 1.5, 5.5, 40 + i)
                                  for i in range(3)])).to(dev)
cr.barcodes_batched(vols, 2, cells=True)
pinned = torch.from_numpy(gen.masked_grf((10, 12, 9), 1.5, 4.5, 7)).pin_memory()
cr.barcodes_host(pinned.numpy(), 2, cells=True)
cr.barcodes_batched_host(vols.cpu().numpy(), 2, cells=True)
imgs = torch.from_numpy(gen.blobs(16, 4)).to(dev)
cr.barcodes_batched(imgs, 1, cells=True)
torch.cuda.synchronize()
print("sanitize workload ok")
