"""Run one volume of the C5b batch alone (measurement helper): python tools/one_volume.py 25 [--debug2]
Times cr_barcodes on that 128^3 volume and, with --debug2, prints K5's critical path for it."""
import sys
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2005_12692_b200 as cr  # noqa: E402
from workloads import generators as gen  # noqa: E402

k = int(sys.argv[1])
rng = np.random.default_rng(6)
for i in range(k + 1):
    v = gen.masked_grf((128, 128, 128), 3.0, 60.0, rng)
t = torch.from_numpy(v).cuda()
cr.barcodes(t, 2)
if "--debug2" in sys.argv:
    cr.set_option("debug", 2)
cr.set_profiling(True)
for r in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bc = cr.barcodes(t, 2)
    e1.record()
    torch.cuda.synchronize()
    print("volume", k, "ms", e0.elapsed_time(e1), cr.last_stats().get("stages"))
