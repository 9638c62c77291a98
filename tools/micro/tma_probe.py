"""Which shapes make the filtration fail (TMA ring vs cp.async ring)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
shapes = [(4, 4), (8, 12), (5, 12, 60), (9, 13, 32), (3, 3, 36), (2, 40, 64), (128, 128, 128)]
no = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for sh in shapes:
    img = gen.small_int_image(sh, 3, seed=1)
    t = torch.from_numpy(img).cuda()
    try:
        with cr.options(kf_tma=1 - no):
            cr.barcodes(t, len(sh) - 1)
        print(sh, "ok", cr.last_stats()["kf_tma"], flush=True)
    except Exception as e:
        print(sh, "FAIL", e, flush=True)
        break
