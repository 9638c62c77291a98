import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
for tma in (0, 1):
    for shape in ((8, 12), (5, 6, 40), (6, 7), (3, 4, 5)):
        for nan in (False, True):
            img = gen.small_int_image(shape, 3, seed=70)
            if nan:
                img.flat[img.size // 2] = np.nan
            try:
                with cr.options(kf_tma=tma):
                    cr.barcodes(torch.from_numpy(img).cuda(), len(shape) - 1)
                torch.cuda.synchronize()
                print(tma, shape, nan, "ok", flush=True)
            except Exception as e:
                print(tma, shape, nan, "ERR", str(e)[:150], flush=True)
                if "illegal" in str(e):
                    sys.exit(1)
