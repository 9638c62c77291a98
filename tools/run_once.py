"""One cr_barcodes / cr_barcodes_batched call on a BASELINE config (for ncu captures).
Usage: python tools/run_once.py c4 [--calls N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_12692_b200 as cr  # noqa: E402
from workloads import generators as gen  # noqa: E402

name = sys.argv[1]
calls = int(sys.argv[sys.argv.index("--calls") + 1]) if "--calls" in sys.argv else 1
img, md = gen.config(name)
t = torch.from_numpy(img).cuda()
for _ in range(calls):
    if name in ("c3", "c5b"):
        cr.barcodes_batched(t, md)
    else:
        cr.barcodes(t, md)
torch.cuda.synchronize()
print("ok", name, cr.last_stats()["path"])
