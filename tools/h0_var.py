"""Per-call stage times over repeated calls (variance hunt): python tools/h0_var.py c5 [maxdim] [reps]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
md = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
img, _ = gen.config(name)
t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
cr.set_profiling(True)
for r in range(reps):
    t0 = time.perf_counter()
    bc = cr.barcodes(t, md)
    torch.cuda.synchronize()
    st = cr.last_stats()
    print(f"{name} md={md} rep {r}: wall {1e3*(time.perf_counter()-t0):8.1f} ms  bars {len(bc.dim)}  " +
          " ".join(f"{k}={v:.2f}" for k, v in st["stages"].items()), flush=True)
