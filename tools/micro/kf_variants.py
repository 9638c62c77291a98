"""Filtration stage time (CUDA events, median of 7) per package root, TMA ring on / off.
python tools/micro/kf_variants.py ROOT [ROOT...]"""
import os, subprocess, sys, json
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 or not sys.argv[1].startswith("@"):
    for root in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, "@" + root])
    sys.exit(0)
root = sys.argv[1][1:]
sys.path.insert(0, root)
sys.path.insert(1, HERE)
import numpy as np, torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
for name in ("c5b", "c5", "c4"):
    img, md = gen.config(name)
    t = torch.from_numpy(img).cuda()
    f = (lambda: cr.barcodes_batched(t, md)) if name == "c5b" else (lambda: cr.barcodes(t, md))
    for no in (0, 1):
        with cr.options(kf_tma=1 - no):
            f(); f()
            cr.set_profiling(True)
            ts = []
            for _ in range(7):
                f()
                ts.append(cr.last_stats()["stages"]["filtration"])
            cr.set_profiling(False)
            print(json.dumps({"root": root, "cfg": name, "no_tma": no, "tma": cr.last_stats()["kf_tma"],
                              "filtration_ms": round(float(np.median(ts)), 4)}), flush=True)
    del t
