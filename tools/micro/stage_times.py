"""Per-stage device ms (CUDA events, median of 5) on c5b / c5 / c4, per package root.
python tools/micro/stage_times.py ROOT [ROOT...]"""
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
opts = dict(kv.split("=") for kv in (os.environ.get("OPTS") or "").split() if kv)
for k, v in opts.items():
    cr.set_option(k, int(v))
for name in (os.environ.get("CFGS") or "c5b c5 c4").split():
    img, md = gen.config(name)
    t = torch.from_numpy(img).cuda()
    f = (lambda: cr.barcodes_batched(t, md)) if name in ("c5b", "c3") else (lambda: cr.barcodes(t, md))
    f(); f()
    cr.set_profiling(True)
    runs = []
    for _ in range(5):
        f()
        runs.append(cr.last_stats()["stages"])
    cr.set_profiling(False)
    med = {k: round(float(np.median([r[k] for r in runs])), 4) for k in runs[0]}
    print(json.dumps({"root": root, "opts": opts, "cfg": name, "total": round(sum(med.values()), 3), "stages": med}), flush=True)
    del t
