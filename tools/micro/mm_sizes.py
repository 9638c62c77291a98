"""Wall ms per cr_barcodes call (and stage ms) on small/medium images, per package root.
python tools/micro/mm_sizes.py ROOT [ROOT...]"""
import os, subprocess, sys, time, json
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
cases = [("c1", *gen.config("c1")), ("iid256", gen.iid_uniform((256, 256), 7), 1),
         ("iid512", gen.iid_uniform((512, 512), 8), 1), ("grf48^3", gen.grf((48, 48, 48), 2.0, 9), 2),
         ("c4", *gen.config("c4"))]
for name, img, md in cases:
    t = torch.from_numpy(img).cuda()
    reps = 200 if img.size <= 300000 else 10
    for _ in range(5): cr.barcodes(t, md)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): cr.barcodes(t, md)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    cr.set_profiling(True); cr.barcodes(t, md); st = cr.last_stats(); cr.set_profiling(False)
    print(json.dumps({"root": root, "case": name, "wall_ms": round(ms, 4),
                      "stages": {k: round(v, 4) for k, v in st["stages"].items()},
                      "rounds": st["rounds"][:2]}), flush=True)
