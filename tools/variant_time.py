"""Measurement helper: wall ms per call of cr_barcodes(_batched) for a package root.
python tools/variant_time.py PKGROOT c1 c4 c5b"""
import sys, os, time
root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
for name in sys.argv[2:]:
    img, md = gen.config(name)
    t = torch.from_numpy(img).cuda()
    f = (lambda: cr.barcodes_batched(t, md)) if name in ("c5b", "c3") else (lambda: cr.barcodes(t, md))
    reps = 200 if name in ("c1", "c2") else 5
    for _ in range(3): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    cr.set_profiling(True); f(); st = cr.last_stats()["stages"]; cr.set_profiling(False)
    print(root, name, round(ms, 3), {k: round(v, 3) for k, v in st.items()}, flush=True)
