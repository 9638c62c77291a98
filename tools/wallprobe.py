import sys, time, os
import torch
sys.path.insert(0, os.getcwd())
import paper_2005_12692_b200 as cr
from workloads import generators as gen
img, md = gen.config("c5b")
t = torch.from_numpy(img).cuda()
for _ in range(3): cr.barcodes_batched(t, md)
torch.cuda.synchronize()
for r in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record()
    out = cr.barcodes_batched(t, md)
    w1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    print("events", round(e0.elapsed_time(e1), 2), "wall call", round((w1 - w0) * 1e3, 2), "wall+sync", round((w2 - w0) * 1e3, 2), flush=True)
    del out
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); cr.barcodes_batched(t, md); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(8)
