import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2005_12692_b200 as cr
from workloads import generators as gen
img, md = gen.config('c1')
t = torch.from_numpy(img).cuda()
for _ in range(20): cr.barcodes(t, md)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N): cr.barcodes(t, md)
torch.cuda.synchronize()
print("c1 wall ms per call", (time.perf_counter() - t0) / N * 1e3)
cr.set_profiling(True)
cr.barcodes(t, md)
print(cr.last_stats())
