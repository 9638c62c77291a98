"""Where the non-kernel time of one C2 call goes: Python wrapper vs C call vs kernels."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2005_12692_b200 as cr
from workloads import generators as gen

x = torch.from_numpy(gen.random_walk(1 << 24, 2)).cuda()
cap = cr.max_pairs(tuple(x.shape), 0)
pairs = torch.empty((cap, 3), dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream()
shp = cr._shape(tuple(x.shape))
n = ctypes.c_int64(0)
sp = ctypes.c_void_p(stream.cuda_stream)


def ev_time(f, reps=30):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    tot = 0.0
    host = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t0 = time.perf_counter()
        f()
        host += time.perf_counter() - t0
        b.record(stream)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1e3, host / reps * 1e6


def wrapper():
    return len(cr.barcodes(x, 0, out=(pairs, None)).pairs)


def direct():
    st = cr._lib.cr_barcodes(x.data_ptr(), shp, 1, 0, pairs.data_ptr(), None, cap, ctypes.byref(n), sp)
    return st


for prof in (False, True):
    cr.set_profiling(prof)
    print("profiling", prof)
    print("  wrapper  events us %.1f  host us %.1f" % ev_time(wrapper))
    print("  direct   events us %.1f  host us %.1f" % ev_time(direct))
    if prof:
        print("  stages", cr.last_stats()["stages"])
t0 = time.perf_counter()
for _ in range(1000):
    torch.cuda.current_stream(x.device)
print("current_stream us", (time.perf_counter() - t0) * 1e3)
