"""Per-stage device times of the 1D path on C2 (CUDA events recorded by the library) and the
path taken for each tile-path test case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
x = torch.from_numpy(gen.random_walk(1 << 24, 2)).cuda()
cap = cr.max_pairs((1 << 24,), 0)
pairs = torch.empty((cap, 3), dtype=torch.int32, device='cuda')
cr.set_profiling(True)
acc = {}
for k in range(15):
    cr.barcodes(x, 0, out=(pairs, None))
    st = cr.last_stats()
    if k >= 5:
        for a, b in st['stages'].items():
            acc[a] = acc.get(a, 0) + b / 10
print('path', st['path'], {a: round(b, 4) for a, b in acc.items()}, 'total', round(sum(acc.values()), 4))
sys.path.insert(0, 'tests')
from test_gpu_parity import _series_cases
for name, s in sorted(_series_cases().items()):
    cr.barcodes(torch.from_numpy(s).cuda(), 0)
    print(name, len(s), 'path', cr.last_stats()['path'])
# tuning sweep of the contraction-round knobs (level-1 stage time)
for l1r in ["1", "2", "3", "6"]:
    for r in ["1", "2", "4"]:
        os.environ["CR_1D_L1ROUNDS"] = l1r
        os.environ["CR_1D_ROUNDS"] = r
        acc = {}
        for k in range(8):
            cr.barcodes(x, 0, out=(pairs, None))
            if k >= 3:
                for a, b in cr.last_stats()['stages'].items():
                    acc[a] = acc.get(a, 0) + b / 5
        print('l1rounds', l1r, 'rounds', r, {a: round(b, 4) for a, b in acc.items()}, 'total', round(sum(acc.values()), 4))
os.environ["CR_1D_L1ROUNDS"] = "6"
os.environ["CR_1D_ROUNDS"] = "1"
cr.barcodes(x, 0, out=(pairs, None))
