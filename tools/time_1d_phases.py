"""Time the 1D level-1 kernel with phases skipped (CR_1D_DBG mask) -- results are wrong when a
phase is skipped; this only measures where the time goes."""
import os, sys, torch
sys.path.insert(0, '.')
import paper_2005_12692_b200 as cr
from workloads import generators as gen
x = torch.from_numpy(gen.random_walk(1 << 24, 2)).cuda()
cap = cr.max_pairs((1 << 24,), 0)
pairs = torch.empty((cap, 3), dtype=torch.int32, device='cuda')
cr.set_profiling(True)
for mask in [0, 1, 2, 4, 6, 7, 8, 9]:
    os.environ['CR_1D_DBG'] = str(mask)
    ts = []
    for k in range(8):
        try:
            cr.barcodes(x, 0, out=(pairs, None))
        except Exception as e:
            pass
        st = cr.last_stats()['stages']
        if k >= 3 and 'stages' and st: ts.append(st.get('1d_level1', 0))
    print(mask, round(sum(ts) / max(1, len(ts)), 4), flush=True)
