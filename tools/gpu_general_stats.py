"""Print general-path statistics (counts, rounds, additions) for the synthetic configs."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2005_12692_b200 as cr
from workloads import generators as gen
cr.set_profiling(True)
for name in sys.argv[1:]:
    if name.startswith('crop'):
        img, md = gen.grf((64, 64, 64), 2.0, 4), 2
    else:
        img, md = gen.config(name)
    t = torch.from_numpy(img).cuda()
    if name in ('c3', 'c5b'):
        cr.barcodes_batched(t, md)
    else:
        cr.barcodes(t, md)
    torch.cuda.synchronize()
    t0 = time.time()
    if name in ('c3', 'c5b'):
        cr.barcodes_batched(t, md)
    else:
        cr.barcodes(t, md)
    torch.cuda.synchronize()
    st = cr.last_stats()
    st['wall_s'] = time.time() - t0
    print(name, json.dumps(st), flush=True)
