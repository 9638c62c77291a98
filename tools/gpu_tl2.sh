for r in 1 2 3 5; do CR_1D_ROUNDS=$r CR_DEBUG_STATS=1 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2005_12692_b200 as cr
from workloads import generators as gen
x = torch.from_numpy(gen.random_walk(1 << 24, 2)).cuda()
for _ in range(3): cr.barcodes(x, 0)
" 2>&1 | grep "coop timeline" | tail -1 | sed "s/^/rounds $r /"; done
