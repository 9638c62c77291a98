mkdir -p gpurun_out
CR_DEBUG_STATS=1 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2005_12692_b200 as cr
from workloads import generators as gen
x = torch.from_numpy(gen.random_walk(1 << 24, 2)).cuda()
cr.barcodes(x, 0)
" > gpurun_out/dbg.log 2>&1; cat gpurun_out/dbg.log | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_levels_coop -s 3 -c 1 -o gpurun_out/coop -f python tools/c2_time.py > gpurun_out/ncu_coop.log 2>&1; echo ncu=$?
