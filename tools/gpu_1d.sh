mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "1d or c2 or host or edge or golden or sin or batched_1d" > gpurun_out/pytest_1d.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_1d.log | grep -v Warn
timeout 300 python tools/c2_time.py > gpurun_out/c2_time.log 2>&1; echo time=$?
cat gpurun_out/c2_time.log
CR_DEBUG_STATS=1 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2005_12692_b200 as cr
from workloads import generators as gen
x = torch.from_numpy(gen.random_walk(1 << 24, 2)).cuda()
cr.barcodes(x, 0)
" 2>&1 | grep "\[cr\]"
