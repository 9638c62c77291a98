python - <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch, paper_2005_12692_b200 as cr
from workloads import generators as gen
for B in (600, 1200, 4800, 65536):
    imgs = torch.from_numpy(gen.blobs(B, 3)).cuda()
    try:
        bc, off = cr.barcodes_batched(imgs, 1); torch.cuda.synchronize(); print(B, "ok", int(off[-1]))
    except Exception as e:
        print(B, "ERR", e); break
PY
python tools/k7_time.py 2>&1 | tail -2
