"""One warm call of the general path per config (for ncu launch lists of K1/K2)."""
import sys
sys.path.insert(0, '.')
import torch, paper_2005_12692_b200 as cr
from workloads import generators as gen
for name in sys.argv[1:]:
    img, md = gen.config(name)
    t = torch.from_numpy(img).cuda()
    for _ in range(2):
        cr.barcodes(t, md)
    torch.cuda.synchronize()
    print(name, 'ok', flush=True)
