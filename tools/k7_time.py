import sys, time
sys.path.insert(0, '.')
import torch, paper_2005_12692_b200 as cr
from workloads import generators as gen
imgs = torch.from_numpy(gen.blobs(65536, 3)).cuda()
for md in (0, 1):
    for _ in range(2):
        cr.barcodes_batched(imgs, md)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        cr.barcodes_batched(imgs, md)
    torch.cuda.synchronize()
    print('maxdim', md, (time.perf_counter() - t) / 5 * 1e3, 'ms', cr.last_stats()['stages'])
