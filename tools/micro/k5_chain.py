"""K5 debug timeline (cr_set_option debug=2) of one C5b call: the chain from the last column."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2005_12692_b200 as cr
from workloads import generators as gen
img, md = gen.config(sys.argv[1] if len(sys.argv) > 1 else "c5b")
t = torch.from_numpy(img).cuda()
cr.barcodes_batched(t, md)
cr.set_option("debug", 2)
cr.barcodes_batched(t, md)
torch.cuda.synchronize()
