"""Small driver for ncu: cfg2-sized substep kernels (k from argv)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
m = M.generate_structured((0, 0, 1, 1), n, n)
sf = F.StreamFunction(16, 2)
u = F.interpolate_curl(m, k, sf)
w = F.transfer_I_host(m, k, u)
inf = F.inflow_values(m, k, sf)
op = ConvectionOperator(m, k)
ud, wd, infd = (torch.from_numpy(x).cuda() for x in (u, w, inf))
r = torch.empty_like(wd)
op.apply(ud, wd, infd, out=r)
op.substeps(ud, wd, 1e-7, 4, infd)
torch.cuda.synchronize()
print("ok", k, n)
