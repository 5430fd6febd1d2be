"""Small driver for ncu on the 3D kernels (cube n from argv, k=3)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields3d as F3  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k = 3
m = M3.generate_cube(n)
vp = F3.VectorPotential(4, 5)
u = F3.interpolate_curl3(m, k, vp)
w = F3.transfer_I3_host(m, k, u)
op = ConvectionOperator(m, k)
ud, wd = torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda()
op.substeps(ud, wd, 1e-7, 3)
torch.cuda.synchronize()
print("ok", m.n_elements)
