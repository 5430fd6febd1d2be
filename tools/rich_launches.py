"""ncu launch-list driver: one Richardson solve (rho = 0, 24 iterations) at cfg2 size."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F, mesh as M
from paper_1508_04245_b200.forms import ConvectionOperator
m = M.generate_structured((0, 0, 1, 1), 256, 256); k = 4
sf = F.StreamFunction(16, 2)
u = F.interpolate_curl(m, k, sf); w = F.transfer_I_host(m, k, u); inf = F.inflow_values(m, k, sf)
op = ConvectionOperator(m, k)
ud, wd, infd = (torch.from_numpy(x).cuda() for x in (u, w, inf))
op.richardson(ud, wd, torch.zeros_like(wd), 1e-5, 0.1, 0.0, 23, infd)
op.substeps(ud, wd, 1e-7, 3, infd)
torch.cuda.synchronize()
