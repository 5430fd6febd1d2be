"""propagate_convection step time at cfg2 size (development tool): (40 - 10 steps) / 30."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1508_04245_b200 import fields as F, mesh as M
from paper_1508_04245_b200.forms import ConvectionOperator
m = M.generate_structured((0, 0, 1, 1), 256, 256)
k = 4
sf = F.StreamFunction(16, 2)
u = F.interpolate_curl(m, k, sf); w = F.transfer_I_host(m, k, u); inf = F.inflow_values(m, k, sf)
op = ConvectionOperator(m, k)
ud, wd, infd = (torch.from_numpy(x).cuda() for x in (u, w, inf))
for scheme in ("euler", "ssprk2"):
    op.propagate(ud, wd, 1e-7, 4, infd, scheme)
    res = {}
    for n in (10, 40):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); op.propagate(ud, wd, 1e-7, n, infd, scheme); e1.record(); torch.cuda.synchronize()
        res[n] = e0.elapsed_time(e1) * 1e3
    print(json.dumps({"scheme": scheme, "us_per_step": (res[40] - res[10]) / 30}))
