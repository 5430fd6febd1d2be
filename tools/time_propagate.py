"""propagate_convection step time at cfg2 size (development tool): (40 - 10 steps) / 30,
Euler and SSP-RK2, frozen velocity and linearly extrapolated velocity (u_prev
at t_prev = -1e-3, u_cur at t_cur = 0: every pseudo-time level needs a fresh
u(s) and frozen-velocity prep)."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F, mesh as M  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402
m = M.generate_structured((0, 0, 1, 1), 256, 256)
k = 4
sf = F.StreamFunction(16, 2)
u = F.interpolate_curl(m, k, sf); w = F.transfer_I_host(m, k, u); inf = F.inflow_values(m, k, sf)
u_prev = F.interpolate_curl(m, k, F.StreamFunction(16, 3))
op = ConvectionOperator(m, k)
ud, wd, infd, upd = (torch.from_numpy(x).cuda() for x in (u, w, inf, u_prev))
for extrap in (False, True):
    for scheme in ("euler", "ssprk2"):
        kw = dict(u_prev=upd, t_prev=-1e-3, t_cur=0.0, t1=0.0) if extrap else {}
        op.propagate(ud, wd.clone(), 1e-7, 4, infd, scheme, **kw)
        res = {}
        for n in (10, 40):
            wc = wd.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); op.propagate(ud, wc, 1e-7, n, infd, scheme, **kw); e1.record(); torch.cuda.synchronize()
            res[n] = e0.elapsed_time(e1) * 1e3
        print(json.dumps({"k": k, "elements": m.n_elements, "scheme": scheme, "extrapolated": extrap,
                          "us_per_step": (res[40] - res[10]) / 30}))
