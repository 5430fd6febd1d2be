"""Richardson / pseudo-time solve cost per iteration at cfg2 size (development
tool): wall time of hdgc_richardson with rho = 0 (never converges, runs
max_iter + 1 iterations) for two max_iter values, difference / iterations —
the per-iteration cost including the device-side norm reduction and the
host's chunked queueing — next to the substep (update) kernel time alone
from a substep batch, and one converging solve (rho = 1e-3).  Prints JSON lines."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402
from paper_1508_04245_b200.timeloop import richardson_ds  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
m = M.generate_structured((0, 0, 1, 1), n, n)
sf = F.StreamFunction(16, 2)
u = F.interpolate_curl(m, k, sf)
w = F.transfer_I_host(m, k, u)
inf = F.inflow_values(m, k, sf)
op = ConvectionOperator(m, k)
ud, wd, infd = (torch.from_numpy(x).cuda() for x in (u, w, inf))
umax = op.max_speed(ud)
dtc = F.cfl_dt(m.h_min(), k, umax)
tau = 20 * dtc
ds = richardson_ds(tau, umax, m.h_min(), k)


def solve(max_iter, rho):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, it, conv, r0, r1 = op.richardson(ud, wd, torch.zeros_like(wd), tau, ds, rho, max_iter, infd)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, it, conv


solve(10, 0.0)
t = {}
for mi in (20, 80):
    t[mi] = min(solve(mi, 0.0)[0] for _ in range(3))
per_it = (t[80] - t[20]) / 60
# substep kernel alone (same update kernel family, SUBSTEP epilogue), batch of 60 vs 20
op.substeps(ud, wd.clone(), 1e-7, 4, infd)
tb = {}
for ns in (20, 60):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wc = wd.clone()
    e0.record()
    op.substeps(ud, wc, 1e-7, ns, infd)
    e1.record()
    torch.cuda.synchronize()
    tb[ns] = e0.elapsed_time(e1) * 1e-3
kern = (tb[60] - tb[20]) / 40
# bare STAGE kernel in-stream: SSP-RK2 propagation runs SUBSTEP + STAGE per step back to back (PDL)
op.propagate(ud, wd.clone(), 1e-7, 4, infd, "ssprk2")
tp = {}
for ns in (10, 40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wc = wd.clone()
    e0.record()
    op.propagate(ud, wc, 1e-7, ns, infd, "ssprk2")
    e1.record()
    torch.cuda.synchronize()
    tp[ns] = e0.elapsed_time(e1) * 1e-3
stage = (tp[40] - tp[10]) / 30 - kern
tc, itc, conv = min(solve(500, 1e-3) for _ in range(3))
print(json.dumps({"k": k, "elements": m.n_elements, "tau_over_dtc": 20, "ds": ds,
                  "richardson_us_per_iteration": per_it * 1e6, "substep_kernel_us": kern * 1e6,
                  "stage_kernel_us": stage * 1e6, "overhead_vs_stage": per_it / stage - 1.0,
                  "solve_rho_1e-3": {"iterations": itc, "converged": conv, "ms": tc * 1e3,
                                     "us_per_iteration": tc / (itc + 1) * 1e6}}))
