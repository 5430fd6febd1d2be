"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck) over
every kernel family (development tool; sizes kept small, the tools are slow):

  cfg1   32x32 k=2 (thread kernel): apply + 5 substeps (PDL batch)
  k4     64x64 k=4 (tile prep on DMMA + TMA/mbarrier sum-factorised kernel):
         apply + 100-substep PDL batch + 6 Richardson iterations (fused STAGE)
  k8     16x16 k=8 (ring mode: cp.async row streaming): apply + 3 substeps
  modal  16x16 k=4 HDGC_MODAL path (three-warp kernel): apply + 3 substeps
  3d     4^3 cube k=3: apply + 2 substeps

  python tools/sanitize_cases.py [case ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import fields3d as F3  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def case2d(n, k, nsub, rich=0):
    m = M.generate_structured((0, 0, 1, 1), n, n)
    sf = F.StreamFunction(4, 1, (1.0, 0.3))
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    inf = F.inflow_values(m, k, sf)
    op = ConvectionOperator(m, k)
    ud, wd, infd = dev(u), dev(w), dev(inf)
    op.apply(ud, wd, infd)
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    op.substeps(ud, wd.clone(), dt, nsub, infd)
    if rich:
        op.richardson(ud, wd, torch.zeros_like(wd), 10 * dt, 0.1, 0.0, rich - 1, infd)
    op.check_finite()


def case3d():
    m = M3.generate_cube(4)
    k = 3
    vp = F3.VectorPotential(3, 5, (0.3, 0.2, -0.5))
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    inf = F3.inflow_values3(m, k, vp)
    op = ConvectionOperator(m, k)
    op.apply(dev(u), dev(w), dev(inf))
    op.substeps(dev(u), dev(w), 1e-4, 2, dev(inf))
    op.check_finite()


CASES = {
    "cfg1": lambda: case2d(32, 2, 5),
    "k4": lambda: case2d(64, 4, 100, rich=6),
    "k8": lambda: case2d(16, 8, 3),
    "modal": lambda: case2d(16, 4, 3),
    "3d": case3d,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        torch.cuda.synchronize()
        print("case", name, "ok", flush=True)
