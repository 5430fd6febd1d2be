"""Quick device timing of one apply / substep at a given mesh size and order
(development tool; bench.py is the contract)."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402


def flops_pinned(k):
    nb = (k + 1) * (k + 2)
    nbs = nb // 2
    nqv = [3, 7, 25, 36, 64, 81, 121, 144][k - 1]
    nf = [3, 4, 6, 7, 9, 10, 12, 13][k - 1]
    return 2 * (nqv * (2 * nb + 6 * nbs) + 3 * nf * ((k + 1) + 3 * nb)), 24 * nb + 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--k", type=str, default="4")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    m = M.generate_structured((0, 0, 1, 1), args.n, args.n)
    out = []
    for k in [int(x) for x in args.k.split(",")]:
        sf = F.StreamFunction(16, 2)
        u = F.interpolate_curl(m, k, sf)
        w = F.transfer_I_host(m, k, u)
        op = ConvectionOperator(m, k)
        ud = torch.from_numpy(u).cuda()
        wd = torch.from_numpy(w).cuda()
        r = torch.empty_like(wd)
        flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
        for _ in range(3):
            op.apply(ud, wd, out=r)
        times = []
        for _ in range(args.reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.apply(ud, wd, out=r)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(times))
        # substep batch of 20, L2 warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        op.substeps(ud, wd, 1e-6, 4)
        e0.record()
        op.substeps(ud, wd, 1e-6, 20)
        e1.record()
        torch.cuda.synchronize()
        ts = e0.elapsed_time(e1) * 1e-3 / 20
        fl, by = flops_pinned(k)
        NT = m.n_elements
        out.append(dict(k=k, NT=NT, apply_us=t * 1e6, substep_us=ts * 1e6,
                        dofs_per_s=NT * (k + 1) * (k + 2) / t,
                        pinned_tflops=NT * fl / t / 1e12, gbs=NT * by / t / 1e9))
        print(json.dumps(out[-1]))




def main3(n=32, k=3, reps=5):
    from paper_1508_04245_b200 import fields3d as F3, mesh3d as M3
    m = M3.generate_cube(n)
    vp = F3.VectorPotential(4, 5)
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    op = ConvectionOperator(m, k)
    ud, wd = torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda()
    r = torch.empty_like(wd)
    op.apply(ud, wd, out=r)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply(ud, wd, out=r)
    e1.record()
    torch.cuda.synchronize()
    ta = e0.elapsed_time(e1) * 1e-3 / reps
    e0.record()
    op.substeps(ud, wd, 1e-7, 20)
    e1.record()
    torch.cuda.synchronize()
    ts = e0.elapsed_time(e1) * 1e-3 / 20
    nb = 3 * (k + 1) * (k + 2) * (k + 3) // 6
    pinned = 159720 if k == 3 else None
    print(json.dumps(dict(dim=3, k=k, NT=m.n_elements, apply_us=ta * 1e6, substep_us=ts * 1e6,
                          dofs_per_s=m.n_elements * nb / ts,
                          pinned_tflops=(m.n_elements * pinned / ts / 1e12) if pinned else None)))


if __name__ == "__main__":
    if "--3d" in sys.argv:
        main3()
    else:
        main()
