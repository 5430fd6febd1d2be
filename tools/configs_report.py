"""Throughput of every BASELINE.json config on one B200 (development / report
tool; bench.py is the driver contract and measures cfg2 only).

One JSON line per (config, k): the single-apply device time (prep + kernel,
median of `reps` calls, L2 flushed by a 512 MB write before each, host enqueue
hidden behind a spin kernel), the substep-batch
time of the config's substep count (whole batch incl. its one prep, divided
by n, L2 flushed before the batch), DOF/s and applies/s for both, and the
pinned-roofline fraction (F(k) flop and B(k) bytes per element;
FP64 bound for k >= 3 and 3D, HBM for k <= 2).  Peaks as in bench.py.

    python tools/configs_report.py > profiles/configs_r01.jsonl
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1508_04245_b200 import basis3d as B3  # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import fields3d as F3  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402


def pinned3(k):
    """SURVEY §8d 3D pinned work per tet (k = 3: 159,720 flop, 1,464 B)."""
    from math import comb
    nbs = comb(k + 3, 3)
    nb = 3 * nbs
    nfd = (k + 1) * (k + 2) // 2
    nqv = ((3 * k + 1) // 2) ** 3
    nf = len(B3.face_rule(k).weights)   # |quad_triangle(3k+1)|
    return 2 * (nqv * (3 * nb + 3 * nbs + 9 * nbs) + 4 * nf * (nfd + 3 * nb)), 3 * nb * 8 + 24


def timed(fn, reps, flush):
    """Device time of fn() (median over reps, L2 flushed before each).  A
    ~100 us spin kernel is queued before the start event, so the host-side
    enqueue cost of fn (Python + ctypes, ~10-20 us) overlaps it instead of
    showing up as device idle time inside the timed region (it dominated the
    small cfg1 / cfg4 applies)."""
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        torch.cuda._sleep(200000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def report(cfg, m, k, u, w, inf, nsub, dim, reps, flush, dt):
    op = ConvectionOperator(m, k)
    ud, wd = torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda()
    infd = torch.from_numpy(inf).cuda() if inf is not None else None
    r = torch.empty_like(wd)
    for _ in range(3):
        op.apply(ud, wd, infd, out=r)
    t_apply = timed(lambda: op.apply(ud, wd, infd, out=r), reps, flush)
    NT = m.n_elements
    nb = wd.shape[1]
    if dim == 2:
        fl, by = bench.pinned_work(k)
    else:
        fl, by = pinned3(k)
    fp64, _, _ = bench.fp64_peak()
    hbm, _ = bench.hbm_peak()
    bound = "hbm" if (dim == 2 and k <= 2) else "fp64"

    def frac(t):
        return (NT * by / t / 1e9 / hbm) if bound == "hbm" else (NT * fl / t / 1e12 / fp64)

    line = dict(cfg=cfg, dim=dim, k=k, elements=NT, dofs_per_apply=NT * nb,
                apply_us=t_apply * 1e6, apply_dof_per_s=NT * nb / t_apply, applies_per_s=1.0 / t_apply,
                apply_roofline=dict(bound=bound, frac=frac(t_apply)))
    if nsub:
        w0 = wd.clone()
        # time the batch alone (copy outside the events)
        ts = []
        for _ in range(max(3, reps // 4)):
            wd.copy_(w0)
            flush.fill_(1.0)
            torch.cuda._sleep(200000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.substeps(ud, wd, dt, nsub, infd)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t_sub = float(np.median(ts)) / nsub
        line.update(substeps=nsub, dt=dt, substep_us=t_sub * 1e6, substep_dof_per_s=NT * nb / t_sub,
                    substep_applies_per_s=1.0 / t_sub, substep_roofline=dict(bound=bound, frac=frac(t_sub)))
    print(json.dumps(line), flush=True)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    torch.cuda.set_device(0)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def cfg2d(n, k, modes, seed, wind=(0.0, 0.0), jitter=None):
        m = M.generate_jittered(n, 0.2, jitter) if jitter is not None else \
            M.generate_structured((0.0, 0.0, 1.0, 1.0), n, n)
        sf = F.StreamFunction(modes, seed, wind)
        u = F.interpolate_curl(m, k, sf)
        w = F.transfer_I_host(m, k, u)
        inf = F.inflow_values(m, k, sf)
        dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
        return m, u, w, inf, dt

    m, u, w, inf, dt = cfg2d(32, 2, 4, 1)
    report("cfg1", m, 2, u, w, inf, 0, 2, reps, flush, dt)
    m, u, w, inf, dt = cfg2d(256, 4, 16, 2)
    report("cfg2", m, 4, u, w, inf, 100, 2, reps, flush, dt)
    m, u, w, inf, dt = cfg2d(512, 6, 32, 3, (1.0, 0.3), jitter=11)
    report("cfg3", m, 6, u, w, inf, 50, 2, reps, flush, dt)
    for k in range(1, 9):
        m, u, w, inf, dt = cfg2d(128, k, 16, 2)
        report("cfg4", m, k, u, w, inf, 0, 2, reps, flush, dt)
    m3 = M3.generate_cube(32)
    vp = F3.VectorPotential(4, 5)
    u = F3.interpolate_curl3(m3, 3, vp)
    w = F3.transfer_I3_host(m3, 3, u)
    inf = F3.inflow_values3(m3, 3, vp)
    dt = 0.1 * m3.h_min() / (9 * F3.max_speed3_host(m3, 3, u))
    report("cfg5", m3, 3, u, w, inf, 20, 3, max(5, reps // 4), flush, dt)


if __name__ == "__main__":
    main()
