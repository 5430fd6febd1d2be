"""bench.py — convection-apply throughput on B200 (BASELINE.json metric).

Workload (BASELINE cfg2, the config the headline metric is quoted on):
256x256 squares -> 131,072 affine triangles, BDM_4 / V_h k=4, fp64, seeded
divergence-free stream-function velocity (modes <= 16), inflow data from the
same field.  One STEP = 100 forward-Euler explicit convection substeps,
device-resident (hdgc_substeps), dt = 0.1 h / (k^2 max|u|).
Metric: DOF/s = NT * nb * substeps / step time (one substep = one apply).

Replicas only (SURVEY §8e / north star: one B200, no inter-GPU exchange):
under torchrun every rank runs an independent replica; value = total DOF over
all ranks / max-over-ranks time ("scaling": "weak").

`--impl reference` times the reference-side CPU path instead: the reference
ships no implementation of this operator, so it is the oracle's
OpenMP C port (oracle/conv_port.c, "kind": "port") on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

K_ORDER = 4
N_CELLS = 256
MODES = 16
SEED = 2
NSUB = 100
METRIC = "convection-apply DOF/s (fp64) at k=4"
UNIT = "DOF/s"


def pinned_work(k):
    """SURVEY §8(d) pinned algorithmic work per element: (flops, bytes)."""
    nb = (k + 1) * (k + 2)
    nbs = nb // 2
    nqv = [3, 7, 25, 36, 64, 81, 121, 144][k - 1]
    nf = [3, 4, 6, 7, 9, 10, 12, 13][k - 1]
    flops = 2 * (nqv * (2 * nb + 2 * nbs + 4 * nbs) + 3 * nf * ((k + 1) + 3 * nb))
    return flops, 3 * nb * 8 + 16


def _latest_profile(pattern):
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", pattern)))
    return files[-1] if files else None


def fp64_peak():
    """Measured FP64 peaks (TFLOP/s) from tools/fp64_peak_run.py on this pool
    (newest profiles/fp64_peak_r*.json, with its clock record); MEASURED_PEAKS.json
    has no fp64 entry.  Returns (max of DMMA / DFMA, DFMA alone, source)."""
    try:
        path = _latest_profile("fp64_peak_r*.json")
        with open(path) as fh:
            d = json.loads(fh.readline())
        src = f"{os.path.relpath(path, ROOT)} (measured; DMMA m8n8k4 {d['dmma_m8n8k4_tflops']}, " \
              f"DFMA {d['dfma_occ8_tflops']}, DMMA+DFMA mixed {d.get('mixed_dmma_dfma_tflops')}: one shared pipe)"
        return max(d["dfma_occ8_tflops"], d["dmma_m8n8k4_tflops"]), d["dfma_occ8_tflops"], src
    except Exception:
        return 37.2, 37.2, "nominal 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (fallback)"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback"


def workload():
    from paper_1508_04245_b200 import fields as F
    from paper_1508_04245_b200 import mesh as M
    m = M.generate_structured((0.0, 0.0, 1.0, 1.0), N_CELLS, N_CELLS)
    sf = F.StreamFunction(MODES, SEED)
    u = F.interpolate_curl(m, K_ORDER, sf)
    w = F.transfer_I_host(m, K_ORDER, u)
    inflow = F.inflow_values(m, K_ORDER, sf)
    dt = F.cfl_dt(m.h_min(), K_ORDER, F.max_speed_host(m, K_ORDER, u))
    return m, u, w, inflow, dt


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if "--impl" not in sys.argv else "gloo")
    return world, rank, local


def max_over_ranks(t: float, world: int, device: str = "cuda") -> float:
    """Max of a per-rank time over all ranks (all_reduce MAX; identity at world 1)."""
    if world <= 1:
        return t
    import torch
    import torch.distributed as dist
    tt = torch.tensor([t], dtype=torch.float64, device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def replica_value(units_per_rank: float, world: int, t_max: float) -> float:
    """Whole-job throughput of independent replicas: all ranks' units / max time."""
    return world * units_per_rank / t_max


def ncu_fp64_flop(nc: dict):
    """FP64 flops per launch actually executed (ncu: 2 dfma + dmul + dadd thread ops)."""
    try:
        cyc = float(nc["sm__cycles_elapsed.avg"]["value"])
        per = {k: float(nc[f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed"]["value"])
               for k in ("dfma", "dmul", "dadd")}
        return cyc * (2 * per["dfma"] + per["dmul"] + per["dadd"])
    except Exception:
        return None


def ncu_fp64_inst(nc: dict):
    """FP64 thread instructions per launch (dfma + dmul + dadd): each occupies one
    lane-slot of the FP64 pipe whatever its flop count, so inst/s over the
    measured DFMA instruction rate is the pipe's utilisation."""
    try:
        cyc = float(nc["sm__cycles_elapsed.avg"]["value"])
        return cyc * sum(float(nc[f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed"]["value"])
                         for k in ("dfma", "dmul", "dadd"))
    except Exception:
        return None


def bench_config(m, dt, world):
    """The `config` object of both arms (identical, so the driver can match them)."""
    nb = (K_ORDER + 1) * (K_ORDER + 2)
    return {"workload": "cfg2: unit square 256x256 -> 131072 affine triangles, BDM_4/V_h k=4, "
                        "seeded div-free stream function (modes<=16), 100 forward-Euler substeps per step",
            "elements": m.n_elements, "k": K_ORDER, "dofs_per_apply": m.n_elements * nb, "substeps_per_step": NSUB,
            "dt": dt, "l2": "flushed (512 MB write) before every timed step",
            "parallelism": f"replicas x{world}"}


def numpy_oracle_sample(n_cells=64):
    """Single-thread numpy oracle (oracle/convection.py textbook form, fp64;
    BASELINE.md §2 asks for it beside the multi-core baseline) on a bounded
    sample: cfg2's field and order on an n x n sub-mesh, one apply."""
    from threadpoolctl import threadpool_limits
    from oracle import convection as O
    from paper_1508_04245_b200 import fields as F
    from paper_1508_04245_b200 import mesh as M
    m = M.generate_structured((0.0, 0.0, 1.0, 1.0), n_cells, n_cells)
    sf = F.StreamFunction(MODES, SEED)
    u = F.interpolate_curl(m, K_ORDER, sf)
    w = F.transfer_I_host(m, K_ORDER, u)
    inflow = F.inflow_values(m, K_ORDER, sf)
    nb = (K_ORDER + 1) * (K_ORDER + 2)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        O.apply_convection(m, K_ORDER, u, w, inflow)
        t = time.perf_counter() - t0
    return {"value": m.n_elements * nb / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"one apply of oracle/convection.py (numpy, 1 thread) on {n_cells}x{n_cells} "
                      f"({m.n_elements} triangles), k={K_ORDER}, cfg2's field: {t:.2f} s"}


def run_reference(args, world, rank):
    """Reference arm: the reference ships no implementation of this operator
    (SURVEY §0), so it is the oracle's OpenMP C port (oracle/conv_port.c,
    "kind": "port") on all host cores, rank 0 only, running the SAME step as
    the GPU arm: 100 forward-Euler substeps of cfg2 per step."""
    if rank != 0:
        return
    from oracle import port as P
    P.build()
    m, u, w, inflow, dt = workload()
    threads = os.cpu_count() or 1
    op = P.PortOperator(m, K_ORDER, threads=threads)
    nb = (K_ORDER + 1) * (K_ORDER + 2)
    steps, warm = max(1, args.steps), max(1, min(args.warmup, 3))
    for _ in range(warm):
        op.substeps(u, w, dt, NSUB, inflow)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        op.substeps(u, w, dt, NSUB, inflow)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = m.n_elements * nb * NSUB / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(m, dt, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{NSUB} forward-Euler substeps of cfg2 per step (the GPU arm's step), "
                                   f"{steps} timed steps after {warm} warm-up, oracle/conv_port.c OpenMP"},
        "numpy_oracle_1thread": numpy_oracle_sample(),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline_sample(m, u, w, inflow, dt, budget_s=10.0):
    from oracle import port as P
    P.build()
    threads = os.cpu_count() or 1
    op = P.PortOperator(m, K_ORDER, threads=threads)
    nb = (K_ORDER + 1) * (K_ORDER + 2)
    op.substeps(u, w, dt, 1, inflow)          # warm
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        op.substeps(u, w, dt, 1, inflow)
        n += 1
    t = time.perf_counter() - t0
    return {"value": m.n_elements * nb * n / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} forward-Euler substeps of cfg2 (131072 tri, k=4) in {t:.1f} s, "
                      f"oracle/conv_port.c OpenMP"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    torch.cuda.set_device(local)
    from paper_1508_04245_b200.forms import ConvectionOperator

    m, u, w, inflow, dt = workload()
    op = ConvectionOperator(m, K_ORDER)
    NT = m.n_elements
    nb = (K_ORDER + 1) * (K_ORDER + 2)
    ud = torch.from_numpy(u).cuda()
    w0 = torch.from_numpy(w).cuda()
    infd = torch.from_numpy(inflow).cuda()
    wd = w0.clone()
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")   # > 126 MB L2

    def step():
        op.substeps(ud, wd, dt, NSUB, infd)

    for _ in range(max(3, args.warmup)):
        wd.copy_(w0)
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- timed region: K steps, L2 flushed before each (flush not timed)
    clocks = ClockSampler(local) if rank == 0 else None
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        wd.copy_(w0)
        flush.fill_(float(i))
        torch.cuda._sleep(200000)   # ~0.1 ms spin: the host enqueue of the step overlaps it, not the timed region
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop() if clocks else None
    step_s = [a.elapsed_time(b) * 1e-3 for a, b in ev]
    t_step = sum(step_s) / len(step_s)
    t_step = max_over_ranks(t_step, world)
    dofs_per_step = NT * nb * NSUB
    value = replica_value(dofs_per_step, world, t_step)

    # ---- average launch duration of the dominant (substep) kernel: the step is
    # one frozen-velocity prep launch + NSUB substep launches back to back on
    # this stream, so step time / NSUB bounds it from above (prep amortised in)
    k_s = t_step / NSUB

    # ---- e2e through the public API with pinned HOST buffers (H2D + 100 substeps + D2H)
    uh = torch.from_numpy(u).pin_memory().numpy()
    wh = torch.from_numpy(w).pin_memory().numpy()
    ih = torch.from_numpy(inflow).pin_memory().numpy()
    op.substeps_host(uh, wh, dt, NSUB, ih, inplace=True)
    e2e_t = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.fill_(0.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.substeps_host(uh, wh, dt, NSUB, ih, inplace=True)   # H2D u, w, inflow; NSUB substeps; D2H w
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_t)

    if rank != 0:
        return
    flops, byts = pinned_work(K_ORDER)
    peak, dfma_peak, peak_src = fp64_peak()
    achieved = NT * flops / k_s / 1e12
    traffic = None     # dram read + write bytes per launch of the substep kernel (ncu --set full)
    measured_flop = None
    measured_inst = None
    ncu_src = _latest_profile("ncu_substep_k4_r*.json")
    try:
        with open(ncu_src) as fh:
            nc = json.load(fh)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = sum(float(nc[k]["value"]) * scale[nc[k]["unit"]]
                      for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        measured_flop = ncu_fp64_flop(nc)
        measured_inst = ncu_fp64_inst(nc)
    except Exception:
        pass
    # in-stream traffic: single-pass ncu capture of a substep batch without cache
    # flushes (tools/dram_instream.py) -- what a launch moves when the L2 holds
    # what the previous launch of the batch left (alternating sweeps)
    traffic_in = None
    in_src = _latest_profile("dram_instream_k4_r*.json")
    try:
        with open(in_src) as fh:
            di = json.load(fh)
        traffic_in = di["dram_read_bytes_median"] + di["dram_write_bytes_median"]
    except Exception:
        pass
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_sample(m, u, w, inflow, dt)
        cpu["numpy_oracle_1thread"] = numpy_oracle_sample()
    hbm, hbm_src = hbm_peak()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(m, dt, world),
        "applies_per_s": world * NSUB / t_step,
        "kernel_us_per_substep": k_s * 1e6,
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     "algorithmic": f"pinned F(k=4)={flops} flop/element (SURVEY 8d) x {NT} elements per launch",
                     "ncu_fp64_flop_per_launch": measured_flop,
                     "ncu_source": os.path.relpath(ncu_src, ROOT) if ncu_src else None,
                     "hbm_frac": NT * byts / k_s / 1e9 / hbm, "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
                     # hardware fractions: what the kernel really executes / moves (ncu counters
                     # per launch) over this run's in-stream launch time
                     "hw_fp64_frac": (measured_flop / k_s / 1e12 / dfma_peak) if measured_flop else None,
                     "hw_fp64_peak_tflops": dfma_peak,
                     # FP64 pipe slots: executed dfma + dmul + dadd thread instructions per second
                     # over the measured DFMA instruction rate (peak TFLOP/s / 2)
                     "hw_fp64_pipe_frac": (measured_inst / k_s / (dfma_peak * 1e12 / 2)) if measured_inst else None,
                     "hw_dram_frac": (traffic / k_s / 1e9 / hbm) if traffic else None,
                     "traffic_over_algorithmic": (traffic / (NT * byts)) if traffic else None,
                     # the same with the in-stream (warm L2, alternating sweeps) DRAM bytes per launch
                     "traffic_instream": traffic_in,
                     "traffic_instream_source": os.path.relpath(in_src, ROOT) if in_src else None,
                     "hw_dram_frac_instream": (traffic_in / k_s / 1e9 / hbm) if traffic_in else None,
                     "traffic_instream_over_algorithmic": (traffic_in / (NT * byts)) if traffic_in else None},
        "cpu_baseline": cpu,
        "e2e": {"value": world * dofs_per_step / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(u.nbytes + w.nbytes + inflow.nbytes),
                "d2h_bytes_per_step": int(w.nbytes)},
        "gpu_launches": args.steps * (NSUB + 1),   # per step: 1 prep + NSUB substep kernels
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
