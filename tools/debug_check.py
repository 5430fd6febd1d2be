"""Race / sync / bounds check without compute-sanitizer (closed on the GPU
pool): run every kernel family with the release library and with the
HDGC_DEBUG build (tools/variants/debug, `python tools/build_variant.py debug
-DHDGC_DEBUG`) and compare the outputs bitwise.

The debug build poisons each CTA's shared memory with NaN at entry, delays
CTAs and warps by pseudo-random amounts (reordering the CTA schedule and
skewing the warps of a CTA against each other) and bounds-checks neighbour
indices with device asserts (common.cuh, hdgc_debug_prologue).  A read of
unwritten smem, a missing barrier / mbarrier / PDL wait, or a cross-CTA race
changes the result; an out-of-range index traps.  Every case also runs twice
per library (run-to-run determinism).

  python tools/debug_check.py            # both libraries, prints a JSON summary
  python tools/debug_check.py split      # the same for the k = 2 component-split kernel
                                         # (HDGC_SPLIT=1; ragged and many-wave meshes)
  python tools/debug_check.py run OUT.npz  # (internal) one library, HDGC_LIB selects it
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "tools", "variants", "debug", "libhdgconv.so")


def run(out):
    import torch
    sys.path.insert(0, ROOT)
    from paper_1508_04245_b200 import fields as F
    from paper_1508_04245_b200 import fields3d as F3
    from paper_1508_04245_b200 import mesh as M
    from paper_1508_04245_b200 import mesh3d as M3
    from paper_1508_04245_b200.forms import ConvectionOperator

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()   # noqa: E731
    res = {}
    if os.environ.get("HDGC_SPLIT") == "1":   # split mode: k = 2 frozen-velocity batches only
        for nx, ny in ((7, 5), (24, 24), (96, 96)):
            m = M.generate_structured((0, 0, 1.3, 0.7), nx, ny)
            sf = F.StreamFunction(4, 1, (1.0, 0.3))
            u = F.interpolate_curl(m, 2, sf)
            w = F.transfer_I_host(m, 2, u)
            inf = F.inflow_values(m, 2, sf)
            op = ConvectionOperator(m, 2)
            ud, wd, infd = dev(u), dev(w), dev(inf)
            dt = F.cfl_dt(m.h_min(), 2, F.max_speed_host(m, 2, u))
            for rep in range(2):
                tag = f"split{nx}x{ny}"
                res[f"{tag}_sub_{rep}"] = op.substeps(ud, wd.clone(), dt, 12, infd).cpu().numpy()
                a = wd.clone()
                op.propagate(ud, a, 0.5 * dt, 6, infd, "ssprk2")
                res[f"{tag}_rk2_{rep}"] = a.cpu().numpy()
                v, it, conv, _, _ = op.richardson(ud, wd, torch.zeros_like(wd), 5 * dt, 0.3, 1e-4, 40, infd)
                res[f"{tag}_rich_{rep}"] = v.cpu().numpy()
                res[f"{tag}_richit_{rep}"] = np.array([it])
            op.check_finite()
        torch.cuda.synchronize()
        np.savez(out, **res)
        return
    for k in range(1, 9):
        for modal in ([False, True] if 4 <= k <= 6 else [False]):
            os.environ["HDGC_MODAL"] = str(k) if modal else "0"
            n = 24 if k <= 4 else 12
            m = M.generate_structured((0, 0, 1, 1), n, n)
            sf = F.StreamFunction(4, 1, (1.0, 0.3))
            u = F.interpolate_curl(m, k, sf)
            w = F.transfer_I_host(m, k, u)
            inf = F.inflow_values(m, k, sf)
            op = ConvectionOperator(m, k)
            ud, wd, infd = dev(u), dev(w), dev(inf)
            dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
            tag = f"k{k}{'m' if modal else ''}"
            for rep in range(2):
                res[f"{tag}_apply_{rep}"] = op.apply(ud, wd, infd).cpu().numpy()
                res[f"{tag}_sub_{rep}"] = op.substeps(ud, wd.clone(), dt, 12, infd).cpu().numpy()
                v, it, conv, _, _ = op.richardson(ud, wd, torch.zeros_like(wd), 5 * dt, 0.3, 1e-4, 40, infd)
                res[f"{tag}_rich_{rep}"] = v.cpu().numpy()
                res[f"{tag}_richit_{rep}"] = np.array([it])
                res[f"{tag}_w_{rep}"] = op.apply_w(ud, infd).cpu().numpy()
            op.check_finite()
    os.environ["HDGC_MODAL"] = "0"
    for k, n in ((1, 3), (2, 3), (3, 3), (4, 3), (3, 10), (2, 8)):
        m = M3.generate_cube(n)
        vp = F3.VectorPotential(3, 5, (0.3, 0.2, -0.5))
        u = F3.interpolate_curl3(m, k, vp)
        w = F3.transfer_I3_host(m, k, u)
        inf = F3.inflow_values3(m, k, vp)
        op = ConvectionOperator(m, k)
        ud, wd, infd = dev(u), dev(w), dev(inf)
        for rep in range(2):
            res[f"3d{k}n{n}_apply_{rep}"] = op.apply(ud, wd, infd).cpu().numpy()
            res[f"3d{k}n{n}_sub_{rep}"] = op.substeps(ud, wd.clone(), 1e-4, 6, infd).cpu().numpy()
        op.check_finite()
    torch.cuda.synchronize()
    np.savez(out, **res)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "run":
        run(sys.argv[2])
        return
    env = dict(os.environ)
    env.pop("HDGC_LIB", None)
    env.pop("HDGC_SPLIT", None)
    if len(sys.argv) > 1 and sys.argv[1] == "split":
        env["HDGC_SPLIT"] = "1"
    subprocess.check_call([sys.executable, __file__, "run", "/tmp/dbg_release.npz"], env=env)
    env["HDGC_LIB"] = DEBUG_LIB
    rc = subprocess.call([sys.executable, __file__, "run", "/tmp/dbg_debug.npz"], env=env)
    summary = {"debug_run_rc": rc}
    if rc == 0:
        a, b = np.load("/tmp/dbg_release.npz"), np.load("/tmp/dbg_debug.npz")
        bad_rep = [n for n in a.files if n.endswith("_1") and not np.array_equal(a[n], a[n[:-2] + "_0"])]
        bad_dbg = [n for n in a.files if not np.array_equal(a[n], b[n])]
        nonfinite = [n for n in b.files if not np.all(np.isfinite(b[n]))]
        summary.update({"outputs": len(a.files), "release_run_to_run_differs": bad_rep,
                        "debug_vs_release_differs": bad_dbg, "debug_nonfinite": nonfinite,
                        "max_abs_diff": max(float(np.max(np.abs(a[n] - b[n]))) for n in a.files)})
    summary["ok"] = rc == 0 and not summary.get("release_run_to_run_differs") and \
        not summary.get("debug_vs_release_differs") and not summary.get("debug_nonfinite")
    print(json.dumps(summary))
    sys.exit(0 if summary["ok"] else 1)


if __name__ == "__main__":
    main()
