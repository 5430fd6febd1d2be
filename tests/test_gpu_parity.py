"""GPU parity: the CUDA path (through the C ABI) vs the oracle.

Tolerances are the north star's: relative l2 <= 1e-12 per apply, <= 1e-10
after 100 substeps (BASELINE.json north_star).  The reference for small cases
is the committed golden vectors computed on the REFERENCE's tables
(tests/golden); at BASELINE's full sizes it is the oracle's C port
(flux-difference form, fp64, pinned to long double by test_oracle.py).
"""

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import convection as O  # noqa: E402
from oracle import port as P  # noqa: E402
from paper_1508_04245_b200 import basis as B  # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200.forms import (ConvectionData, ConvectionOperator, FEField, FESpace,  # noqa: E402
                                         apply_convection, apply_convection_W, apply_transfer)
from paper_1508_04245_b200.timeloop import propagate_convection  # noqa: E402

APPLY_TOL = 1e-12
SUBSTEP_TOL = 1e-10
CASES = ["cfg1"] + [f"sweep_k{k}" for k in range(1, 9)] + ["jit_k3", "jit_k6", "sub_k4"]


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _case(name):
    g = load_golden(f"conv_{name}.npz")
    m = M.build_mesh(g["vertices"], g["triangles"])
    inflow = g["inflow"] if "inflow" in g.files else None
    return g, m, int(g["k"]), inflow


@pytest.mark.parametrize("name", CASES)
def test_apply_vs_golden(name):
    g, m, k, inflow = _case(name)
    op = ConvectionOperator(m, k)
    infd = None if inflow is None else dev(inflow)
    r = op.apply(dev(g["u"]), dev(g["w"]), infd)
    assert rel(r, g["r_ld"]) < APPLY_TOL
    assert rel(r, g["r"]) < APPLY_TOL          # the textbook-form golden too
    rr = op.apply(dev(g["u"]), dev(g["w_rand"]), infd)
    assert rel(rr, g["r_rand_ld"]) < APPLY_TOL


@pytest.mark.parametrize("name", ["jit_k3", "jit_k6", "sub_k4"])
def test_substeps_vs_golden(name):
    g, m, k, inflow = _case(name)
    op = ConvectionOperator(m, k)
    w = dev(g["w"])
    op.substeps(dev(g["u"]), w, float(g["dt"]), int(g["nsub"]), None if inflow is None else dev(inflow))
    assert rel(w, g["w_sub_ld"]) < SUBSTEP_TOL
    assert rel(w, g["w_sub"]) < SUBSTEP_TOL


@pytest.mark.parametrize("name", ["cfg1", "sweep_k5", "jit_k6"])
def test_transfer_and_apply_w(name):
    g, m, k, inflow = _case(name)
    op = ConvectionOperator(m, k)
    assert rel(op.transfer(dev(g["u"])), g["w"]) < 1e-13
    f = np.random.default_rng(0).standard_normal(g["w"].shape)
    assert rel(op.transfer(dev(f), transpose=True), O.transfer_IT(m, k, f)) < 1e-13
    infd = None if inflow is None else dev(inflow)
    rw = op.apply_w(dev(g["u"]), infd).cpu().numpy()
    # I^T applied to the device's own r_V: checks the fused I^T epilogue alone
    rv = op.apply(dev(g["u"]), op.transfer(dev(g["u"])), infd).cpu().numpy()
    assert rel(rw, O.transfer_IT(m, k, rv)) < 1e-13
    # end to end vs the golden r_V: I^T has condition number ~cond(BDM Vandermonde)
    # (97..1549 for k=3..8), so the 1e-12 apply bound maps to cond * 1e-12 here
    cond = B.build_bdm_basis(k).cond
    assert rel(rw, O.transfer_IT(m, k, g["r_ld"])) < APPLY_TOL * cond


def test_reference_named_entry_points():
    g, m, k, inflow = _case("jit_k3")
    sp = FESpace(m, "Hdiv", k)
    uf = FEField(sp, g["u"])
    r = apply_convection(uf, g["w"], ConvectionData(inflow=inflow))     # numpy in -> numpy out
    assert isinstance(r, np.ndarray) and rel(r, g["r_ld"]) < APPLY_TOL
    rw = apply_convection_W(uf, ConvectionData(inflow=inflow))
    assert rel(rw, O.transfer_IT(m, k, g["r_ld"])) < APPLY_TOL * B.build_bdm_basis(k).cond
    assert rel(apply_transfer("I", g["u"], sp), g["w"]) < 1e-13
    v, nsub, ds = propagate_convection(g["w"], 0.0, float(g["dt"]) * int(g["nsub"]), uf,
                                       ConvectionData(inflow=inflow), dt=float(g["dt"]), scheme="euler")
    assert nsub == int(g["nsub"]) and rel(v, g["w_sub_ld"]) < SUBSTEP_TOL


def test_host_variants_match_device():
    g, m, k, inflow = _case("sub_k4")
    op = ConvectionOperator(m, k)
    rd = op.apply(dev(g["u"]), dev(g["w"]), dev(inflow)).cpu().numpy()
    rh = op.apply_host(g["u"], g["w"], inflow)
    assert np.array_equal(rd, rh)
    wh = op.substeps_host(g["u"], g["w"], float(g["dt"]), int(g["nsub"]), inflow)
    assert rel(wh, g["w_sub_ld"]) < SUBSTEP_TOL
    # in place on a pinned host buffer (the bench's e2e path): same bits
    wp = torch.from_numpy(np.array(g["w"])).pin_memory().numpy()
    out = op.substeps_host(g["u"], wp, float(g["dt"]), int(g["nsub"]), inflow, inplace=True)
    assert out is wp and np.array_equal(wp, wh)


def test_deterministic_bitwise():
    g, m, k, inflow = _case("jit_k6")
    op = ConvectionOperator(m, k)
    a = op.apply(dev(g["u"]), dev(g["w_rand"]), dev(inflow)).cpu().numpy()
    for _ in range(3):
        b = op.apply(dev(g["u"]), dev(g["w_rand"]), dev(inflow)).cpu().numpy()
        assert np.array_equal(a, b)


def test_max_speed_and_mass():
    m = M.generate_jittered(16, 0.2, 2)
    k = 4
    u = F.interpolate_curl(m, k, F.StreamFunction(6, 3, (1.0, 0.3)))
    op = ConvectionOperator(m, k)
    assert abs(op.max_speed(dev(u)) - F.max_speed_host(m, k, u)) < 1e-12 * F.max_speed_host(m, k, u)
    assert rel(op.mass_inverse(), O.mass_inverse(m)) < 1e-15


def test_edge_cases():
    # single element, all facets on the boundary, with and without inflow
    m = M.build_mesh(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]))
    for k in (1, 4, 8):
        op = ConvectionOperator(m, k)
        rng = np.random.default_rng(k)
        u = rng.standard_normal((1, B.nb_of(k)))
        w = rng.standard_normal((1, B.nb_of(k)))
        inf = rng.standard_normal((3, B.facet_rule(k).weights.size, 2))
        for data in (None, inf):
            ref = O.apply_convection_flux_form(m, k, u, w, data).astype(float)
            assert rel(op.apply(dev(u), dev(w), None if data is None else dev(data)), ref) < APPLY_TOL
        # zero velocity -> zero output
        assert np.abs(op.apply(dev(np.zeros_like(u)), dev(w)).cpu().numpy()).max() == 0.0
    # bad arguments fail loudly
    with pytest.raises(ValueError):
        op.apply(dev(np.zeros((2, B.nb_of(8)))), dev(np.zeros((2, B.nb_of(8)))))
    with pytest.raises(RuntimeError):
        w = dev(np.zeros((1, B.nb_of(8))))
        op.apply(w, w, out=w)


# ---------------------------------------------------------------------------
# BASELINE full sizes vs the oracle's C port

def _full(n, k, modes, seed, wind=(0.0, 0.0), jitter=None):
    m = M.generate_jittered(n, 0.2, jitter) if jitter is not None else M.generate_structured((0, 0, 1, 1), n, n)
    sf = F.StreamFunction(modes, seed, wind)
    u = F.interpolate_curl(m, k, sf)
    return m, sf, u, F.transfer_I_host(m, k, u), F.inflow_values(m, k, sf)


def test_cfg2_apply_and_100_substeps():
    m, sf, u, w, inf = _full(256, 4, 16, 2)
    op = ConvectionOperator(m, k=4)
    port = P.PortOperator(m, 4)
    ud, wd, infd = dev(u), dev(w), dev(inf)
    assert rel(op.apply(ud, wd, infd), port.apply(u, w, inf)) < APPLY_TOL
    dt = F.cfl_dt(m.h_min(), 4, F.max_speed_host(m, 4, u))
    op.substeps(ud, wd, dt, 100, infd)
    ref = port.substeps(u, w, dt, 100, inf)
    assert rel(wd, ref) < SUBSTEP_TOL
    # random w, no cancellation: the textbook oracle itself agrees at full size
    x = np.random.default_rng(7).standard_normal(w.shape)
    assert rel(op.apply(ud, dev(x), infd), O.apply_convection(m, 4, u, x, inf)) < APPLY_TOL


@pytest.mark.slow
def test_cfg3_apply_and_50_substeps():
    m, sf, u, w, inf = _full(512, 6, 32, 3, (1.0, 0.3), jitter=11)
    op = ConvectionOperator(m, 6)
    port = P.PortOperator(m, 6)
    ud, wd, infd = dev(u), dev(w), dev(inf)
    assert rel(op.apply(ud, wd, infd), port.apply(u, w, inf)) < APPLY_TOL
    dt = F.cfl_dt(m.h_min(), 6, F.max_speed_host(m, 6, u))
    op.substeps(ud, wd, dt, 50, infd)
    assert rel(wd, port.substeps(u, w, dt, 50, inf)) < SUBSTEP_TOL


@pytest.mark.parametrize("k", range(1, 9))
def test_cfg4_order_sweep(k):
    m, sf, u, w, inf = _full(128, k, 16, 2)
    op = ConvectionOperator(m, k)
    r = op.apply(dev(u), dev(w), dev(inf))
    assert rel(r, P.PortOperator(m, k).apply(u, w, inf)) < APPLY_TOL


@pytest.mark.parametrize("k", [1, 2, 3, 4, 7])
def test_pdl_batch_bitwise_equals_single_substeps(k):
    """hdgc_substeps launches substeps 2..n with programmatic dependent launch
    (the next kernel stages its prep tile while the previous one drains); a
    missing dependency would read a stale w.  The batch must be bit-identical
    to n separate one-substep calls (no PDL), on a mesh with many waves."""
    m = M.generate_structured((0.0, 0.0, 1.0, 1.0), 96, 96)
    sf = F.StreamFunction(8, 2)
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    inflow = F.inflow_values(m, k, sf)
    op = ConvectionOperator(m, k)
    ud, infd = dev(u), dev(inflow)
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    n = 40
    batch = op.substeps(ud, dev(w), dt, n, infd)
    one = dev(w)
    for _ in range(n):
        one = op.substeps(ud, one, dt, 1, infd)
    assert torch.equal(batch, one)
    for _ in range(3):   # repeated batches: identical (no race on w)
        assert torch.equal(op.substeps(ud, dev(w), dt, n, infd), batch)


_AB_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from conftest import load_golden
from paper_1508_04245_b200 import mesh as M, mesh3d as M3
from paper_1508_04245_b200.forms import ConvectionOperator
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
out = []
for name in ("sweep_k4", "sweep_k5", "jit_k6", "sweep_k8"):
    g = load_golden(f"conv_{name}.npz")
    m = M.build_mesh(g["vertices"], g["triangles"])
    inf = dev(g["inflow"]) if "inflow" in g.files else None
    op = ConvectionOperator(m, int(g["k"]))
    r = op.apply(dev(g["u"]), dev(g["w_rand"]), inf).cpu().numpy()
    out.append(np.linalg.norm(r - g["r_rand_ld"]) / np.linalg.norm(g["r_rand_ld"]))
g = load_golden("conv3d_k3.npz")
op = ConvectionOperator(M3.generate_cube(int(g["n"])), 3)
r = op.apply(dev(g["u"]), dev(g["w_rand"]), dev(g["inflow"])).cpu().numpy()
out.append(np.linalg.norm(r - g["r_rand_ld"]) / np.linalg.norm(g["r_rand_ld"]))
print(" ".join(f"{x:.3e}" for x in out))
"""


def test_prep_fallback_paths_hdgc_prep_0():
    """HDGC_PREP=0 keeps the pre-tile prep paths (fused thread-per-element,
    DGEMM + rows, thread-per-element 3D) for A/B timing; they must stay at
    parity too (the default tile path is covered by the golden tests)."""
    import os
    import subprocess
    import sys
    tests = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, HDGC_PREP="0")
    res = subprocess.run([sys.executable, "-c", _AB_SCRIPT, tests], env=env, capture_output=True, text=True,
                         timeout=600, cwd=os.path.dirname(tests))
    assert res.returncode == 0, res.stderr[-2000:]
    errs = [float(x) for x in res.stdout.split()]
    assert len(errs) == 5 and max(errs) < APPLY_TOL, errs


@pytest.mark.parametrize("k", [1, 2, 3, 4, 6, 8])
def test_ragged_tail_tiles(k):
    """Element counts that are not a multiple of any tile size (7 x 5 cells =
    70 triangles; 16-element sf tiles, 32-element prep tiles, 64-thread blocks):
    apply + an 8-substep PDL batch vs the C port, with inflow data."""
    m = M.generate_structured((0.0, 0.0, 1.3, 0.7), 7, 5)
    sf = F.StreamFunction(5, 4, (0.8, -0.5))
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    inflow = F.inflow_values(m, k, sf)
    op = ConvectionOperator(m, k)
    port = P.PortOperator(m, k, threads=2)
    assert rel(op.apply(dev(u), dev(w), dev(inflow)), port.apply(u, w, inflow)) < APPLY_TOL
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    wd = op.substeps(dev(u), dev(w), dt, 8, dev(inflow))
    assert rel(wd, port.substeps(u, w, dt, 8, inflow)) < SUBSTEP_TOL


def test_zero_substeps_is_identity():
    m = M.generate_structured((0.0, 0.0, 1.0, 1.0), 4, 4)
    k = 4
    u = F.interpolate_curl(m, k, F.StreamFunction(3, 1))
    w = F.transfer_I_host(m, k, u)
    op = ConvectionOperator(m, k)
    assert torch.equal(op.substeps(dev(u), dev(w), 1e-3, 0), dev(w))


@pytest.mark.parametrize("k", [3, 4, 6, 7])
def test_shuffled_element_order_halo_paths(k):
    """Random element numbering on a jittered mesh: almost every neighbour of a
    16-element tile lies outside it, so lanes have two or three halo edges (the
    out-of-line halo rounds of facets_v2) and tiles ask for more than 32 halo
    rows (the global-memory overflow path).  Apply + 6 substeps vs the C port."""
    base = M.generate_jittered(12, 0.2, seed=3)
    perm = np.random.default_rng(11).permutation(base.n_elements)
    m = M.build_mesh(base.vertices, base.triangles[perm])
    sf = F.StreamFunction(4, 7, (1.0, 0.3))
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    inflow = F.inflow_values(m, k, sf)
    op = ConvectionOperator(m, k)
    port = P.PortOperator(m, k, threads=2)
    assert rel(op.apply(dev(u), dev(w), dev(inflow)), port.apply(u, w, inflow)) < APPLY_TOL
    wr = np.random.default_rng(5).standard_normal(w.shape)
    assert rel(op.apply(dev(u), dev(wr), dev(inflow)), port.apply(u, wr, inflow)) < APPLY_TOL
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    wd = op.substeps(dev(u), dev(w), dt, 6, dev(inflow))
    assert rel(wd, port.substeps(u, w, dt, 6, inflow)) < SUBSTEP_TOL


_SPLIT_SCRIPT = r"""
import sys, hashlib, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import port as P
from paper_1508_04245_b200 import fields as F, mesh as M, timeloop as TL
from paper_1508_04245_b200.forms import ConvectionOperator
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
k = 2
h = hashlib.sha256()
errs = []
for (nx, ny) in ((7, 5), (96, 96)):   # ragged tail tile; many CTA waves
    m = M.generate_structured((0.0, 0.0, 1.3, 0.7), nx, ny)
    sf = F.StreamFunction(5, 4, (0.8, -0.5))
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    inflow = F.inflow_values(m, k, sf)
    op = ConvectionOperator(m, k)
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    ud, infd = dev(u), dev(inflow)
    batch = op.substeps(ud, dev(w), dt, 12, infd)          # prep + 12 update kernels (PDL)
    assert torch.equal(batch, op.substeps(ud, dev(w), dt, 12, infd))
    ref = P.PortOperator(m, k, threads=2).substeps(u, w, dt, 12, inflow)
    errs.append(float(np.linalg.norm(batch.cpu().numpy() - ref) / np.linalg.norm(ref)))
    h.update(batch.cpu().numpy().tobytes())
    a = dev(w)
    op.propagate(ud, a, 0.5 * dt, 6, infd, "ssprk2")      # SUBSTEP + STAGE kernels
    h.update(a.cpu().numpy().tobytes())
    g = dev(np.random.default_rng(3).standard_normal(w.shape))
    v, it, conv, r0, rn = op.richardson(ud, g, torch.zeros_like(g), 3 * dt, dt, 1e-6, 300, infd)
    h.update(v.cpu().numpy().tobytes()); h.update(np.float64([it, r0, rn]).tobytes())
    op.check_finite()
print(h.hexdigest(), " ".join(f"{x:.3e}" for x in errs))
"""


def test_component_split_kernel_bitwise_equals_thread_kernel():
    """k = 2 frozen-velocity batches on large meshes run the component-split
    update kernel (one thread per (element, component), conv2d_thread.cuh);
    HDGC_SPLIT=1 / 0 force it on / off.  Substep batches (ragged tail tile and a
    many-wave mesh, inflow data), SSP-RK2 propagation (STAGE mode) and a
    Richardson solve must be bitwise identical between the two kernels, and the
    split batch within the substep tolerance of the C port."""
    import os
    import subprocess
    import sys
    tests = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, HDGC_SPLIT=flag)
        res = subprocess.run([sys.executable, "-c", _SPLIT_SCRIPT, tests], env=env, capture_output=True, text=True,
                             timeout=600, cwd=os.path.dirname(tests))
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(res.stdout.split())
    assert outs[0][0] == outs[1][0], outs
    assert max(float(x) for x in outs[0][1:]) < SUBSTEP_TOL, outs


def test_component_split_kernel_curved_and_oracle_cases():
    """The k = 2 curved-element batches (raw residual rows handed to the curved
    fix-up kernel, no PDL) and the Richardson-vs-oracle case again with the
    component-split kernel forced on (HDGC_SPLIT=1, read once per process)."""
    import os
    import subprocess
    import sys
    tests = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, HDGC_SPLIT="1")
    nodes = ["tests/test_gpu_curved.py::test_apply_substeps_transfer[2]",
             "tests/test_gpu_curved.py::test_propagate_and_richardson[2]",
             "tests/test_gpu_timeloop.py::test_richardson_vs_oracle[2]"]
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", *nodes],
                         env=env, capture_output=True, text=True, timeout=900, cwd=os.path.dirname(tests))
    assert res.returncode == 0 and "3 passed" in res.stdout, res.stdout[-2000:] + res.stderr[-1000:]
