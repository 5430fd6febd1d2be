"""GPU parity for the 3D (tetrahedra) path, BASELINE cfg5 (through the C ABI)."""

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import convection3d as O3  # noqa: E402
from oracle import port as P  # noqa: E402
from paper_1508_04245_b200 import basis3d as B3  # noqa: E402
from paper_1508_04245_b200 import fields3d as F3  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402

APPLY_TOL = 1e-12
SUBSTEP_TOL = 1e-10


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("name", ["k1", "k2", "k3", "k4"])
def test_apply3d_vs_golden(name):
    g = load_golden(f"conv3d_{name}.npz")
    m = M3.generate_cube(int(g["n"]))
    k = int(g["k"])
    op = ConvectionOperator(m, k)
    r = op.apply(dev(g["u"]), dev(g["w"]), dev(g["inflow"]))
    assert rel(r, g["r_ld"]) < APPLY_TOL and rel(r, g["r"]) < APPLY_TOL
    rr = op.apply(dev(g["u"]), dev(g["w_rand"]), dev(g["inflow"]))
    assert rel(rr, g["r_rand_ld"]) < APPLY_TOL
    # I = P coef: rounding scales with cond(BDM3 Vandermonde) (866 at k=3, 1.2e4 at k=4)
    assert rel(op.transfer(dev(g["u"])), g["w"]) < max(1e-13, 1e-16 * B3.build_bdm3_basis(k).cond)
    f = np.random.default_rng(0).standard_normal(g["w"].shape)
    # I^T is the adjoint of I: <I^T f, u> = <f, I u>
    itf = op.transfer(dev(f), transpose=True).cpu().numpy()
    assert abs(np.sum(itf * g["u"]) - np.sum(f * g["w"])) < 1e-12 * np.abs(f * g["w"]).sum()


def test_substeps3d_vs_golden():
    g = load_golden("conv3d_k3.npz")
    m = M3.generate_cube(int(g["n"]))
    op = ConvectionOperator(m, 3)
    w = dev(g["w"])
    op.substeps(dev(g["u"]), w, float(g["dt"]), int(g["nsub"]), dev(g["inflow"]))
    assert rel(w, g["w_sub_ld"]) < SUBSTEP_TOL


def test_3d_deterministic_and_speed():
    g = load_golden("conv3d_k2.npz")
    m = M3.generate_cube(int(g["n"]))
    op = ConvectionOperator(m, 2)
    a = op.apply(dev(g["u"]), dev(g["w_rand"]), dev(g["inflow"])).cpu().numpy()
    b = op.apply(dev(g["u"]), dev(g["w_rand"]), dev(g["inflow"])).cpu().numpy()
    assert np.array_equal(a, b)
    ms = F3.max_speed3_host(m, 2, g["u"])
    assert abs(op.max_speed(dev(g["u"])) - ms) < 1e-12 * ms


@pytest.mark.slow
def test_cfg5_apply_and_20_substeps():
    """BASELINE cfg5 in full: 32^3 cubes x 6 tets, BDM_3, apply + 20 substeps."""
    m = M3.generate_cube(32)
    k = 3
    vp = F3.VectorPotential(4, 5)
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    inf = F3.inflow_values3(m, k, vp)
    op = ConvectionOperator(m, k)
    r = op.apply(dev(u), dev(w), dev(inf)).cpu().numpy()
    port = P.Port3Operator(m, k)                  # OpenMP C port of the flux-form oracle
    assert rel(r, port.apply(u, w, inf)) < APPLY_TOL
    rr = op.apply(dev(u), dev(w_rand := np.random.default_rng(3).standard_normal(w.shape)), dev(inf))
    assert rel(rr, port.apply(u, w_rand, inf)) < APPLY_TOL
    # 20 forward-Euler substeps at full size vs the port (north star: <= 1e-10)
    dt = 0.1 * m.h_min() / (k * k * op.max_speed(dev(u)))
    wd = dev(w)
    op.substeps(dev(u), wd, dt, 20, dev(inf))
    op.check_finite()
    assert rel(wd, port.substeps(u, w, dt, 20, inf)) < SUBSTEP_TOL
    # full-size invariant: constants stay put
    nbs = B3.nbs3_of(k)
    c = np.zeros_like(w)
    c[:, 0] = 1.0
    cd = dev(c)
    op.substeps(dev(u), cd, dt, 20, None)
    assert np.abs(cd.cpu().numpy() - c).max() < 1e-10


def test_cfg5_shape_substeps_small():
    m = M3.generate_cube(4)
    k = 3
    vp = F3.VectorPotential(4, 5, (0.3, 0.2, -0.5))
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    inf = F3.inflow_values3(m, k, vp)
    dt = 0.1 * m.h_min() / (k * k * F3.max_speed3_host(m, k, u))
    op = ConvectionOperator(m, k)
    wd = dev(w)
    op.substeps(dev(u), wd, dt, 20, dev(inf))
    ref = O3.substeps3(m, k, u, w, dt, 20, inf)
    assert rel(wd, ref) < SUBSTEP_TOL


def test_pdl_batch_bitwise_equals_single_substeps_3d():
    """3D substep batches use programmatic dependent launch between substeps:
    bit-identical to one-substep calls (no stale w)."""
    m = M3.generate_cube(12)
    k = 3
    vp = F3.VectorPotential(4, 5)
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    op = ConvectionOperator(m, k)
    ud = dev(u)
    n, dt = 12, 1e-4
    batch = op.substeps(ud, dev(w), dt, n)
    one = dev(w)
    for _ in range(n):
        one = op.substeps(ud, one, dt, 1)
    assert torch.equal(batch, one)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_wind_inflow_20_substeps_vs_port(k):
    """Inflow faces (uniform wind through the cube): apply + 20 substeps vs the C port."""
    m = M3.generate_cube(8)
    vp = F3.VectorPotential(3, 11, (0.6, -0.3, 0.4))
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    inf = F3.inflow_values3(m, k, vp)
    op = ConvectionOperator(m, k)
    port = P.Port3Operator(m, k)
    assert rel(op.apply(dev(u), dev(w), dev(inf)), port.apply(u, w, inf)) < APPLY_TOL
    dt = 0.1 * m.h_min() / (k * k * op.max_speed(dev(u)))
    wd = dev(w)
    op.substeps(dev(u), wd, dt, 20, dev(inf))
    assert rel(wd, port.substeps(u, w, dt, 20, inf)) < SUBSTEP_TOL
