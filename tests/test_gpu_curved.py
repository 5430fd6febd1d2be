"""GPU parity on CURVED meshes (MESH:555-615):
the device path (hdgc_set_curved: block mass inverse in the update epilogues,
L2-projection transfer, per-point Piola max speed) against the curved-mesh
oracle (oracle/curved.py: physical coordinates, Newton pull-backs) through the
C ABI, for the thread (k <= 2), sum-factorised (k = 3..6) and ring (k >= 7)
kernel variants."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import curved as OC  # noqa: E402
from oracle import timeloop as OT  # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200 import timeloop as TL  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "curved.npz"))
CIRCLE = M.Circle((0.5, 0.5), 0.15)


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ring(g, n_theta=16, n_layers=3):
    m = M.generate_ring(CIRCLE, (0.0, 0.0, 1.0, 1.0), n_theta, n_layers)
    return M.curve_boundary(m, "obstacle", CIRCLE, g)


def case(k, g=3):
    m = ring(g)
    sf = F.StreamFunction(4, 11, (1.0, 0.3))
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, F.interpolate_curl(m, k, F.StreamFunction(4, 12)))
    inflow = F.inflow_values(m, k, sf)
    return m, u, w, inflow


def test_reference_fixture():
    """the fixture made on the reference's own curved mesh and polybasis"""
    m = ring(3)
    k = int(GOLD["k"])
    op = ConvectionOperator(m, k)
    assert op.curved is not None and op.curved["elems"].size == 16
    u, w, inf = (dev(GOLD[n]) for n in ("u", "w", "inflow"))
    assert rel(op.apply(u, w, inf), GOLD["r"]) < 1e-12
    assert rel(op.transfer(u), GOLD["w"]) < 1e-12
    assert rel(op.transfer(dev(GOLD["r"]), transpose=True), GOLD["r_w"]) < 1e-12
    assert rel(op.substeps(u, w.clone(), float(GOLD["dt"]), int(GOLD["nsub"]), inf), GOLD["w_sub"]) < 1e-10


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 7, 8])
def test_apply_substeps_transfer(k):
    m, u, w, inflow = case(k, g=max(2, min(k, 4)))
    op = ConvectionOperator(m, k)
    ud, wd, infd = dev(u), dev(w), dev(inflow)
    assert rel(op.apply(ud, wd, infd), OC.apply_convection(m, k, u, w, inflow)) < 1e-12
    dt = 0.2 * TL.cfl_substep(F.max_speed_host(m, k, u), m.h_min(), k)
    ref = OC.substeps(m, k, u, w, dt, 6, inflow)
    assert rel(op.substeps(ud, wd.clone(), dt, 6, infd), ref) < 1e-10
    assert rel(op.transfer(ud), OC.transfer_I(m, k, u)) < 1e-12
    r = OC.apply_convection(m, k, u, w, inflow)
    assert rel(op.transfer(dev(r), transpose=True), OC.transfer_IT(m, k, r)) < 1e-12
    # C^U u = I^T C^V(I u; I u)
    wi = OC.transfer_I(m, k, u)
    ref_w = OC.transfer_IT(m, k, OC.apply_convection(m, k, u, wi, inflow))
    assert rel(op.apply_w(ud, infd), ref_w) < 1e-11
    assert abs(op.max_speed(ud) - F.max_speed_host(m, k, u)) < 1e-12 * F.max_speed_host(m, k, u)


@pytest.mark.parametrize("k", [2, 4])
def test_propagate_and_richardson(k):
    m, u, w, inflow = case(k)
    op = ConvectionOperator(m, k)
    apply = lambda uu, v: OC.apply_convection(m, k, uu, v, inflow)  # noqa: E731
    minv = OC.mass_inverse_apply(m, k)
    dt = 0.2 * TL.cfl_substep(F.max_speed_host(m, k, u), m.h_min(), k)
    ref = OT.propagate(apply, minv, u, w, dt, 5, "ssprk2")
    wd = dev(w)
    op.propagate(dev(u), wd, dt, 5, dev(inflow), "ssprk2")
    assert rel(wd, ref) < 1e-10
    tau = 4 * dt
    ds = TL.richardson_ds(tau, F.max_speed_host(m, k, u), m.h_min(), k)
    vr, it_ref, conv_ref, _, _ = OT.richardson(apply, minv, u, w, tau, ds, rho=1e-6, max_iter=200)
    v, it, conv, _, _ = op.richardson(dev(u), dev(w), dev(np.zeros_like(w)), tau, ds, 1e-6, 200, dev(inflow))
    assert conv == conv_ref and abs(it - it_ref) <= 1
    assert rel(v, vr) < 1e-9


def test_mass_inverse_flags_and_affine_rows():
    m, u, w, inflow = case(3)
    op = ConvectionOperator(m, 3)
    mi = op.mass_inverse().cpu().numpy()
    ce = m.curved_elements()
    np.testing.assert_array_equal(mi[ce], -(np.arange(ce.size) + 1.0))
    aff = np.setdiff1d(np.arange(m.n_elements), ce)
    np.testing.assert_allclose(mi[aff], 2.0 / m.affine_det[aff], rtol=1e-15)
