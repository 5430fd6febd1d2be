"""The oracle itself, pinned (CPU).

* textbook restatement (physical coordinates, facet-wise) on this package's
  tables reproduces the golden vectors computed on the REFERENCE's tables;
* the flux-difference form agrees with the textbook form (divergence
  theorem) and, in long double, is the accuracy anchor;
* the C port (fast checker / CPU baseline) agrees with both;
* the SPEC known-answer properties.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import convection as O
from oracle import port as P
from paper_1508_04245_b200 import basis as B
from paper_1508_04245_b200 import fields as F
from paper_1508_04245_b200 import mesh as M

CASES = ["cfg1"] + [f"sweep_k{k}" for k in range(1, 9)] + ["jit_k3", "jit_k6", "sub_k4"]


def _case(name):
    g = load_golden(f"conv_{name}.npz")
    m = M.build_mesh(g["vertices"], g["triangles"])
    inflow = g["inflow"] if "inflow" in g.files else None
    return g, m, int(g["k"]), inflow


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", CASES)
def test_textbook_oracle_vs_golden(name):
    g, m, k, inflow = _case(name)
    assert rel(O.apply_convection(m, k, g["u"], g["w"], inflow), g["r"]) < 1e-12
    assert rel(O.apply_convection(m, k, g["u"], g["w_rand"], inflow), g["r_rand"]) < 1e-13


@pytest.mark.parametrize("name", CASES)
def test_flux_form_vs_golden_and_textbook(name):
    g, m, k, inflow = _case(name)
    rl = O.apply_convection_flux_form(m, k, g["u"], g["w"], inflow).astype(float)
    assert rel(rl, g["r_ld"]) < 1e-13                 # our tables vs reference tables
    assert rel(g["r"], g["r_ld"]) < 1e-12             # textbook == flux form (div. theorem)
    assert rel(g["r_rand"], g["r_rand_ld"]) < 1e-13


@pytest.mark.parametrize("name", CASES)
def test_port_vs_golden(name):
    g, m, k, inflow = _case(name)
    op = P.PortOperator(m, k, threads=2)
    assert rel(op.apply(g["u"], g["w"], inflow), g["r_ld"]) < 1e-13
    assert rel(op.apply(g["u"], g["w_rand"], inflow), g["r_rand_ld"]) < 1e-13
    if "w_sub" in g.files:
        ws = op.substeps(g["u"], g["w"], float(g["dt"]), int(g["nsub"]), inflow)
        assert rel(ws, g["w_sub_ld"]) < 1e-13
        assert rel(g["w_sub"], g["w_sub_ld"]) < 1e-12


def test_port_vs_reference_tables():
    """The port with the reference's tables injected would equal the port
    with ours: tables agree to rounding (test_basis), so outputs agree."""
    g, m, k, inflow = _case("jit_k6")
    a = P.PortOperator(m, k, threads=2).apply(g["u"], g["w_rand"], inflow)
    assert rel(a, g["r_rand_ld"]) < 1e-13


def test_transfer_I_and_IT_golden():
    g, m, k, _ = _case("cfg1")
    w = O.transfer_I(m, k, g["u"])
    assert rel(w, g["w"]) < 1e-14
    assert rel(F.transfer_I_host(m, k, g["u"]), g["w"]) < 1e-14
    assert rel(O.transfer_IT(m, k, g["r"]), g["r_w"]) < 1e-13


def test_flux_form_is_the_accurate_one():
    """fp64 textbook form loses digits to cancellation on fine meshes; the
    fp64 flux form does not.  Measured against long double."""
    m = M.generate_structured((0, 0, 1, 1), 48, 48)
    k = 4
    sf = F.StreamFunction(16, 2)
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    ld = O.apply_convection_flux_form(m, k, u, w).astype(float)
    fp = O.apply_convection_flux_form(m, k, u, w, dtype=np.float64)
    tb = O.apply_convection(m, k, u, w)
    port = P.PortOperator(m, k, threads=2).apply(u, w)
    assert rel(fp, ld) < 5e-14
    assert rel(port, ld) < 5e-14
    assert rel(tb, ld) < 1e-11          # textbook: correct but less accurate
    assert rel(tb, ld) > rel(fp, ld)


# ---------------------------------------------------------------------------
# SPEC known-answer properties

@pytest.fixture(scope="module")
def closed_field():
    m = M.generate_structured((0, 0, 1, 1), 8, 8)
    k = 3
    u = F.interpolate_curl(m, k, F.StreamFunction(4, 7))   # u.n = 0 on the boundary
    return m, k, u


def test_constant_transported_exactly(closed_field):
    m, k, u = closed_field
    w = np.zeros((m.n_elements, B.nb_of(k)))
    w[:, 0] = 1.0
    w[:, B.nbs_of(k)] = -0.5
    assert np.abs(O.apply_convection(m, k, u, w)).max() < 1e-11
    assert np.abs(P.PortOperator(m, k, threads=1).apply(u, w)).max() < 1e-11


def test_zero_velocity_zero_output(closed_field):
    m, k, u = closed_field
    w = np.random.default_rng(1).standard_normal((m.n_elements, B.nb_of(k)))
    assert np.abs(O.apply_convection(m, k, np.zeros_like(u), w)).max() == 0.0


def test_quadratic_form_nonnegative(closed_field):
    m, k, u = closed_field
    rng = np.random.default_rng(2)
    op = P.PortOperator(m, k, threads=2)
    for _ in range(100):
        w = rng.standard_normal((m.n_elements, B.nb_of(k)))
        assert np.sum(w * op.apply(u, w)) >= -1e-11


def test_stability_identity_with_inflow():
    m = M.generate_jittered(8, 0.2, 4)
    k = 2
    u = F.interpolate_curl(m, k, F.StreamFunction(4, 9, (1.0, 0.3)))
    rng = np.random.default_rng(3)
    for _ in range(10):
        w = rng.standard_normal((m.n_elements, B.nb_of(k)))
        c, inflow_term = O.quadratic_form_inflow(m, k, u, w)
        assert c + inflow_term >= -1e-11


def test_transfer_embedding_and_adjoint(closed_field):
    m, k, u = closed_field
    w = F.transfer_I_host(m, k, u)
    rng = np.random.default_rng(4)
    b = B.build_bdm_basis(k)
    for _ in range(20):
        T = rng.integers(m.n_elements)
        p = rng.random(2)
        p = p if p.sum() < 1 else 1 - p
        uh = b.values(p[None])[0].T @ u[T]
        u_phys = m.affine_jac[T] @ uh / m.affine_det[T]
        wv = B.dubiner_values(k, p[None])[0] @ w[T].reshape(2, -1).T
        assert np.abs(u_phys - wv).max() < 1e-11
    f = rng.standard_normal(w.shape)
    lhs = np.sum(O.transfer_IT(m, k, f) * u)
    assert abs(lhs - np.sum(f * w)) < 1e-12 * abs(lhs) + 1e-12


def test_propagation_properties(closed_field):
    m, k, u = closed_field
    op = P.PortOperator(m, k, threads=2)
    w = np.random.default_rng(5).standard_normal((m.n_elements, B.nb_of(k)))
    assert np.array_equal(op.substeps(np.zeros_like(u), w, 1e-3, 5), w)        # C=0: identity
    c = np.zeros_like(w)
    c[:, 0] = 2.0
    assert np.abs(op.substeps(u, c, 1e-3, 10) - c).max() < 1e-10               # constants invariant
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    wi = F.transfer_I_host(m, k, u)
    w100 = op.substeps(u, wi, dt, 100)
    # upwind dissipativity: SSP-RK2 keeps ||w|| non-increasing; the
    # BASELINE's forward Euler adds O(dt^2) per step, so bound loosely
    assert np.linalg.norm(w100) <= np.linalg.norm(wi) * (1 + 1e-2)
