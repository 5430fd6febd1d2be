"""CPU checks of the time-integration restatement (oracle/timeloop.py) against
the SPEC.md timeloop examples, and of the host-side step rules."""

import math

import pytest

import numpy as np

from oracle import convection as O
from oracle import timeloop as OT
from paper_1508_04245_b200 import fields as F
from paper_1508_04245_b200 import mesh as M
from paper_1508_04245_b200 import timeloop as TL


def linear_apply(A):
    """apply(u, v) = (A v) per element row, ignoring u: a stand-in operator."""
    return lambda u, v: v @ A.T


def test_ssprk2_is_second_order_and_euler_first():
    # dv/ds = -A v on one "element" with minv = 1; exact solution expm(-A s) v0
    rng = np.random.default_rng(0)
    A = rng.standard_normal((4, 4)) * 0.3 + np.eye(4)
    v0 = rng.standard_normal((1, 4))
    lam, V = np.linalg.eig(A)
    exact = np.real(v0 @ (V @ np.diag(np.exp(-lam)) @ np.linalg.inv(V)).T)
    err = {}
    for scheme in ("euler", "ssprk2"):
        err[scheme] = [np.linalg.norm(OT.propagate(linear_apply(A), [1.0], None, v0, 1.0 / n, n, scheme) - exact)
                       for n in (20, 40, 80)]
    rate = lambda e: math.log2(e[1] / e[2])  # noqa: E731
    assert 0.9 < rate(err["euler"]) < 1.1
    assert 1.9 < rate(err["ssprk2"]) < 2.1


def test_extrapolated_velocity():
    u0, u1 = np.ones((3, 2)), 3 * np.ones((3, 2))
    assert np.allclose(OT.velocity_at(2.0, u1, u0, 0.0, 1.0), 5.0)   # linear through (0,1), (1,3)
    assert OT.velocity_at(7.0, u1) is u1                              # frozen


def test_richardson_trivial_examples():
    # conv = 0, ds = 1 -> 1 iteration, v = g;  tau = 0 -> v = g regardless of conv
    rng = np.random.default_rng(1)
    g = rng.standard_normal((5, 6))
    zero = lambda u, v: np.zeros_like(v)  # noqa: E731
    v, it, conv, _, _ = OT.richardson(zero, np.ones(5), None, g, tau=0.7, ds=1.0)
    assert conv and it == 1 and np.array_equal(v, g)
    A = rng.standard_normal((6, 6))
    v, it, conv, _, _ = OT.richardson(linear_apply(A), np.ones(5), None, g, tau=0.0, ds=1.0)
    assert conv and it == 1 and np.array_equal(v, g)
    # non-convergence is flagged with the last iterate returned
    v, it, conv, r0, rn = OT.richardson(linear_apply(A + 5 * np.eye(6)), np.ones(5), None, g, tau=1.0,
                                        ds=0.01, rho=1e-8, max_iter=3)
    assert not conv and it == 3 and rn > 1e-8 * r0


def test_richardson_solves_the_implicit_problem():
    # v + tau M^-1 C v = g on a real mesh with the oracle apply (no inflow: C positive semi-definite)
    m = M.generate_structured((0, 0, 1, 1), 4, 4)
    k = 2
    sf = F.StreamFunction(4, 3)
    u = F.interpolate_curl(m, k, sf)
    minv = O.mass_inverse(m)
    apply = lambda uu, v: O.apply_convection_flux_form(m, k, uu, v, dtype=np.float64)  # noqa: E731
    g = np.random.default_rng(2).standard_normal((m.n_elements, (k + 1) * (k + 2)))
    tau = 0.2 * TL.cfl_substep(F.max_speed_host(m, k, u), m.h_min(), k)
    ds = TL.richardson_ds(tau, F.max_speed_host(m, k, u), m.h_min(), k)
    v, it, conv, r0, rn = OT.richardson(apply, minv, u, g, tau, ds, rho=1e-10, max_iter=400)
    assert conv and it > 1
    res = g - v - tau * minv[:, None] * apply(u, v)
    assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(g) * 1.0001


def test_propagate_constants_and_dissipativity():
    # constants invariant under div-free convection without inflow; norm non-increasing
    m = M.generate_structured((0, 0, 1, 1), 4, 4)
    k = 2
    u = F.interpolate_curl(m, k, F.StreamFunction(4, 5))
    u_prev = F.interpolate_curl(m, k, F.StreamFunction(4, 6))
    minv = O.mass_inverse(m)
    apply = lambda uu, v: O.apply_convection_flux_form(m, k, uu, v, dtype=np.float64)  # noqa: E731
    nbs = (k + 1) * (k + 2) // 2
    const = np.zeros((m.n_elements, 2 * nbs))
    const[:, 0], const[:, nbs] = 1.3, -0.4   # Dubiner mode 0 is constant
    ds = 0.5 * TL.cfl_substep(F.max_speed_host(m, k, u), m.h_min(), k)
    for scheme in ("euler", "ssprk2"):
        out = OT.propagate(apply, minv, u, const, ds, 5, scheme, u_prev, -1e-3, 0.0, 0.0)
        assert np.abs(out - const).max() < 1e-10
    w = F.transfer_I_host(m, k, u)
    mass = 1.0 / minv
    nrm = lambda x: float(np.sum(mass[:, None] * x * x))  # noqa: E731
    out = OT.propagate(apply, minv, u, w, ds, 10, "ssprk2")
    assert nrm(out) <= nrm(w) * (1 + 1e-8)


def test_step_rules():
    assert TL.richardson_ds(0.0, 2.0, 0.1, 2) == 1.0
    assert TL.richardson_ds(1.0, 0.0, 0.1, 2) == 1.0          # zero velocity: full step
    dtc = TL.cfl_substep(2.0, 0.1, 2)
    assert abs(TL.richardson_ds(1e6, 2.0, 0.1, 2) * 1e6 - dtc) < 1e-6 * dtc


def test_cfl_substep_spec_examples():
    """ds = safety h_min / ((2k+1) u_max); u_max -> 0 gives the
    interval; halving h_min halves ds."""
    assert TL.cfl_substep(1.0, 0.1, 2, 0.5) == pytest.approx(0.01, rel=1e-15)
    assert TL.cfl_substep(0.0, 0.1, 2, 0.5, interval=0.25) == 0.25
    assert TL.cfl_substep(1.0, 0.05, 2, 0.5) == pytest.approx(0.005, rel=1e-15)


def test_propagate_convection_defaults_to_ssprk2():
    import inspect
    assert inspect.signature(TL.propagate_convection).parameters["scheme"].default == "ssprk2"
