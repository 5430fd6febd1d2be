"""CPU: the 3D OpenMP C port (oracle/conv3d_port.c, the full-size cfg5
checker) against the numpy oracles of oracle/convection3d.py — the
long-double flux form and the physical-coordinate textbook form."""

import numpy as np
import pytest

from oracle import convection3d as O3
from oracle import port as P
from paper_1508_04245_b200 import fields3d as F3
from paper_1508_04245_b200 import mesh3d as M3


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_port3_apply_matches_oracles(k):
    m = M3.generate_cube(3)
    vp = F3.VectorPotential(3, 5, (0.3, 0.2, -0.5))
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    inf = F3.inflow_values3(m, k, vp)
    op = P.Port3Operator(m, k, threads=2)
    for ww in (w, np.random.default_rng(k).standard_normal(w.shape)):
        r = op.apply(u, ww, inf)
        assert rel(r, O3.apply_convection3_flux_form(m, k, u, ww, inf).astype(float)) < 1e-12
        assert rel(r, O3.apply_convection3(m, k, u, ww, inf)) < 1e-12
    # no inflow data: exterior = own trace
    assert rel(op.apply(u, w), O3.apply_convection3_flux_form(m, k, u, w).astype(float)) < 1e-12


def test_port3_substeps_match_oracle():
    m = M3.generate_cube(3)
    k = 3
    vp = F3.VectorPotential(3, 5, (0.3, 0.2, -0.5))
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    inf = F3.inflow_values3(m, k, vp)
    dt = 0.1 * m.h_min() / (k * k * F3.max_speed3_host(m, k, u))
    a = P.Port3Operator(m, k, threads=2).substeps(u, w, dt, 5, inf)
    assert rel(a, O3.substeps3(m, k, u, w, dt, 5, inf)) < 1e-12


def test_port3_constants_invariant():
    m = M3.generate_cube(3)
    k = 2
    u = F3.interpolate_curl3(m, k, F3.VectorPotential(3, 7))    # u.n = 0 on the boundary
    c = np.zeros((m.n_elements, 3 * 10))
    c[:, 0] = 1.0
    r = P.Port3Operator(m, k, threads=2).apply(u, c)
    assert np.abs(r).max() < 1e-12
