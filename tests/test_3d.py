"""3D (tetrahedra, BASELINE cfg5) host pieces and oracle (CPU).

No reference code exists for 3D; the tables are pinned by
their defining properties (the 3D analogues of TPB:14-173) and the oracle by
agreement of two independent restatements (physical textbook form vs the
geometry-free flux-difference form with sign(detJ)) plus the SPEC known-answer
properties.
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import convection3d as O3
from paper_1508_04245_b200 import basis as B2
from paper_1508_04245_b200 import basis3d as B3
from paper_1508_04245_b200 import fields3d as F3
from paper_1508_04245_b200 import mesh3d as M3


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("deg", [0, 2, 5, 8, 10])
def test_tet_rule_exact(deg):
    q = B3.quad_tet(deg)
    assert (q.weights > 0).all() and abs(q.weights.sum() - 1 / 6) < 1e-15
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            for c in range(deg + 1 - a - b):
                exact = math.factorial(a) * math.factorial(b) * math.factorial(c) / math.factorial(a + b + c + 3)
                val = np.dot(q.weights, q.points[:, 0] ** a * q.points[:, 1] ** b * q.points[:, 2] ** c)
                assert abs(val - exact) < 1e-15


@pytest.mark.parametrize("k", [1, 3, 5])
def test_tet_dubiner_gram_and_ordering(k):
    q = B3.quad_tet(2 * k)
    v = B3.dubiner3_values(k, q.points)
    assert np.abs((v * q.weights[:, None]).T @ v - np.eye(v.shape[1]) / 6).max() < 1e-13
    assert np.allclose(v[:, 0], 1.0)
    degs = [sum(t) for t in B3.dubiner3_index(k)]
    assert degs == sorted(degs) and len(degs) == B3.nbs3_of(k)


def test_tet_dubiner_gradients_fd():
    pts = np.array([[0.1, 0.2, 0.3], [0.3, 0.1, 0.2], [0.05, 0.6, 0.1]])
    _, g = B3.dubiner3_values(4, pts, with_grads=True)
    h = 1e-6
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        fd = (B3.dubiner3_values(4, pts + e) - B3.dubiner3_values(4, pts - e)) / (2 * h)
        assert np.abs(fd - g[:, :, d]).max() < 1e-6


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_bdm3_dual_traces_divergence(k):
    b = B3.build_bdm3_basis(k)
    assert b.nb == 3 * B3.nbs3_of(k) and b.n_face == 4 * (k + 1) * (k + 2) // 2
    qf, qv = B2.quad_triangle(2 * k + 6), B3.quad_tet(2 * k + 6)
    fv = np.stack([b.values(B3.face_points(f, qf.points)) for f in range(4)])
    rows = B3.bdm3_functionals_applied(k, fv, b.values(qv.points), qf=qf, qv=qv)
    assert np.abs(rows - np.eye(b.nb)).max() < 1e-11 * b.cond
    st = np.array([[0.2, 0.3], [0.5, 0.1], [0.25, 0.25]])
    for f in range(4):
        vn = b.values(B3.face_points(f, st)) @ B3.TET_FACE_NORMALS[f]
        others = [j for j in range(b.nb) if not (f * (b.n_face // 4) <= j < (f + 1) * (b.n_face // 4))]
        assert np.abs(vn[:, others]).max() < 1e-10 * b.cond
    q = B3.quad_tet(2 * k + 2)
    proj = (B3.dubiner3_values(k, q.points) * q.weights[:, None]).T @ b.divergence(q.points)
    assert np.abs(proj[B3.nbs3_of(k - 1):, :]).max() < 1e-10 * b.cond


def test_cube_mesh():
    m = M3.generate_cube(4)
    assert m.n_elements == 6 * 64 and abs(m.total_volume() - 1.0) < 1e-13
    assert 0.3 < (m.affine_det > 0).mean() < 0.7          # sorted vertices flip orientation
    fe, fl = m.facet_elems, m.facet_local
    inn = fe[:, 1] >= 0
    loc = [[v for v in range(4) if v != f] for f in range(4)]
    a = np.array([m.tets[e][loc[f]] for e, f in zip(fe[inn, 0], fl[inn, 0])])
    b = np.array([m.tets[e][loc[f]] for e, f in zip(fe[inn, 1], fl[inn, 1])])
    assert np.array_equal(a, b)                           # identical face parametrisation
    assert m.boundary_facets.size == 6 * 2 * 16


@pytest.mark.parametrize("k", [1, 2, 3])
def test_curl_interpolant_divfree_conforming(k):
    m = M3.generate_cube(3)
    vp = F3.VectorPotential(3, 5, (0.5, -0.2, 0.1))
    u = F3.interpolate_curl3(m, k, vp)
    b = B3.build_bdm3_basis(k)
    q = B3.quad_tet(2 * k)
    div = np.einsum("pj,nj->np", b.divergence(q.points), u) / m.affine_det[:, None]
    assert np.abs(div).max() < 1e-11 * np.abs(u).max() / m.h_min() * k
    st = np.array([[0.2, 0.3], [0.6, 0.1]])
    fe, fl = m.facet_elems, m.facet_local
    for fi in np.nonzero(fe[:, 1] >= 0)[0][:100]:
        fl_ = []
        for s in range(2):
            T, f = fe[fi, s], fl[fi, s]
            uh = np.einsum("pjc,j->pc", b.values(B3.face_points(f, st)), u[T])
            fl_.append((m.affine_jac[T] @ uh.T).T / m.affine_det[T])
        a, bb, c = m.vertices[m.facet_vertices[fi]]
        n = np.cross(bb - a, c - a)
        assert np.abs((fl_[0] - fl_[1]) @ n).max() < 1e-12 * (1 + np.abs(fl_[0] @ n).max())


@pytest.mark.parametrize("name", ["k1", "k2", "k3", "k4"])
def test_oracle3d_forms_agree_and_golden(name):
    g = load_golden(f"conv3d_{name}.npz")
    m = M3.generate_cube(int(g["n"]))
    k = int(g["k"])
    r = O3.apply_convection3_flux_form(m, k, g["u"], g["w"], g["inflow"]).astype(float)
    assert rel(r, g["r_ld"]) < 1e-14
    assert rel(g["r"], g["r_ld"]) < 1e-12           # textbook (physical) == flux form
    assert rel(g["r_rand"], g["r_rand_ld"]) < 1e-13


def test_oracle3d_properties():
    m = M3.generate_cube(3)
    k = 2
    u = F3.interpolate_curl3(m, k, F3.VectorPotential(3, 7))      # u.n = 0 on the boundary
    nbs = B3.nbs3_of(k)
    c = np.zeros((m.n_elements, 3 * nbs))
    c[:, 0], c[:, nbs], c[:, 2 * nbs] = 1.0, -2.0, 0.5
    assert np.abs(O3.apply_convection3(m, k, u, c)).max() < 1e-11         # constants transported
    assert np.abs(O3.apply_convection3(m, k, np.zeros_like(u), c)).max() == 0.0
    rng = np.random.default_rng(3)
    for _ in range(5):
        w = rng.standard_normal(c.shape)
        assert np.sum(w * O3.apply_convection3_flux_form(m, k, u, w).astype(float)) >= -1e-11
