"""Host basis tables vs the reference (CPU).

Two layers of pinning:
1. golden vectors written by the reference's own ``hdgflow.polybasis``
   (tests/golden/make_golden.py -> tables.npz): quadrature rules, Legendre,
   Dubiner values/gradients, BDM dual basis, at k = 1..8;
2. the reference's own test suite (pkg/tests/test_polybasis.py, TPB:14-173),
   restated against this package's basis module.
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from paper_1508_04245_b200 import basis as B

G = load_golden("tables.npz")


# ---------------------------------------------------------------------------
# 1. golden vectors from the reference

@pytest.mark.parametrize("deg", range(0, 26))
def test_quadrature_rules_bit_identical(deg):
    qi = B.quad_interval(deg)
    qt = B.quad_triangle(deg)
    assert np.array_equal(qi.points, G[f"qi{deg}_p"]) and np.array_equal(qi.weights, G[f"qi{deg}_w"])
    assert np.array_equal(qt.points, G[f"qt{deg}_p"]) and np.array_equal(qt.weights, G[f"qt{deg}_w"])


def test_legendre_golden():
    t = G["leg_t"]
    assert np.abs(B.legendre_values(10, t) - G["leg_v"]).max() < 1e-13
    assert np.abs(B.legendre_derivs(10, t) - G["leg_d"]).max() < 1e-11


@pytest.mark.parametrize("k", range(1, 9))
def test_dubiner_golden(k):
    pts = np.vstack([B.quad_triangle(3 * k + 1).points, G["rand_pts"]])
    v, g = B.dubiner_values(k, pts, with_grads=True)
    gv, gg = G[f"dub{k}_v"], G[f"dub{k}_g"]
    assert np.abs(v - gv).max() <= 1e-13 * max(1.0, np.abs(gv).max())
    assert np.abs(g - gg).max() <= 1e-13 * max(1.0, np.abs(gg).max())


@pytest.mark.parametrize("k", range(1, 9))
def test_bdm_golden(k):
    b = B.build_bdm_basis(k)
    gc = G[f"bdm{k}_coef"]
    tol = 1e-15 * float(G[f"bdm{k}_cond"]) * np.abs(gc).max()
    assert np.abs(b.coef - gc).max() <= max(tol, 1e-14)
    assert np.abs(b.vandermonde - G[f"bdm{k}_V"]).max() < 1e-12
    assert abs(b.cond - float(G[f"bdm{k}_cond"])) < 1e-8 * b.cond
    gvals = G[f"bdm{k}_vals"]
    assert np.abs(b.values(G["rand_pts"]) - gvals).max() <= 1e-12 * max(1.0, np.abs(gvals).max())


# ---------------------------------------------------------------------------
# 2. the reference's own polybasis tests (TPB), restated

def _tri_monomial(a, b):
    return math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)


def test_interval_weight_sum():                                   # TPB:15-19
    for deg in range(25):
        q = B.quad_interval(deg)
        assert abs(q.weights.sum() - 1.0) < 1e-14 and (q.weights > 0).all()


def test_interval_two_point_cubic():                              # TPB:21-25
    q = B.quad_interval(3)
    assert len(q.points) == 2 and abs(np.dot(q.weights, q.points ** 3) - 0.25) < 1e-15


@pytest.mark.parametrize("deg", range(0, 22))
def test_triangle_exactness(deg):                                 # TPB:27-35
    q = B.quad_triangle(deg)
    assert (q.weights > 0).all() and abs(q.weights.sum() - 0.5) < 1e-13
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            val = np.dot(q.weights, q.points[:, 0] ** a * q.points[:, 1] ** b)
            assert abs(val - _tri_monomial(a, b)) < 1e-13


def test_unknown_domain():                                        # TPB:42-44
    with pytest.raises(ValueError):
        B.quad_rule("square", 2)


def test_legendre_orthonormal_and_closed_form():                  # TPB:48-66
    v = B.legendre_values(3, np.array([0.75]))
    assert abs(v[0, 2] / math.sqrt(5.0) + 0.125) < 1e-14
    q = B.quad_interval(12)
    v = B.legendre_values(6, q.points)
    assert np.abs((v * q.weights[:, None]).T @ v - np.eye(7)).max() < 1e-12


def test_legendre_derivative_fd():                                # TPB:68-73
    t = np.linspace(0.05, 0.95, 7)
    h = 1e-6
    fd = (B.legendre_values(5, t + h) - B.legendre_values(5, t - h)) / (2 * h)
    assert np.abs(B.legendre_derivs(5, t) - fd).max() < 1e-7


@pytest.mark.parametrize("k", [1, 3, 6])
def test_dubiner_gram(k):                                         # TPB:77-84
    q = B.quad_triangle(2 * k)
    v = B.dubiner_values(k, q.points)
    assert np.abs((v * q.weights[:, None]).T @ v - 0.5 * np.eye(v.shape[1])).max() < 1e-12


def test_dubiner_member0_and_ordering():                          # TPB:86-96
    q = B.quad_triangle(3)
    assert np.allclose(B.dubiner_values(2, q.points)[:, 0], 1.0)
    degs = [i + j for i, j in B.dubiner_index(3)]
    assert degs == sorted(degs) and len(degs) == 10


def test_dubiner_gradients_fd():                                  # TPB:98-111
    rng = np.random.default_rng(0)
    pts = rng.random((20, 2)) * 0.45 + 0.05
    pts[:, 1] *= 1.0 - pts[:, 0]
    _, g = B.dubiner_values(4, pts, with_grads=True)
    h = 1e-6
    for d in range(2):
        dp, dm = pts.copy(), pts.copy()
        dp[:, d] += h
        dm[:, d] -= h
        fd = (B.dubiner_values(4, dp) - B.dubiner_values(4, dm)) / (2 * h)
        assert np.abs(g[:, :, d] - fd).max() < 1e-6


def test_dubiner_collapsed_vertex_finite():
    # the homogeneous recurrence is valid at (0, 1), where the collapsed map is singular
    v, g = B.dubiner_values(5, np.array([[0.0, 1.0]]), with_grads=True)
    assert np.isfinite(v).all() and np.isfinite(g).all()


def test_eval_orthobasis_dispatch():                              # TPB:113-117
    assert B.eval_orthobasis("DubinerTri", 2, np.array([[0.25, 0.25]])).shape == (1, 6)
    with pytest.raises(ValueError):
        B.eval_orthobasis("MonomialTri", 2, np.array([[0.25, 0.25]]))


def test_bdm_dimension_counts():                                  # TPB:121-126
    b1, b3 = B.build_bdm_basis(1), B.build_bdm_basis(3)
    assert (b1.nb, b1.n_edge, b1.n_interior) == (6, 6, 0)
    assert (b3.nb, b3.n_edge, b3.n_interior) == (20, 12, 8)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 8])
def test_bdm_dual_kronecker(k):                                   # TPB:128-143
    b = B.build_bdm_basis(k)
    qe, qv = B.quad_interval(2 * k + 8), B.quad_triangle(2 * k + 8)
    ev = np.stack([b.values(B.ref_edge_points(e, qe.points)) for e in range(3)])
    rows = B.bdm_functionals_applied(k, ev, b.values(qv.points), qe=qe, qv=qv)
    assert np.abs(rows - np.eye(b.nb)).max() < 1e-10


@pytest.mark.parametrize("k", [2, 3, 4])
def test_bdm_interior_zero_normal_trace(k):                       # TPB:145-152
    b = B.build_bdm_basis(k)
    t = np.linspace(0.1, 0.9, 7)
    for e in range(3):
        vn = b.values(B.ref_edge_points(e, t)) @ B.REF_EDGE_NORMALS[e]
        assert np.abs(vn[:, b.n_edge:]).max() < 1e-9


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_bdm_divergence_in_pkm1(k):                               # TPB:154-164
    b = B.build_bdm_basis(k)
    q = B.quad_triangle(2 * k + 2)
    proj = (B.dubiner_values(k, q.points) * q.weights[:, None]).T @ b.divergence(q.points)
    assert np.abs(proj[k * (k + 1) // 2:, :]).max() < 1e-10


def test_bdm_degree_bounds():                                     # TPB:166-173
    with pytest.raises(ValueError):
        B.build_bdm_basis(0)
    assert np.isfinite(B.build_bdm_basis(6).cond)


@pytest.mark.parametrize("k", range(1, 9))
def test_divergence_modal_table(k):
    """Device table: div of each member in the P_{k-1} Dubiner modes."""
    b = B.build_bdm_basis(k)
    q = B.quad_triangle(3 * k)
    M = B.bdm_divergence_modal(k)
    rec = B.dubiner_values(k - 1, q.points) @ M
    ref = b.divergence(q.points)
    assert np.abs(rec - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


def test_device_rules():
    nqv = [3, 7, 25, 36, 64, 81, 121, 144]
    nf = [3, 4, 6, 7, 9, 10, 12, 13]
    for k in range(1, 9):
        assert B.volume_rule(k).weights.size == nqv[k - 1]
        assert B.facet_rule(k).weights.size == nf[k - 1]


@pytest.mark.parametrize("k", range(1, 9))
def test_dubiner_edge_trace_structure(k):
    """The structure csrc/conv2d_sf.cuh's facets_v2 builds on (and sf_setup
    re-checks on the uploaded tables): with R_e[l][m] = int_0^1 D_m(x_e(t)) L_l(t) dt,
    R_0 is zero unless l == i, R_1 is zero for l > i + j, and
    R_2[l][m] = (-1)^(i+l) R_1[l][m]   (m = (i, j) in dubiner_index order)."""
    qf = B.facet_rule(k)
    L = B.legendre_values(k, qf.points)                      # (nf, k+1)
    R = [np.einsum("q,qm,ql->lm", qf.weights, B.dubiner_values(k, B.ref_edge_points(e, qf.points)), L)
         for e in range(3)]
    for m, (i, j) in enumerate(B.dubiner_index(k)):
        for l in range(k + 1):
            if l != i:
                assert abs(R[0][l, m]) < 1e-13
            if l > i + j:
                assert abs(R[1][l, m]) < 1e-13
            assert abs(R[2][l, m] - (-1) ** (i + l) * R[1][l, m]) < 1e-13
    # the traces are exact: the expansion reproduces the point values
    for e in range(3):
        assert np.allclose(L @ R[e], B.dubiner_values(k, B.ref_edge_points(e, qf.points)), atol=1e-12)


@pytest.mark.parametrize("k", [3, 4, 5, 6, 7, 8])
def test_mirror_symmetry_of_collapsed_and_facet_tables(k):
    """The device kernels evaluate the Gauss-Legendre direction in mirror pairs
    (conv2d_sf.cuh SF::SYM; sf_setup rejects tables without the symmetry):
    A_i(n-1-a) = (-1)^i A_i(a), A'_i(n-1-a) = (-1)^(i+1) A'_i(a) on the collapsed
    rule, and L_l(t_{nf-1-q}) = (-1)^l L_l(t_q) on the facet rule."""
    t = B.collapsed_tables(k)
    sg = (-1.0) ** np.arange(k + 1)
    assert np.abs(t["A"][::-1] - sg * t["A"]).max() < 1e-13
    assert np.abs(t["Ad"][::-1] + sg * t["Ad"]).max() < 1e-12
    L = B.legendre_values(k, B.facet_rule(k).points)
    assert np.abs(L[::-1] - sg * L).max() < 1e-13


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_mirror_symmetry_of_collapsed_tables_3d(k):
    """Same for the a direction of the collapsed tet rule (conv3d.cuh HDGC_3D_SYM)."""
    from paper_1508_04245_b200 import basis3d as B3
    t = B3.collapsed_tables3(k)
    sg = (-1.0) ** np.arange(k + 1)
    assert np.abs(t["A"][::-1] - sg * t["A"]).max() < 1e-13
    assert np.abs(t["Ad"][::-1] + sg * t["Ad"]).max() < 1e-12
