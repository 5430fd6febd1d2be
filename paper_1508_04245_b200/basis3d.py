"""Reference-tetrahedron tables for the 3D convection path (BASELINE cfg5).

The reference package is 2D only (SURVEY §2 "3D: none"),
so this module has no reference code to follow; it carries the 2D
conventions of ``hdgflow.polybasis`` (PB:3-13, restated in ``basis.py``) to
the tetrahedron, as SURVEY §7 item 7 and Appendix A.5 prescribe:

* reference tet ``{x, y, z >= 0, x + y + z <= 1}`` (measure 1/6), vertices
  v0 = 0, v1 = e_x, v2 = e_y, v3 = e_z; local face f is opposite vertex f;
* collapsed (Duffy) volume rule: Gauss-Legendre x Gauss-Jacobi(1,0) x
  Gauss-Jacobi(2,0), n = (degree+2)//2 points per direction;
* orthogonal tet Dubiner modes, ordered by total degree, Gram = I/6, member
  0 is the constant 1 (the 3D analogue of PB:8-9);
* BDM_k = full [P_k]^3 with a basis dual to
    - face normal moments against the 2D Dubiner modes of degree <= k on each
      face, in the face parameters (s, t) of x = p0 + s (p1 - p0) + t (p2 - p0),
      (p0, p1, p2) = the face's vertices in increasing local index, and
    - interior moments against Nedelec (first kind) N_{k-1}:
      [P_{k-2}]^3 plus x cross p for homogeneous p of degree k-2 (a maximal
      independent subset, selected greedily in a fixed order) —
  the 3D counterpart of the 2D functional set (PB:315-354; "any spanning set
  is acceptable since only the spanned space matters").
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache
from itertools import product

import numpy as np
from scipy.special import roots_jacobi, roots_legendre

from . import basis as B2

__all__ = ["TET_VERTICES", "TET_FACES", "TET_FACE_NORMALS", "TET_FACE_AREAS", "nbs3_of", "nb3_of",
           "quad_tet", "face_rule", "volume_rule3", "dubiner3_index", "dubiner3_values",
           "face_points", "BDM3Basis", "build_bdm3_basis", "bdm3_divergence_modal"]

TET_VERTICES = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
# face f = vertices other than f, in increasing local index
TET_FACES = tuple(tuple(v for v in range(4) if v != f) for f in range(4))
_S3 = 1.0 / math.sqrt(3.0)
TET_FACE_NORMALS = np.array([[_S3, _S3, _S3], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, -1.0]])
TET_FACE_AREAS = np.array([math.sqrt(3.0) / 2.0, 0.5, 0.5, 0.5])


def nbs3_of(k: int) -> int:
    return (k + 1) * (k + 2) * (k + 3) // 6


def nb3_of(k: int) -> int:
    return 3 * nbs3_of(k)


@dataclass(frozen=True)
class QuadRule3:
    points: np.ndarray    # (n, 3)
    weights: np.ndarray   # (n,)
    degree: int
    n1: int               # points per collapsed direction


def _gj01(n, alpha):
    x, w = roots_jacobi(n, alpha, 0.0)
    return 0.5 * (x + 1.0), w / 2.0 ** (alpha + 1)


@lru_cache(maxsize=None)
def quad_tet(degree: int) -> QuadRule3:
    """Collapsed tensor rule exact to `degree`: x = a(1-b)(1-c), y = b(1-c),
    z = c; Gauss-Legendre in a, Gauss-Jacobi (1,0) in b, (2,0) in c.  Point
    order: c outer, b, a inner.  Weights sum to 1/6."""
    n = max(1, (degree + 2) // 2)
    xa, wa = roots_legendre(n)
    a, wa = 0.5 * (xa + 1.0), 0.5 * wa
    b, wb = _gj01(n, 1.0)
    c, wc = _gj01(n, 2.0)
    C, Bb, A = np.meshgrid(c, b, a, indexing="ij")
    WC, WB, WA = np.meshgrid(wc, wb, wa, indexing="ij")
    pts = np.stack([(A * (1 - Bb) * (1 - C)).ravel(), (Bb * (1 - C)).ravel(), C.ravel()], axis=1)
    return QuadRule3(points=pts, weights=(WA * WB * WC).ravel(), degree=2 * n - 1, n1=n)


def volume_rule3(k: int) -> QuadRule3:
    """Device volume rule, exact for the degree 3k-1 integrand (SURVEY 8d:
    nqv = ((3k+1)//2)^3)."""
    return quad_tet(3 * k - 1)


def face_rule(k: int):
    """Facet rule on each face: quad_triangle(3k+1) in (s, t)."""
    return B2.quad_triangle(3 * k + 1)


def face_points(face: int, st) -> np.ndarray:
    """Reference-tet points of face `face` at face parameters st (n, 2)."""
    p0, p1, p2 = (TET_VERTICES[v] for v in TET_FACES[face])
    st = np.atleast_2d(np.asarray(st, dtype=float))
    return p0[None] + st[:, :1] * (p1 - p0)[None] + st[:, 1:2] * (p2 - p0)[None]


# ---------------------------------------------------------------------------
# tetrahedral Dubiner modes


def dubiner3_index(k: int):
    """(i, j, l) ordered by total degree d, then l, then j."""
    return [(d - j - l, j, l) for d in range(k + 1) for l in range(d + 1) for j in range(d - l + 1)]


def _scaled_jacobi(nmax, alpha, s, t, gs, gt):
    """Q_n = t^n P_n^{(alpha,0)}(s/t) and gradients for n = 0..nmax, with s, t
    affine in x (gradients gs, gt constant 3-vectors).  Homogeneous three-term
    recurrence — no division by t."""
    npts = s.size
    Q = np.zeros((nmax + 1, npts))
    G = np.zeros((nmax + 1, npts, 3))
    Q[0] = 1.0
    if nmax >= 1:
        Q[1] = 0.5 * ((alpha + 2.0) * s + alpha * t)
        G[1] = 0.5 * ((alpha + 2.0) * gs + alpha * gt)[None, :]
    a = alpha
    for n in range(1, nmax):
        den = 2.0 * (n + 1) * (n + a + 1) * (2 * n + a)
        An = (2 * n + a + 1) * (2 * n + a + 2) * (2 * n + a) / den
        Bn = (2 * n + a + 1) * a * a / den
        Cn = 2.0 * n * (n + a) * (2 * n + a + 2) / den
        lin = An * s + Bn * t
        glin = An * gs + Bn * gt
        Q[n + 1] = lin * Q[n] - Cn * t * t * Q[n - 1]
        G[n + 1] = (glin[None, :] * Q[n][:, None] + lin[:, None] * G[n]
                    - Cn * (2.0 * t[:, None] * gt[None, :] * Q[n - 1][:, None] + (t * t)[:, None] * G[n - 1]))
    return Q, G


@lru_cache(maxsize=None)
def _dub3_norms(k: int):
    q = quad_tet(2 * k + 2)
    v = _dubiner3_raw(k, q.points)[0]
    return 1.0 / np.sqrt(6.0 * (v * v * q.weights[:, None]).sum(0))


def _dubiner3_raw(k, pts, with_grads=False):
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    ex, ey, ez = np.eye(3)
    s1, t1 = 2 * x + y + z - 1, 1 - y - z
    s2, t2 = 2 * y + z - 1, 1 - z
    s3, t3 = 2 * z - 1, np.ones_like(z)
    Qa, Ga = _scaled_jacobi(k, 0.0, s1, t1, np.array([2.0, 1.0, 1.0]), np.array([0.0, -1.0, -1.0]))
    out = np.empty((pts.shape[0], nbs3_of(k)))
    grads = np.empty((pts.shape[0], nbs3_of(k), 3)) if with_grads else None
    cache_b, cache_c = {}, {}
    for m, (i, j, l) in enumerate(dubiner3_index(k)):
        if i not in cache_b:
            cache_b[i] = _scaled_jacobi(k - i, 2.0 * i + 1.0, s2, t2, np.array([0.0, 2.0, 1.0]),
                                        np.array([0.0, 0.0, -1.0]))
        if (i + j) not in cache_c:
            cache_c[i + j] = _scaled_jacobi(k - i - j, 2.0 * (i + j) + 2.0, s3, t3, np.array([0.0, 0.0, 2.0]),
                                            np.zeros(3))
        Qb, Gb = cache_b[i]
        Qc, Gc = cache_c[i + j]
        fa, fb, fc = Qa[i], Qb[j], Qc[l]
        out[:, m] = fa * fb * fc
        if with_grads:
            grads[:, m, :] = (Ga[i] * (fb * fc)[:, None] + Gb[j] * (fa * fc)[:, None] + Gc[l] * (fa * fb)[:, None])
    return out, grads


def dubiner3_values(k: int, pts, with_grads: bool = False):
    """Orthogonal tet modes D_m (Gram I/6, D_0 = 1): values (n, nbs3) and,
    with `with_grads`, gradients (n, nbs3, 3)."""
    v, g = _dubiner3_raw(k, pts, with_grads)
    c = _dub3_norms(k)
    if with_grads:
        return v * c[None, :], g * c[None, :, None]
    return v * c[None, :]


# ---------------------------------------------------------------------------
# BDM_k on the tetrahedron


@dataclass
class BDM3Basis:
    k: int
    coef: np.ndarray          # (nb, nb) raw modal (e_c D_m, index c*nbs+m) -> member
    vandermonde: np.ndarray
    cond: float
    n_face: int
    n_interior: int

    @property
    def nb(self) -> int:
        return self.coef.shape[0]

    def raw_values(self, pts):
        d = dubiner3_values(self.k, pts)
        nbs = d.shape[1]
        out = np.zeros((d.shape[0], 3 * nbs, 3))
        for c in range(3):
            out[:, c * nbs:(c + 1) * nbs, c] = d
        return out

    def values(self, pts):
        return np.einsum("pqc,qj->pjc", self.raw_values(pts), self.coef)

    def raw_divergence(self, pts):
        _, g = dubiner3_values(self.k, pts, with_grads=True)
        return np.concatenate([g[:, :, 0], g[:, :, 1], g[:, :, 2]], axis=1)

    def divergence(self, pts):
        return self.raw_divergence(pts) @ self.coef


def _interior_test_fields(k, pts):
    """Values (npts, n_int, 3) of a basis of N_{k-1} (first kind) at pts."""
    if k < 2:
        return np.zeros((pts.shape[0], 0, 3))
    fields = []
    d = dubiner3_values(k - 2, pts)                       # [P_{k-2}]^3
    for c in range(3):
        for m in range(d.shape[1]):
            f = np.zeros((pts.shape[0], 3))
            f[:, c] = d[:, m]
            fields.append(f)
    # x cross (e_c x^alpha), |alpha| = k-2, greedy independent selection
    q = quad_tet(2 * k + 2)
    def gram_rank(fs):
        V = np.stack([f for f in fs], axis=1)              # on q.points
        Gm = np.einsum("p,pic,pjc->ij", q.weights, V, V)
        ev = np.linalg.eigvalsh(Gm)
        return int((ev > 1e-12 * ev.max()).sum())
    base_q = []
    d_q = dubiner3_values(k - 2, q.points)
    for c in range(3):
        for m in range(d_q.shape[1]):
            f = np.zeros((q.points.shape[0], 3))
            f[:, c] = d_q[:, m]
            base_q.append(f)
    chosen = []
    X = q.points
    rank = gram_rank(base_q)
    exps = [(a, b, k - 2 - a - b) for a in range(k - 1) for b in range(k - 1 - a)]
    for c in range(3):
        for (ax, ay, az) in exps:
            mono = X[:, 0] ** ax * X[:, 1] ** ay * X[:, 2] ** az
            p = np.zeros_like(X)
            p[:, c] = mono
            cand = np.cross(X, p)
            r = gram_rank(base_q + [cq for _, cq in chosen] + [cand])
            if r > rank:
                rank = r
                chosen.append(((c, ax, ay, az), cand))
    for (c, ax, ay, az), _ in chosen:
        mono = pts[:, 0] ** ax * pts[:, 1] ** ay * pts[:, 2] ** az
        p = np.zeros_like(pts)
        p[:, c] = mono
        fields.append(np.cross(pts, p))
    return np.stack(fields, axis=1)


def bdm3_functionals_applied(k, face_vals, vol_vals, qf=None, qv=None):
    """Apply the BDM3_k functionals.  face_vals: (4, nqf, nfields, 3) at
    face_points(f, qf.points); vol_vals: (nqv, nfields, 3) at qv.points."""
    qf = qf or B2.quad_triangle(2 * k + 2)
    qv = qv or quad_tet(2 * k + 2)
    D2 = B2.dubiner_values(k, qf.points)                   # (nqf, nbs2)
    rows = []
    for f in range(4):
        vn = np.einsum("qnc,c->qn", face_vals[f], TET_FACE_NORMALS[f])
        rows.append((D2 * qf.weights[:, None]).T @ vn)     # (nbs2, nfields)
    T = _interior_test_fields(k, qv.points)                # (nqv, nint, 3)
    if T.shape[1]:
        rows.append(np.einsum("p,pic,pnc->in", qv.weights, T, vol_vals))
    return np.vstack(rows)


@lru_cache(maxsize=None)
def build_bdm3_basis(k: int) -> BDM3Basis:
    if not 1 <= k <= 6:
        raise ValueError("3D BDM degree must be in [1, 6]")
    nb = nb3_of(k)
    qf = B2.quad_triangle(2 * k + 2)
    qv = quad_tet(2 * k + 2)
    shell = BDM3Basis(k=k, coef=np.eye(nb), vandermonde=np.eye(nb), cond=1.0, n_face=0, n_interior=0)
    fv = np.stack([shell.raw_values(face_points(f, qf.points)) for f in range(4)])
    V = bdm3_functionals_applied(k, fv, shell.raw_values(qv.points), qf=qf, qv=qv)
    if V.shape != (nb, nb):
        raise RuntimeError(f"BDM3 functional count {V.shape[0]} != dimension {nb}")
    cond = float(np.linalg.cond(V))
    if not np.isfinite(cond) or cond > 1e12:
        raise RuntimeError("singular BDM3 dual Vandermonde")
    n_face = 4 * (k + 1) * (k + 2) // 2
    return BDM3Basis(k=k, coef=np.linalg.solve(V, np.eye(nb)), vandermonde=V, cond=cond,
                     n_face=n_face, n_interior=nb - n_face)


@lru_cache(maxsize=None)
def bdm3_divergence_modal(k: int) -> np.ndarray:
    """(nbs3(k-1), nb): div of each member in the tet Dubiner P_{k-1} modes."""
    q = quad_tet(2 * k)
    D = dubiner3_values(k - 1, q.points)
    return 6.0 * (D * q.weights[:, None]).T @ build_bdm3_basis(k).divergence(q.points)


def midx3(i: int, j: int, l: int) -> int:
    """Position of mode (i, j, l) in dubiner3_index order."""
    d = i + j + l
    return d * (d + 1) * (d + 2) // 6 + l * (d + 1) - l * (l - 1) // 2 + j


@lru_cache(maxsize=None)
def collapsed_tables3(k: int) -> dict:
    """Sum-factorisation tables of the tet Dubiner modes on volume_rule3(k)
    (collapsed coordinates x = a(1-b)(1-c), y = b(1-c), z = c):
        D_ijl(a, b, c) = A_i(a) B_ij(b) C_ijl(c),
        A_i = P_i(2a-1),  B_ij = (1-b)^i P_j^(2i+1,0)(2b-1),
        C_ijl = c_ijl (1-c)^(i+j) P_l^(2i+2j+2,0)(2c-1),
    with derivatives Ad, Bd, Cd.  B/Bd columns are indexed by the pair
    (i, j) in 2D Dubiner order ((i+j)(i+j+1)/2 + j), C/Cd columns by the mode.
    Returns also the 1D points a, b, c, and per-point t1 = (1-b)(1-c),
    t2 = 1-c are implied by them."""
    n = (3 * k + 1) // 2
    q = volume_rule3(k)
    assert q.n1 == n
    xa, _ = roots_legendre(n)
    a = 0.5 * (xa + 1.0)
    b, _ = _gj01(n, 1.0)
    c, _ = _gj01(n, 2.0)
    norms = _dub3_norms(k)
    A = np.zeros((n, k + 1))
    Ad = np.zeros((n, k + 1))
    lv, ld = B2._legendre_pd(k, a)
    sc = np.sqrt(2.0 * np.arange(k + 1) + 1.0)
    A[:] = lv / sc
    Ad[:] = ld / sc
    npair = (k + 1) * (k + 2) // 2
    Bt = np.zeros((n, npair))
    Bd = np.zeros((n, npair))
    for i in range(k + 1):
        P, dP = B2._jacobi_a0(k - i, 2.0 * i + 1.0, 2.0 * b - 1.0)
        for j in range(k - i + 1):
            pi = (i + j) * (i + j + 1) // 2 + j
            Bt[:, pi] = (1 - b) ** i * P[j]
            Bd[:, pi] = (-i * (1 - b) ** (i - 1) if i else 0.0) * P[j] + (1 - b) ** i * 2.0 * dP[j]
    nbs = nbs3_of(k)
    Ct = np.zeros((n, nbs))
    Cd = np.zeros((n, nbs))
    for (i, j, l) in dubiner3_index(k):
        m = midx3(i, j, l)
        P, dP = B2._jacobi_a0(l, 2.0 * (i + j) + 2.0, 2.0 * c - 1.0)
        e = i + j
        Ct[:, m] = norms[m] * (1 - c) ** e * P[l]
        Cd[:, m] = norms[m] * ((-e * (1 - c) ** (e - 1) if e else 0.0) * P[l] + (1 - c) ** e * 2.0 * dP[l])
    return {"n": n, "A": A, "Ad": Ad, "B": Bt, "Bd": Bd, "C": Ct, "Cd": Cd, "a": a, "b": b, "c": c}
