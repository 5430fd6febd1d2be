"""Seeded synthetic workloads for the convection path (host side, fp64).

BASELINE.json configs 1-4 transport by the curl of a seeded stream function

    psi(x, y) = sum_{m,n=1..M} a_mn sin(m pi x) sin(n pi y) + psi_wind,
    a_mn ~ N(0, 1/(m^2+n^2)),     u = curl psi = (d_y psi, -d_x psi)

(the paper's convention).  ``psi_wind = wx*y - wy*x`` gives the
uniform background wind (wx, wy) of cfg3.  Coefficients are drawn
row-major (m outer, n inner) from ``np.random.default_rng(seed)``.

The BDM_k interpolant is built element-locally with the exact-moment recipe
of SURVEY Appendix A.5, so the discrete field is divergence-free to rounding
(a plain quadrature interpolant is only div-free to ~1e-8):

* edge dofs by parts along the CCW edge, using u.n ds = d psi:
  ``c_em = (psi(b) L_m(1) - psi(a) L_m(0) - int psi L_m' dt) / |e_ref|``
* gradient-moment dofs from the discrete divergence theorem
  ``sum_e |e_ref| int (sum_m c_em L_m) q_j dt``;
* curl-bubble dofs by quadrature of the Piola pull-back (PB:342-352).

Adjacent elements then agree on the normal trace, so the
element-local coefficient array is an H(div)-conforming field.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import basis as B

__all__ = ["StreamFunction", "interpolate_curl", "inflow_values", "transfer_I_host",
           "max_speed_host", "cfl_dt"]


@dataclass(frozen=True)
class StreamFunction:
    """Seeded stream function with M x M sine modes plus a uniform wind."""

    modes: int
    seed: int
    wind: tuple = (0.0, 0.0)

    @property
    def coeffs(self) -> np.ndarray:
        M = self.modes
        rng = np.random.default_rng(self.seed)
        m = np.arange(1, M + 1)
        std = 1.0 / np.sqrt(m[:, None] ** 2 + m[None, :] ** 2)
        return rng.normal(0.0, 1.0, size=(M, M)) * std

    def _trig(self, x, y):
        M = self.modes
        k = np.pi * np.arange(1, M + 1)
        x = np.asarray(x, dtype=float)[..., None]
        y = np.asarray(y, dtype=float)[..., None]
        return np.sin(k * x), np.cos(k * x) * k, np.sin(k * y), np.cos(k * y) * k

    def psi(self, x, y):
        sx, _, sy, _ = self._trig(x, y)
        a = self.coeffs
        wx, wy = self.wind
        return np.einsum("...m,mn,...n->...", sx, a, sy) + wx * np.asarray(y) - wy * np.asarray(x)

    def velocity(self, x, y):
        """u = (d_y psi, -d_x psi), shape (..., 2)."""
        sx, cx, sy, cy = self._trig(x, y)
        a = self.coeffs
        wx, wy = self.wind
        ux = np.einsum("...m,mn,...n->...", sx, a, cy) + wx
        uy = -np.einsum("...m,mn,...n->...", cx, a, sy) + wy
        return np.stack([ux, uy], axis=-1)


def _edge_geometry(mesh):
    """Physical start/end vertices of each element's local edges: (NT, 3, 2)."""
    tri = mesh.triangles
    V = mesh.vertices
    a = np.stack([V[tri[:, s]] for s, _ in B.REF_EDGES], axis=1)
    b = np.stack([V[tri[:, e]] for _, e in B.REF_EDGES], axis=1)
    return a, b


def interpolate_curl(mesh, k: int, sf: StreamFunction, chunk: int = 65536) -> np.ndarray:
    """Element-local BDM_k coefficients (NT, nb) of curl(psi), exactly
    divergence-free.  Layout: BDMBasis member order (PB:265-268)."""
    bdm = B.build_bdm_basis(k)
    nb = bdm.nb
    NT = mesh.n_elements
    out = np.empty((NT, nb))
    qe = B.quad_interval(2 * k + 2)
    qv = B.quad_triangle(2 * k + 2)
    L0 = B.legendre_values(k, np.array([0.0]))[0]
    L1 = B.legendre_values(k, np.array([1.0]))[0]
    dL = B.legendre_derivs(k, qe.points)                      # (nq, k+1)
    Lq = B.legendre_values(k, qe.points)                      # (nq, k+1)
    elen = B.REF_EDGE_LENGTHS
    n_int = (k + 1) * (k - 1)
    if k >= 2:
        # q_j on the three reference edges, for the gradient moments
        nlow = B.nbs_of(k - 1)
        qedge = np.stack([B.dubiner_values(k - 1, B.ref_edge_points(e, qe.points))[:, 1:nlow]
                          for e in range(3)])                 # (3, nq, nlow-1)
        # curl-bubble test functions at the volume points
        b, gb = B._bubble_and_grad(qv.points)
        q2, gq2 = B.dubiner_values(k - 2, qv.points, with_grads=True)
        gbq = q2[:, :, None] * gb[:, None, :] + b[:, None, None] * gq2
        curl = np.stack([gbq[:, :, 1], -gbq[:, :, 0]], axis=-1) * qv.weights[:, None, None]
    A_all, B_all = _edge_geometry(mesh)
    t = qe.points

    def rows(A, Bv, X, xq, J, det):
        """coefficients of n elements from the physical edge points X (n,3,nq,2)
        and the physical volume points xq (n,p,2) with their J, detJ"""
        n = A.shape[0]
        res = np.empty((n, nb))
        psi_a = sf.psi(A[..., 0], A[..., 1])                   # (n, 3)
        psi_b = sf.psi(Bv[..., 0], Bv[..., 1])
        psi_q = sf.psi(X[..., 0], X[..., 1])                   # (n, 3, nq)
        integ = np.einsum("neq,q,qm->nem", psi_q, qe.weights, dL)
        c = (psi_b[:, :, None] * L1[None, None, :] - psi_a[:, :, None] * L0[None, None, :] - integ)
        c /= elen[None, :, None]
        res[:, :3 * (k + 1)] = c.reshape(n, 3 * (k + 1))
        if n_int:
            # gradient moments: sum_e |e| int (sum_m c_em L_m) q_j dt
            tr = np.einsum("nem,qm->neq", c, Lq)              # normal trace at points
            g = np.einsum("e,neq,q,eqj->nj", elen, tr, qe.weights, qedge)
            # curl-bubble moments of the pulled-back exact field u_hat = detJ J^-1 u
            u = sf.velocity(xq[..., 0], xq[..., 1])            # (n, p, 2)
            adj = np.stack([np.stack([J[..., 1, 1], -J[..., 0, 1]], -1),
                            np.stack([-J[..., 1, 0], J[..., 0, 0]], -1)], -2)   # detJ J^-1
            uhat = np.einsum("n...cd,n...d->n...c", adj, u)
            cb = np.einsum("pjc,npc->nj", curl, uhat)
            res[:, 3 * (k + 1):] = np.concatenate([g, cb], axis=1)
        return res

    for s in range(0, NT, chunk):
        sl = slice(s, min(NT, s + chunk))
        A, Bv = A_all[sl], B_all[sl]
        X = A[:, :, None, :] + t[None, None, :, None] * (Bv - A)[:, :, None, :]   # (n,3,nq,2)
        if n_int:
            J = mesh.affine_jac[sl]
            xq = mesh.affine_origin[sl][:, None, :] + np.einsum("ncd,pd->npc", J, qv.points)
            Jp = np.broadcast_to(J[:, None], (J.shape[0], qv.points.shape[0], 2, 2))
            det = np.broadcast_to(mesh.affine_det[sl][:, None], Jp.shape[:2])
        else:
            xq = Jp = det = None
        out[sl] = rows(A, Bv, X, xq, Jp, det)
    ce = _curved(mesh)
    if ce.size:
        # curved elements: edge points on the mapped (curved) edges, per-point J
        X = np.stack([mesh.geometry_batch(ce, B.ref_edge_points(e, t))[0] for e in range(3)], axis=1)
        xq, Jp, det = mesh.geometry_batch(ce, qv.points) if n_int else (None, None, None)
        out[ce] = rows(A_all[ce], B_all[ce], X, xq, Jp, det)
    return out


def _curved(mesh) -> np.ndarray:
    f = getattr(mesh, "curved_elements", None)
    return f() if f is not None and getattr(mesh, "curved_maps", None) else np.zeros(0, dtype=np.int64)


def inflow_values(mesh, k: int, sf: StreamFunction) -> np.ndarray:
    """Exterior (Dirichlet) values of curl(psi) at the facet rule points of
    every boundary facet, shape (NBF, nf, 2), rows in ``boundary_facets``
    order, points in the owner's traversal direction."""
    qf = B.facet_rule(k)
    bf = mesh.boundary_facets
    a = mesh.vertices[mesh.facet_vertices[bf, 0]]
    b = mesh.vertices[mesh.facet_vertices[bf, 1]]
    X = a[:, None, :] + qf.points[None, :, None] * (b - a)[:, None, :]
    if _curved(mesh).size:
        # curved boundary facets: the points on the owner's mapped edge
        own, loc = mesh.facet_elems[bf, 0], mesh.facet_local[bf, 0]
        for i in np.nonzero([mesh.is_curved(e) for e in own])[0]:
            X[i] = mesh.geometry_batch([own[i]], B.ref_edge_points(int(loc[i]), qf.points))[0][0]
    return np.ascontiguousarray(sf.velocity(X[..., 0], X[..., 1]))


def transfer_I_host(mesh, k: int, u_loc: np.ndarray) -> np.ndarray:
    """w = I u on affine elements: the V_h coefficients
    w[c*nbs+m] = sum_d (J/detJ)[c,d] (coef u)[d*nbs+m]."""
    bdm = B.build_bdm_basis(k)
    nbs = B.nbs_of(k)
    uh = (u_loc @ bdm.coef.T).reshape(-1, 2, nbs)
    P = mesh.affine_jac / mesh.affine_det[:, None, None]
    w = np.einsum("ncd,ndm->ncm", P, uh).reshape(-1, 2 * nbs)
    ce = _curved(mesh)
    if ce.size:
        # curved elements: element-wise L2 projection
        from .curved import curved_tables
        tab = curved_tables(mesh, k)
        w[ce] = np.einsum("nij,nj->ni", tab["itrans"], u_loc[ce])
    return w


def max_speed_host(mesh, k: int, u_loc: np.ndarray, chunk: int = 65536) -> float:
    """max |J u_hat / detJ| over elements x volume_rule(k) points (BASELINE cfg2)."""
    q = B.volume_rule(k)
    bdm = B.build_bdm_basis(k)
    phi = bdm.values(q.points)                                 # (p, nb, 2)
    best = 0.0
    for s in range(0, mesh.n_elements, chunk):
        sl = slice(s, min(mesh.n_elements, s + chunk))
        uh = np.einsum("pjd,nj->npd", phi, u_loc[sl])
        P = mesh.affine_jac[sl] / mesh.affine_det[sl, None, None]
        u = np.einsum("ncd,npd->npc", P, uh)
        sp = np.sqrt((u ** 2).sum(-1))
        cur = _curved(mesh)
        if cur.size:
            sp[np.isin(np.arange(sl.start, sl.stop), cur)] = 0.0     # curved rows: per-point J below
        best = max(best, float(sp.max()))
    ce = _curved(mesh)
    if ce.size:
        _, J, det = mesh.geometry_batch(ce, q.points)
        u = np.einsum("npcd,pjd,nj->npc", J, phi, u_loc[ce]) / det[..., None]
        best = max(best, float(np.sqrt((u ** 2).sum(-1)).max()))
    return best


def cfl_dt(h: float, k: int, umax: float, safety: float = 0.1) -> float:
    """Substep size dt = safety * h / (k^2 * max|u|) (BASELINE cfg2; replaces
    the SPEC's (2k+1) rule)."""
    if umax <= 0.0:
        return float("inf")
    return safety * h / (k * k * umax)
