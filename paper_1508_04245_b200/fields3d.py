"""Seeded divergence-free velocity for the 3D convection path (BASELINE cfg5).

u = curl A with each component of the vector potential
    A_i(x) = sum_{l,m,n=1..M} b^i_lmn sin(l pi x) sin(m pi y) sin(n pi z),
    b^i_lmn ~ N(0, 1/(l^2+m^2+n^2))   (drawn i, l, m, n row-major from
                                        np.random.default_rng(seed)).
The BDM_k field is u_h = curl(Pi_{k+1} A) with Pi_{k+1} the element-local
Lagrange interpolation of degree k+1 at the equispaced lattice (SURVEY A.5,
3D suggestion): Pi A is continuous (shared faces carry the same nodes), so
its curl is H(div)-conforming and exactly divergence-free; it is a
polynomial of degree k, so the BDM_k interpolant reproduces it and the dofs
are computed with exact quadrature.  u.n = 0 on the cube boundary.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import basis as B2
from . import basis3d as B3

__all__ = ["VectorPotential", "interpolate_curl3", "inflow_values3", "transfer_I3_host", "max_speed3_host",
           "lattice"]


@dataclass(frozen=True)
class VectorPotential:
    """Seeded sine-mode vector potential plus an optional uniform wind w,
    realised as A_wind = (w x x)/2 (curl A_wind = w), so the wind is part of
    the interpolated potential and stays exactly divergence-free."""

    modes: int
    seed: int
    wind: tuple = (0.0, 0.0, 0.0)

    @property
    def coeffs(self) -> np.ndarray:
        M = self.modes
        rng = np.random.default_rng(self.seed)
        m = np.arange(1, M + 1)
        var = m[:, None, None] ** 2 + m[None, :, None] ** 2 + m[None, None, :] ** 2
        return rng.normal(0.0, 1.0, size=(3, M, M, M)) / np.sqrt(var)[None]

    def _trig(self, x):
        k = np.pi * np.arange(1, self.modes + 1)
        x = np.asarray(x, dtype=float)[..., None]
        return np.sin(k * x), np.cos(k * x) * k

    def potential(self, X):
        sx, _ = self._trig(X[..., 0])
        sy, _ = self._trig(X[..., 1])
        sz, _ = self._trig(X[..., 2])
        A = np.einsum("ilmn,...l,...m,...n->...i", self.coeffs, sx, sy, sz)
        return A + 0.5 * np.cross(np.asarray(self.wind, dtype=float), X)

    def velocity(self, X):
        """curl A, shape (..., 3)."""
        sx, cx = self._trig(X[..., 0])
        sy, cy = self._trig(X[..., 1])
        sz, cz = self._trig(X[..., 2])
        b = self.coeffs
        dA = lambda i, gx, gy, gz: np.einsum("lmn,...l,...m,...n->...", b[i], gx, gy, gz)
        ux = dA(2, sx, cy, sz) - dA(1, sx, sy, cz)
        uy = dA(0, sx, sy, cz) - dA(2, cx, sy, sz)
        uz = dA(1, cx, sy, sz) - dA(0, sx, cy, sz)
        return np.stack([ux, uy, uz], axis=-1) + np.asarray(self.wind, dtype=float)


def lattice(p: int) -> np.ndarray:
    """Equispaced degree-p lattice on the reference tet, (n, 3)."""
    return np.array([[i / p, j / p, l / p] for l in range(p + 1) for j in range(p + 1 - l)
                     for i in range(p + 1 - l - j)])


def interpolate_curl3(mesh, k: int, vp: VectorPotential, chunk: int = 16384) -> np.ndarray:
    """Element-local BDM3_k coefficients (NT, nb) of curl(Pi_{k+1} A)."""
    p = k + 1
    nodes = lattice(p)
    V = B3.dubiner3_values(p, nodes)                       # (nn, nbs3(p))
    Vinv = np.linalg.inv(V)
    qf = B2.quad_triangle(2 * k + 2)
    qv = B3.quad_tet(2 * k + 2)
    fpts = [B3.face_points(f, qf.points) for f in range(4)]
    allpts = np.vstack(fpts + [qv.points])
    _, G = B3.dubiner3_values(p, allpts, with_grads=True)  # (P, nbs3(p), 3)
    NT = mesh.n_elements
    nb = B3.nb3_of(k)
    out = np.empty((NT, nb))
    nf = qf.points.shape[0]
    for s in range(0, NT, chunk):
        sl = slice(s, min(NT, s + chunk))
        J, det, Ji = mesh.affine_jac[sl], mesh.affine_det[sl], mesh.affine_inv[sl]
        X = mesh.affine_origin[sl][:, None, :] + np.einsum("ncd,pd->npc", J, nodes)
        A = vp.potential(X)                                 # (n, nn, 3)
        a = np.einsum("mj,njc->nmc", Vinv, A)               # modal coefficients per component
        gref = np.einsum("nmc,pmd->npcd", a, G)             # d(A_c)/d(xhat_d)
        gphys = np.einsum("npce,ned->npcd", gref, Ji)       # d(A_c)/dx_d = sum_e dxhat_e/dx_d
        curl = np.stack([gphys[..., 2, 1] - gphys[..., 1, 2],
                         gphys[..., 0, 2] - gphys[..., 2, 0],
                         gphys[..., 1, 0] - gphys[..., 0, 1]], axis=-1)
        uhat = det[:, None, None] * np.einsum("ncd,npd->npc", Ji, curl)     # detJ J^-1 u
        fv = np.stack([uhat[:, f * nf:(f + 1) * nf] for f in range(4)])     # (4, n, nf, 3)
        vv = uhat[:, 4 * nf:]
        rows = B3.bdm3_functionals_applied(k, fv.transpose(0, 2, 1, 3), vv.transpose(1, 0, 2), qf=qf, qv=qv)
        out[sl] = rows.T
    return out


def inflow_values3(mesh, k: int, vp: VectorPotential) -> np.ndarray:
    """Exact velocity at the face rule points of boundary faces, (NBF, nf, 3),
    rows in boundary-facet order, points in the owner's face parametrisation."""
    qf = B3.face_rule(k)
    bf = mesh.boundary_facets
    T = mesh.facet_elems[bf, 0]
    f = mesh.facet_local[bf, 0]
    out = np.empty((bf.size, qf.points.shape[0], 3))
    for face in range(4):
        sel = f == face
        xr = B3.face_points(face, qf.points)
        X = mesh.affine_origin[T[sel]][:, None, :] + np.einsum("ncd,pd->npc", mesh.affine_jac[T[sel]], xr)
        out[sel] = vp.velocity(X)
    return out


def transfer_I3_host(mesh, k: int, u_loc: np.ndarray) -> np.ndarray:
    """w = I u: V_h coefficients w[c*nbs+m] = sum_d (J/detJ)[c,d] (coef u)[d*nbs+m]."""
    bdm = B3.build_bdm3_basis(k)
    nbs = B3.nbs3_of(k)
    uh = (u_loc @ bdm.coef.T).reshape(-1, 3, nbs)
    P = mesh.affine_jac / mesh.affine_det[:, None, None]
    return np.einsum("ncd,ndm->ncm", P, uh).reshape(-1, 3 * nbs)


def max_speed3_host(mesh, k: int, u_loc: np.ndarray, chunk: int = 16384) -> float:
    q = B3.volume_rule3(k)
    phi = B3.build_bdm3_basis(k).values(q.points)
    best = 0.0
    for s in range(0, mesh.n_elements, chunk):
        sl = slice(s, min(mesh.n_elements, s + chunk))
        uh = np.einsum("pjd,nj->npd", phi, u_loc[sl])
        u = np.einsum("ncd,npd->npc", mesh.affine_jac[sl] / mesh.affine_det[sl, None, None], uh)
        best = max(best, float(np.sqrt((u ** 2).sum(-1)).max()))
    return best
