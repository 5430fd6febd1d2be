"""ORACLE — test infrastructure only.  CPU restatement of the global H(div)
space of the reference's ``fespace`` module for the convection path's
callers:

* numbering: facet dofs first, facet-major then mode
  (dof = f (k+1) + m), then element-interior dofs (element-major);
* orientation (mesh2d.py:201): the global facet dof is the flux
  moment int_F u.n_f L_m ds along the OWNER's outward normal and edge
  parametrisation; it is evaluated here from the physical field by
  quadrature (``flux_moments``), independently of the device's factor table;
* gather  u_loc[T, j] = s[T, j] g[dof[T, j]],
  scatter r_glob = sum over occurrences (np.add.at) — the global I^T assembly.

Only tests/ may import this module.
"""
from __future__ import annotations

import numpy as np


def numbering(mesh, k):
    """(element_dofs (NT, nb), ndof) by the SPEC rule, built facet by facet."""
    ne = k + 1
    nb = (k + 1) * (k + 2)
    NT, NF = mesh.n_elements, mesh.n_facets
    dofs = -np.ones((NT, nb), dtype=np.int64)
    for f in range(NF):
        for side in (0, 1):
            T = mesh.facet_elems[f, side]
            if T < 0:
                continue
            e = mesh.facet_local[f, side]
            for m in range(ne):
                dofs[T, e * ne + m] = f * ne + m
    nint = nb - 3 * ne
    for T in range(NT):
        for i in range(nint):
            dofs[T, 3 * ne + i] = NF * ne + T * nint + i
    return dofs, NF * ne + NT * nint


def flux_moments(mesh, k, velocity, nq=None):
    """g[f, m] = int_F u.n_f L_m(t) ds with the owner's normal and
    parametrisation (t from facet_vertices[f, 0] to [1]), orthonormal Legendre
    on [0, 1], Gauss-Legendre with nq points."""
    from numpy.polynomial.legendre import leggauss, legval
    nq = nq or (k + 6)
    x, wq = leggauss(nq)
    t, wq = 0.5 * (x + 1.0), 0.5 * wq
    L = np.stack([np.sqrt(2 * m + 1) * legval(2 * t - 1, np.eye(k + 1)[m]) for m in range(k + 1)], axis=1)
    a = mesh.vertices[mesh.facet_vertices[:, 0]]
    b = mesh.vertices[mesh.facet_vertices[:, 1]]
    d = b - a
    length = np.linalg.norm(d, axis=1)
    # owner's outward normal: rotate the edge direction, pointing away from the owner's centroid
    n = np.stack([d[:, 1], -d[:, 0]], axis=1) / length[:, None]
    own = mesh.facet_elems[:, 0]
    cen = mesh.vertices[mesh.triangles[own]].mean(axis=1)
    flip = np.sum(n * (0.5 * (a + b) - cen), axis=1) < 0
    n[flip] *= -1
    X = a[:, None, :] + t[None, :, None] * d[:, None, :]
    U = velocity(X[..., 0], X[..., 1])                     # (NF, nq, 2)
    un = np.einsum("fqc,fc->fq", U, n)
    return np.einsum("fq,q,qm->fm", un, wq, L) * length[:, None]


def gather(dofs, factors, g):
    return factors * g[dofs]


def scatter(dofs, factors, r_loc, ndof):
    out = np.zeros(ndof)
    np.add.at(out, dofs.ravel(), (factors * r_loc).ravel())
    return out
