"""Global H(div) dof map — the W_h gather/scatter either side of the convection
path (reference module ``fespace``).

SPEC.md:184-194 fixes the numbering: facet dofs first, ordered by facet index
then Legendre mode, then element-interior dofs; the edge dof's orientation
follows the facet's owning element (``facet_elems[f, 0]``, mesh2d.py:201).

The device path keeps W_h fields element-local: the local
edge dof of element T on its edge e is the *parameter-measure* moment
c[T,e,m] = int_0^1 u_hat.n_hat_e L_m(t) dt (polybasis.py:329-334).  The global
facet dof is the physical flux moment along the owner's normal and
parametrisation,

    g[f, m] = int_F u.n_f L_m ds = c[T_own, e_own, m] |e_own|          (A.3: u.n ds = u_hat.n_hat |e_hat| dt)

so the local coefficient is a scaled copy of the global one:

    c[T, e, m] = s[T, e, m] g[f, m],
    s = 1/|e_hat_e|                                  on the owner side,
    s = -(+-1)^m / |e_hat_e'|  (-(-1)^m if the neighbour traverses F backwards)
                                                     on the other side,

which reproduces SURVEY A.2's conformity relation c|e| = (-1)^{m+1} c'|e'|.
Interior dofs are element-owned (s = 1).

``element_dofs`` (NT, nb) int64 and ``factors`` (NT, nb) float64 are uploaded
to the context (hdgc_set_dofmap); the device gather is
u_loc[T, j] = factors[T, j] u_glob[element_dofs[T, j]] and the scatter (the
global I^T assembly) r_glob[d] = sum_{(T, j) -> d} factors[T, j] r_loc[T, j],
computed per global dof from an inverse map in a fixed order (no atomics).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import basis as B

__all__ = ["HdivDofMap", "build_hdiv_dofmap", "hdiv_ndof", "global_from_local"]


@dataclass(frozen=True)
class HdivDofMap:
    k: int
    ndof: int
    n_facet_dofs: int
    element_dofs: np.ndarray     # (NT, nb) int64
    factors: np.ndarray          # (NT, nb) float64


def hdiv_ndof(n_facets: int, n_elements: int, k: int) -> int:
    """#facets (k+1) + #elements (k+1)(k-1)."""
    return n_facets * (k + 1) + n_elements * (k + 1) * (k - 1)


def build_hdiv_dofmap(mesh, k: int) -> HdivDofMap:
    if not hasattr(mesh, "facet_flip"):
        raise NotImplementedError("global H(div) numbering is defined for triangle meshes (2D)")
    NT, NF = mesh.n_elements, mesh.n_facets
    ne = k + 1
    nb = B.nb_of(k)
    nint = nb - 3 * ne
    dofs = np.empty((NT, nb), dtype=np.int64)
    fac = np.ones((NT, nb), dtype=np.float64)
    lens = B.REF_EDGE_LENGTHS
    m = np.arange(ne)
    alt = np.where(m % 2 == 0, 1.0, -1.0)           # (-1)^m
    for side in (0, 1):
        sel = np.nonzero(mesh.facet_elems[:, side] >= 0)[0]
        T = mesh.facet_elems[sel, side]
        e = mesh.facet_local[sel, side]
        cols = e[:, None] * ne + m[None, :]
        dofs[T[:, None], cols] = sel[:, None] * ne + m[None, :]
        if side == 0:
            fac[T[:, None], cols] = 1.0 / lens[e][:, None]
        else:
            rev = mesh.facet_flip[sel, 1]
            s = -np.where(rev[:, None], alt[None, :], 1.0)
            fac[T[:, None], cols] = s / lens[e][:, None]
    base = NF * ne
    dofs[:, 3 * ne:] = base + np.arange(NT)[:, None] * nint + np.arange(nint)[None, :]
    return HdivDofMap(k, hdiv_ndof(NF, NT, k), base, dofs, fac)


def global_from_local(dm: HdivDofMap, u_loc: np.ndarray) -> np.ndarray:
    """Global coefficients of a conforming element-local field: each dof read
    from its first occurrence in (T, j) order, g = u_loc / factor (any
    occurrence gives the same value for a conforming field)."""
    g = np.zeros(dm.ndof)
    flat_d = dm.element_dofs.ravel()
    first = np.full(dm.ndof, -1, dtype=np.int64)
    order = np.arange(flat_d.size)[::-1]
    first[flat_d[order]] = order                      # smallest (T, j) index wins
    g[:] = u_loc.ravel()[first] / dm.factors.ravel()[first]
    return g
