"""Curved-element data for the device path (host side, fp64).

On the elements that carry a degree-g isoparametric map (``mesh.curve_boundary``,
restating MESH:555-615) the convection form needs no geometry at all — with
Piola velocities and pulled-back V_h test functions both the volume term and
the facet flux are exactly the reference-element expressions (SURVEY A.3
holds pointwise), so the apply kernels are unchanged.  What changes is
(PAPER.md:473-475):

* the V_h mass is block diagonal with a full block per curved element,
  M_T[m, n] = int D_m D_n detJ dx_hat (the same block for both components);
  the explicit update needs M_T^{-1};
* the transfer I: U_h -> V_h is the element-wise L2 projection
  I_T[(c, m), j] = sum_n (M_T^{-1})[m, n] int (J phi_hat_j)_c D_n dx_hat
  (the detJ of the Piola map cancels against the measure); I^T = I_T^T;
* max|u| needs the point-dependent Piola factor J(x_hat)/detJ(x_hat).

``curved_tables`` computes these small dense per-element matrices once on
the host (a handful of elements along a curved boundary); the device gets
them through ``hdgc_set_curved``.
"""

from __future__ import annotations

import numpy as np

from . import basis as B

__all__ = ["curved_tables"]


def curved_tables(mesh, k: int) -> dict:
    """Per curved element (ascending id): ``elems`` (n,) int32, ``minv``
    (n, nbs, nbs) = M_T^{-1}, ``itrans`` (n, nb, nb) = I_T (V_h rows c*nbs+m,
    BDM columns), ``piola`` (n, nqv, 4) = J/detJ at the volume_rule(k) points
    (row-major 00, 01, 10, 11)."""
    ce = mesh.curved_elements() if getattr(mesh, "curved_maps", None) else np.zeros(0, np.int64)
    nbs = B.nbs_of(k)
    nb = 2 * nbs
    qv = B.volume_rule(k)
    n = ce.size
    out = dict(elems=ce.astype(np.int32), minv=np.zeros((n, nbs, nbs)), itrans=np.zeros((n, nb, nb)),
               piola=np.zeros((n, qv.points.shape[0], 4)))
    if n == 0:
        return out
    g = int(mesh.geometry_order)
    bdm = B.build_bdm_basis(k)
    qm = B.quad_triangle(2 * k + 2 * (g - 1))
    Dm = B.dubiner_values(k, qm.points)
    _, _, det = mesh.geometry_batch(ce, qm.points)
    M = np.einsum("p,np,pm,pl->nml", qm.weights, det, Dm, Dm)
    Minv = np.linalg.inv(M)
    Minv = 0.5 * (Minv + np.transpose(Minv, (0, 2, 1)))
    qi = B.quad_triangle(2 * k + g + 1)
    Di = B.dubiner_values(k, qi.points)
    phi = bdm.values(qi.points)                                  # (p, nb, 2)
    _, J, _ = mesh.geometry_batch(ce, qi.points)
    Jphi = np.einsum("npcd,pjd->npjc", J, phi)                   # (n, p, nb, 2)
    rhs = np.einsum("p,npjc,pl->nclj", qi.weights, Jphi, Di)      # (n, 2, nbs, nb)
    out["minv"] = np.ascontiguousarray(Minv)
    out["itrans"] = np.ascontiguousarray(np.einsum("nml,nclj->ncmj", Minv, rhs).reshape(n, nb, nb))
    _, Jv, dv = mesh.geometry_batch(ce, qv.points)
    out["piola"] = np.ascontiguousarray((Jv / dv[..., None, None]).reshape(n, -1, 4))
    return out
