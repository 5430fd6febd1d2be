"""ORACLE — test infrastructure only.  CPU restatement of the convection
apply, the V_h mass and the transfer on CURVED meshes; never imported by the
product package (only ``tests/`` may import it, as the checker).

What it restates
-----------------------------------
The reference attaches degree-g isoparametric maps to the elements along a
circular boundary (``mesh2d.curve_boundary``, MESH:555-615; per-point
geometry ``Mesh.geometry_map``, MESH:254-278).  On such elements

* the H(div) velocity is the contravariant Piola image, now with a
  point-dependent Jacobian: u(x) = J(x_hat) u_hat(x_hat) / detJ(x_hat)
  ("also on curved elements, where J varies");
* the V_h test functions are pull-backs z_{c,m} = e_c D_m(F_T^{-1} x), so the
  V_h mass is block diagonal, with full (nbs x nbs) blocks
  M_T[m, n] = int_T z_m z_n dx on curved elements only (PAPER.md:473-475,
  SPEC.md:283 "block-diagonal on curved elements");
* the transfer I: U_h -> V_h is no longer an embedding but the element-wise
  L2 projection; I^T is its matrix transpose.

The convection form itself is evaluated here literally,
in PHYSICAL coordinates and element by element: physical quadrature points
x = F_T(x_hat), J^{-T} gradients, physical outward normals and arc length
|dx/dt| on every (possibly curved) edge, and neighbour traces found by
pulling the physical facet points back through the neighbour's own map by
Newton iteration.  The device never does any of that — it uses the
geometry-free reference form, which the Piola identities make
exact on curved elements too — so agreement checks that claim independently.

Volume rule quad_triangle(3k+1) (the integrand is the degree 3k-1 polynomial
w_c u_hat . grad_hat D_m in reference coordinates), facet rule
quad_interval(3k+1); mass blocks with quad_triangle(2k + 2(g-1)) (detJ has
degree 2(g-1)), projections with quad_triangle(2k + g + 1).

Works on any mesh object with the ``hdgflow.mesh2d.Mesh`` attributes and a
``geometry_map(elem, ref_pts) -> (x, J, detJ)`` method (the reference's own
Mesh, or the product's TriMesh), and any basis provider with the
``hdgflow.polybasis`` API.
"""

from __future__ import annotations

import numpy as np

__all__ = ["geometry", "apply_convection", "mass_blocks", "mass_inverse_apply", "transfer_I", "transfer_IT",
           "substeps"]


def _provider(basis):
    if basis is None:
        from paper_1508_04245_b200 import basis as default   # tables only
        return default
    return basis


def geometry(mesh, elems, pts):
    """x (n,p,2), J (n,p,2,2), detJ (n,p) through the mesh's own geometry_map."""
    pts = np.atleast_2d(pts)
    xs, Js, ds = [], [], []
    for e in np.asarray(elems).reshape(-1):
        x, J, d = mesh.geometry_map(int(e), pts)
        xs.append(np.asarray(x))
        Js.append(np.asarray(J))
        ds.append(np.asarray(d))
    return np.array(xs), np.array(Js), np.array(ds)


def _curved_order(mesh):
    return int(getattr(mesh, "geometry_order", 1)) if getattr(mesh, "curved_maps", None) else 1


def _pull_back(mesh, T, x, tol=1e-15, iters=30):
    """x_hat with F_T(x_hat) = x (Newton from the affine inverse)."""
    xh = np.einsum("cd,qd->qc", mesh.affine_inv[T], x - mesh.affine_origin[T])
    for _ in range(iters):
        xm, J, _ = mesh.geometry_map(int(T), xh)
        res = np.asarray(xm) - x
        if np.abs(res).max() <= tol * max(1.0, np.abs(x).max()):
            break
        xh = xh - np.linalg.solve(np.asarray(J), res[..., None])[..., 0]
    xm, _, _ = mesh.geometry_map(int(T), xh)
    assert np.abs(np.asarray(xm) - x).max() < 1e-12, "pull-back did not converge"
    return xh


def apply_convection(mesh, k, u_loc, w, inflow=None, basis=None):
    """r = C^V(u; w) in physical coordinates, curved-aware."""
    basis = _provider(basis)
    bdm = basis.build_bdm_basis(k)
    nbs = w.shape[1] // 2
    NT = mesh.n_elements
    W = w.reshape(NT, 2, nbs)
    r = np.zeros((NT, 2, nbs))
    # ---- volume: -int_T (w (x) u) : grad z dx
    qv = basis.quad_triangle(3 * k + 1)
    D, G = basis.dubiner_values(k, qv.points, with_grads=True)       # (p,nbs), (p,nbs,2)
    phi = bdm.values(qv.points)                                      # (p, nb, 2)
    _, J, det = geometry(mesh, np.arange(NT), qv.points)
    Jinv = np.linalg.inv(J)                                          # (n,p,2,2)
    uh = np.einsum("pjd,nj->npd", phi, u_loc)
    u = np.einsum("npcd,npd->npc", J, uh) / det[..., None]
    gphys = np.einsum("npdc,pmd->npmc", Jinv, G)                     # J^{-T} grad_hat D_m
    wq = np.einsum("pm,ncm->npc", D, W)
    ugrad = np.einsum("npc,npmc->npm", u, gphys)
    r -= np.einsum("p,np,npc,npm->ncm", qv.weights, det, wq, ugrad)
    # ---- element boundaries: int_dT (u.n) w_hat . z ds, upwind w_hat
    qf = basis.quad_interval(3 * k + 1)
    bslot = np.full(mesh.n_facets, -1, dtype=np.int64)
    bf = np.nonzero(mesh.facet_elems[:, 1] < 0)[0]
    bslot[bf] = np.arange(bf.size)
    for e in range(3):
        xh = basis.ref_edge_points(e, qf.points)                     # (q, 2)
        De = basis.dubiner_values(k, xh)                             # (q, nbs)
        phe = bdm.values(xh)                                         # (q, nb, 2)
        va, vb = (basis.REF_VERTICES[v] for v in basis.REF_EDGES[e])
        x, J, det = geometry(mesh, np.arange(NT), xh)
        tang = np.einsum("nqcd,d->nqc", J, vb - va)                  # dx/dt
        speed = np.hypot(tang[..., 0], tang[..., 1])
        nrm = np.stack([tang[..., 1], -tang[..., 0]], axis=-1) / speed[..., None]   # outward (CCW)
        ue = np.einsum("nqcd,qjd,nj->nqc", J, phe, u_loc) / det[..., None]
        un = np.einsum("nqc,nqc->nq", ue, nrm)
        own = np.einsum("qm,ncm->nqc", De, W)
        for T in range(NT):
            inflow_pts = un[T] < 0.0
            f = int(mesh.elem_facets[T, e])
            side = 0 if mesh.facet_elems[f, 0] == T else 1
            nbr = int(mesh.facet_elems[f, 1 - side])
            ext = own[T].copy()
            if not inflow_pts.any():
                pass                                                 # outflow only: w_hat = own trace
            elif nbr >= 0:
                xn = _pull_back(mesh, nbr, x[T])
                Dn = basis.dubiner_values(k, xn)
                ext = np.einsum("qm,cm->qc", Dn, W[nbr])
            elif inflow is not None:
                ext = np.asarray(inflow[bslot[f]], dtype=float)      # owner's traversal = this edge
            wt = qf.weights * speed[T] * un[T]
            hat = np.where(inflow_pts[:, None], ext, own[T])
            r[T] += np.einsum("q,qc,qm->cm", wt, hat, De)
    return r.reshape(NT, 2 * nbs)


def mass_blocks(mesh, k, basis=None):
    """M_T[m, n] = int_T z_m z_n dx = int D_m D_n detJ dx_hat, (NT, nbs, nbs)
    (diagonal detJ/2 on affine elements, full on curved ones)."""
    basis = _provider(basis)
    g = _curved_order(mesh)
    q = basis.quad_triangle(2 * k + 2 * (g - 1))
    D = basis.dubiner_values(k, q.points)
    _, _, det = geometry(mesh, np.arange(mesh.n_elements), q.points)
    return np.einsum("p,np,pm,pl->nml", q.weights, det, D, D)


def mass_inverse_apply(mesh, k, basis=None):
    """Callable r -> (M^V)^{-1} r with the block-diagonal V_h mass."""
    M = mass_blocks(mesh, k, basis)
    Minv = np.linalg.inv(M)
    nbs = M.shape[1]

    def apply(r):
        R = np.asarray(r).reshape(len(Minv), 2, nbs)
        return np.einsum("nml,ncl->ncm", Minv, R).reshape(len(Minv), 2 * nbs)
    return apply


def transfer_I(mesh, k, u_loc, basis=None):
    """I u: element-wise L2 projection of the Piola field onto V_h
    (PAPER.md:473-475): M_T^{-1} int_T u . z_{c,m} dx."""
    basis = _provider(basis)
    g = _curved_order(mesh)
    q = basis.quad_triangle(2 * k + g + 1)
    bdm = basis.build_bdm_basis(k)
    D = basis.dubiner_values(k, q.points)
    phi = bdm.values(q.points)
    NT = mesh.n_elements
    _, J, det = geometry(mesh, np.arange(NT), q.points)
    u = np.einsum("npcd,pjd,nj->npc", J, phi, u_loc) / det[..., None]
    rhs = np.einsum("p,np,npc,pm->ncm", q.weights, det, u, D)
    Minv = np.linalg.inv(mass_blocks(mesh, k, basis))
    return np.einsum("nml,ncl->ncm", Minv, rhs).reshape(NT, -1)


def transfer_IT(mesh, k, r_v, basis=None):
    """I^T r: r_W[j] = sum_i I_T[i, j] r_V[i], columns of I_T
    from unit BDM coefficient vectors."""
    nb = r_v.shape[1]
    out = np.empty_like(r_v)
    for j in range(nb):
        e = np.zeros_like(r_v)
        e[:, j] = 1.0
        out[:, j] = np.einsum("ni,ni->n", transfer_I(mesh, k, e, basis), r_v)
    return out


def substeps(mesh, k, u_loc, w0, dt, nsteps, inflow=None, basis=None):
    """Forward Euler w <- w - dt (M^V)^{-1} C^V(u; w) with the block mass."""
    minv = mass_inverse_apply(mesh, k, basis)
    w = np.array(w0, dtype=float, copy=True)
    for _ in range(nsteps):
        w = w - dt * minv(apply_convection(mesh, k, u_loc, w, inflow, basis))
    return w
