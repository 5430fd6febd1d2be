"""ORACLE — test infrastructure only.  CPU restatement of the reference's
convection apply; never imported by the product package.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker.

What it restates
----------------
The reference package does not implement ``forms.apply_convection``; it
exists as a contract over the paper's upwind-DG trilinear
form.  This module evaluates that contract literally, in
physical coordinates and facet-wise, on top of a *basis provider* (a module
exposing the ``hdgflow.polybasis`` API) and a *mesh* (any object with the
``hdgflow.mesh2d.Mesh`` attributes):

    r[T, c*nbs+m] = - sum_T int_T (w (x) u) : grad z_{c,m} dx
                    + int_{dT} (u . n) w_hat . z_{c,m} ds
    w_hat = own trace if u.n >= 0 else the neighbour's trace
            (the Dirichlet inflow value on boundary facets)
    u(x) = J u_hat(x_hat) / detJ   (contravariant Piola)
    z_{c,m}(x) = e_c D_m(F_T^{-1} x)   (V_h basis, L2-orthogonal)
    volume rule quad_triangle(3k+1), facet rule quad_interval(3k+1)
    facets visited once, contributions to both sides

Unlike the device path it does NOT use the geometry-free reference form
(SURVEY A.3): physical points, J^{-T} gradients, physical normals and arc
length are used throughout, and neighbour traces are found by pulling the
physical facet points back through the neighbour's own affine map (no
reversal convention assumed).  Agreement with the device therefore checks
the geometry cancellation, the edge-flux shortcut and the
neighbour-orientation logic independently.

Parity pin: with the reference's own ``hdgflow.polybasis`` and
``hdgflow.mesh2d`` plugged in (``tests/golden/make_golden.py``, run where
/root/reference exists) this module produced the committed golden vectors
``tests/golden/conv_*.npz``.  The operator itself has no golden vector in
the reference: its outputs are pinned by those fixtures plus
the SPEC known-answer properties.
"""

from __future__ import annotations

import numpy as np

__all__ = ["apply_convection", "transfer_I", "transfer_IT", "mass_inverse", "substeps",
           "quadratic_form_inflow"]


def _provider(basis):
    if basis is None:
        from paper_1508_04245_b200 import basis as default   # tables only
        return default
    return basis


def _tables(basis, k):
    qv = basis.quad_triangle(3 * k + 1)
    qf = basis.quad_interval(3 * k + 1)
    bdm = basis.build_bdm_basis(k)
    return qv, qf, bdm


def transfer_I(mesh, k, u_loc, basis=None):
    """I u: V_h coefficients of the Piola
    field by L2 projection with the diagonal V_h mass (exact embedding on
    affine elements)."""
    basis = _provider(basis)
    q = basis.quad_triangle(2 * k)
    bdm = basis.build_bdm_basis(k)
    D = basis.dubiner_values(k, q.points)                      # (p, nbs)
    phi = bdm.values(q.points)                                 # (p, nb, 2)
    uh = np.einsum("pjd,nj->npd", phi, u_loc)
    u = np.einsum("ncd,npd->npc", mesh.affine_jac, uh) / mesh.affine_det[:, None, None]
    # (M^V)^{-1} M^{U,V} u with int_T D_m D_m' = detJ/2 delta: projection
    w = 2.0 * np.einsum("p,pm,npc->ncm", q.weights, D, u)
    return w.reshape(len(u_loc), -1)


def transfer_IT(mesh, k, r_v, basis=None):
    """I^T r: r_W[j] = sum_i I[i, j] r_V[i], with I assembled
    column by column from the embedding of each BDM member."""
    basis = _provider(basis)
    nb = r_v.shape[1]
    eye = np.eye(nb)
    out = np.empty_like(r_v)
    # I_T columns: I applied to unit BDM coefficient vectors (per element)
    for j in range(nb):
        cols = transfer_I(mesh, k, np.broadcast_to(eye[j], r_v.shape).copy(), basis)
        out[:, j] = np.einsum("ni,ni->n", cols, r_v)
    return out


def mass_inverse(mesh):
    """(M^V)^{-1} per element on affine meshes: 2/detJ."""
    return 2.0 / mesh.affine_det


def _volume(mesh, k, u_loc, w, basis, qv, bdm, r, chunk):
    nbs = w.shape[1] // 2
    D, G = basis.dubiner_values(k, qv.points, with_grads=True)  # (p,nbs), (p,nbs,2)
    phi = bdm.values(qv.points)                                  # (p, nb, 2)
    for s in range(0, mesh.n_elements, chunk):
        sl = slice(s, min(mesh.n_elements, s + chunk))
        J = mesh.affine_jac[sl]
        det = mesh.affine_det[sl]
        Jinv = mesh.affine_inv[sl]
        u = np.einsum("ncd,pjd,nj->npc", J, phi, u_loc[sl]) / det[:, None, None]
        gphys = np.einsum("ndc,pmd->npmc", Jinv, G)              # J^{-T} grad_hat
        wq = np.einsum("pm,ncm->npc", D, w[sl].reshape(-1, 2, nbs))
        ugrad = np.einsum("npd,npmd->npm", u, gphys)             # u . grad D_m
        r[sl] -= np.einsum("p,n,npc,npm->ncm", qv.weights, det, wq, ugrad).reshape(-1, 2 * nbs)


def _facets(mesh, k, u_loc, w, inflow, basis, qf, bdm, r, chunk):
    nbs = w.shape[1] // 2
    fe = mesh.facet_elems
    V = mesh.vertices
    bnd = np.full(mesh.n_facets, -1, dtype=np.int64)
    bf = np.nonzero(fe[:, 1] < 0)[0]
    bnd[bf] = np.arange(bf.size)
    W = w.reshape(-1, 2, nbs)
    for s in range(0, mesh.n_facets, chunk):
        f = np.arange(s, min(mesh.n_facets, s + chunk))
        a = V[mesh.facet_vertices[f, 0]]
        b = V[mesh.facet_vertices[f, 1]]
        X = a[:, None, :] + qf.points[None, :, None] * (b - a)[:, None, :]   # (F, q, 2)
        ds = mesh.facet_h[f][:, None] * qf.weights[None, :]
        n = mesh.facet_normal[f]
        nf = qf.points.size

        def pull(T):
            xh = np.einsum("ncd,nqd->nqc", mesh.affine_inv[T], X - mesh.affine_origin[T][:, None, :])
            return xh.reshape(-1, 2)

        T0 = fe[f, 0]
        xh0 = pull(T0)
        phi0 = bdm.values(xh0).reshape(len(f), nf, -1, 2)
        u0 = np.einsum("ncd,nqjd,nj->nqc", mesh.affine_jac[T0], phi0, u_loc[T0])
        u0 /= mesh.affine_det[T0][:, None, None]
        un = np.einsum("nqc,nc->nq", u0, n)                       # u . n_T0
        D0 = basis.dubiner_values(k, xh0).reshape(len(f), nf, nbs)
        w0 = np.einsum("nqm,ncm->nqc", D0, W[T0])

        inner = fe[f, 1] >= 0
        wext = np.empty_like(w0)
        T1 = fe[f[inner], 1]
        if T1.size:
            xh1 = np.einsum("ncd,nqd->nqc", mesh.affine_inv[T1],
                            X[inner] - mesh.affine_origin[T1][:, None, :]).reshape(-1, 2)
            D1 = basis.dubiner_values(k, xh1).reshape(T1.size, nf, nbs)
            wext[inner] = np.einsum("nqm,ncm->nqc", D1, W[T1])
        if (~inner).any():
            if inflow is None:
                wext[~inner] = w0[~inner]
            else:
                wext[~inner] = inflow[bnd[f[~inner]]]
        what = np.where((un >= 0.0)[..., None], w0, wext)
        flux = (un * ds)[..., None] * what                        # (F, q, c)
        r0 = np.einsum("nqc,nqm->ncm", flux, D0).reshape(len(f), -1)
        np.add.at(r, T0, r0)
        if T1.size:
            r1 = np.einsum("nqc,nqm->ncm", flux[inner], D1).reshape(T1.size, -1)
            np.add.at(r, T1, -r1)


def apply_convection(mesh, k, u_loc, w, inflow=None, basis=None, chunk=8192):
    """r = C^V(u; w) in V_h layout (NT, nb).

    ``inflow`` (NBF, nf, 2) holds the exterior values on boundary facets in
    ``boundary_facets`` order at ``quad_interval(3k+1)`` points along the
    owner's traversal; ``None`` means 'use the interior trace' (outflow
    everywhere), which is exact when u.n = 0 on the boundary."""
    basis = _provider(basis)
    qv, qf, bdm = _tables(basis, k)
    u_loc = np.asarray(u_loc, dtype=float)
    w = np.asarray(w, dtype=float)
    r = np.zeros_like(w)
    _volume(mesh, k, u_loc, w, basis, qv, bdm, r, chunk)
    _facets(mesh, k, u_loc, w, inflow, basis, qf, bdm, r, chunk)
    return r


def substeps(mesh, k, u_loc, w0, dt, nsteps, inflow=None, basis=None):
    """Forward-Euler propagation w <- w - dt (M^V)^{-1} C^V(u; w) with u
    frozen (BASELINE replaces SPEC:432's SSP-RK2)."""
    minv = mass_inverse(mesh)[:, None]
    w = np.array(w0, dtype=float, copy=True)
    for _ in range(nsteps):
        w = w - dt * minv * apply_convection(mesh, k, u_loc, w, inflow, basis)
    return w


def quadratic_form_inflow(mesh, k, u_loc, w, basis=None):
    """Stability identity terms: returns
    (C(u; w, w), 1/2 int_{inflow} |u.n| w^2 ds) with w's own boundary trace."""
    basis = _provider(basis)
    qf = basis.quad_interval(3 * k + 1)
    bdm = basis.build_bdm_basis(k)
    r = apply_convection(mesh, k, u_loc, w, None, basis)
    c = float(np.sum(r * w))
    nbs = w.shape[1] // 2
    bf = mesh.boundary_facets
    T = mesh.facet_elems[bf, 0]
    a = mesh.vertices[mesh.facet_vertices[bf, 0]]
    b = mesh.vertices[mesh.facet_vertices[bf, 1]]
    X = a[:, None, :] + qf.points[None, :, None] * (b - a)[:, None, :]
    xh = np.einsum("ncd,nqd->nqc", mesh.affine_inv[T], X - mesh.affine_origin[T][:, None, :]).reshape(-1, 2)
    nf = qf.points.size
    phi = bdm.values(xh).reshape(len(T), nf, -1, 2)
    u = np.einsum("ncd,nqjd,nj->nqc", mesh.affine_jac[T], phi, u_loc[T]) / mesh.affine_det[T][:, None, None]
    un = np.einsum("nqc,nc->nq", u, mesh.facet_normal[bf])
    D = basis.dubiner_values(k, xh).reshape(len(T), nf, nbs)
    wq = np.einsum("nqm,ncm->nqc", D, w.reshape(-1, 2, nbs)[T])
    ds = mesh.facet_h[bf][:, None] * qf.weights[None, :]
    inflow_term = 0.5 * float(np.sum(np.where(un < 0, -un, 0.0) * (wq ** 2).sum(-1) * ds))
    return c, inflow_term


def apply_convection_flux_form(mesh, k, u_loc, w, inflow=None, basis=None, dtype=np.longdouble):
    """C^V(u; w) in the flux-difference form, element-owned, in `dtype`
    (default x87 long double, eps 1.1e-19):

        r = sum_p w_p (u_hat.grad_hat w_c + w_c div_hat u_hat) D_m
          + sum_e sum_{q: F<0} w_q F (w_ext - w_own)_c D_m(x_e(t_q))

    equal to the textbook form (``apply_convection``) by the divergence
    theorem, since every rule integrates its polynomial integrand exactly
    (volume degree 3k-1 <= 3k+1 rule; facet degree 3k <= 3k+1 rule).  The
    textbook form cancels two O(|w||u|/h) terms into an O(|u||grad w|)
    result, so in fp64 it loses ~log10(1/(h k_flow)) digits; this form in
    extended precision is the high-accuracy reference the fp64 paths are
    measured against (tests/test_oracle.py, tests/test_gpu_parity.py).
    Tables are evaluated in fp64 by the provider and promoted to `dtype`.
    """
    basis = _provider(basis)
    nbs = w.shape[1] // 2
    q = basis.quad_triangle(3 * k + 1)
    D, G = basis.dubiner_values(k, q.points, with_grads=True)
    bdm = basis.build_bdm_basis(k)
    # raw modal divergence table: div(e_c D_m) = d_c D_m
    cast = lambda a: np.asarray(a, dtype=dtype)
    D, G, coef, wq = cast(D), cast(G), cast(bdm.coef), cast(q.weights)
    U = cast(u_loc)
    W = cast(w).reshape(-1, 2, nbs)
    uh = (U @ coef.T).reshape(-1, 2, nbs)
    up = np.einsum("ndm,pm->npd", uh, D)
    div = np.einsum("ndm,pmd->np", uh, G)
    wp = np.einsum("ncm,pm->npc", W, D)
    gw = np.einsum("ncm,pmd->npcd", W, G)
    f = np.einsum("npd,npcd->npc", up, gw) + wp * div[:, :, None]
    r = np.einsum("p,npc,pm->ncm", wq, f, D)
    qf = basis.quad_interval(3 * k + 1)
    L = cast(basis.legendre_values(k, qf.points))
    fD = cast(np.stack([basis.dubiner_values(k, basis.ref_edge_points(e, qf.points)) for e in range(3)]))
    fw = cast(qf.weights)
    elen = np.asarray(basis.REF_EDGE_LENGTHS, dtype=float)
    NT = len(u_loc)
    fe, fl = mesh.facet_elems, mesh.facet_local
    nbr = np.full((NT, 3), -1, dtype=np.int64)
    nbe = np.full((NT, 3), -1, dtype=np.int64)
    bsl = np.full((NT, 3), -1, dtype=np.int64)
    inner = fe[:, 1] >= 0
    for s, o in ((0, 1), (1, 0)):
        nbr[fe[inner, s], fl[inner, s]] = fe[inner, o]
        nbe[fe[inner, s], fl[inner, s]] = fl[inner, o]
    bf = np.nonzero(~inner)[0]
    bsl[fe[bf, 0], fl[bf, 0]] = np.arange(bf.size)
    for e in range(3):
        F = cast(elen[e]) * np.einsum("nl,ql->nq", U[:, e * (k + 1):(e + 1) * (k + 1)], L)
        own = np.einsum("ncm,qm->nqc", W, fD[e])
        ext = own.copy()
        inn = nbr[:, e] >= 0
        # the neighbour traverses the shared edge backwards: point q <-> nf-1-q
        ext[inn] = np.einsum("ncm,nqm->nqc", W[nbr[inn, e]], fD[nbe[inn, e]][:, ::-1, :])
        if inflow is not None:
            bb = ~inn
            ext[bb] = cast(inflow)[bsl[bb, e]]
        jump = np.where((F < 0)[..., None], ext - own, 0)
        r += np.einsum("q,nq,nqc,qm->ncm", fw, F, jump, fD[e])
    return r.reshape(NT, 2 * nbs)
