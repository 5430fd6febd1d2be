"""ORACLE — test infrastructure only.  3D (tetrahedral) restatement of the
convection apply for BASELINE cfg5; never imported by the product.

The reference has no 3D code; this restates the same
SPEC contract and trilinear form on
tetrahedra, on top of a 3D basis provider (``paper_1508_04245_b200.basis3d``,
pinned by tests/test_basis3d.py: quadrature exactness, Gram, BDM duality,
zero interior normal traces, div in P_{k-1}) and a ``TetMesh``:

* ``apply_convection3`` — textbook form in physical coordinates, faces
  visited once with contributions to both sides, neighbour
  traces by pulling the physical face points back through the neighbour's
  own affine map, physical outward normals (no sign(detJ) shortcut);
* ``apply_convection3_flux_form`` — the element-owned geometry-free
  flux-difference form the device uses, in `dtype`
  (default long double): r = sign(detJ) [ sum_p w_p (u_hat.grad w + w div u_hat) D
  + sum_{inflow q} w_q F_hat (w_ext - w_own) D ].
"""

from __future__ import annotations

import numpy as np

__all__ = ["apply_convection3", "apply_convection3_flux_form", "substeps3", "mass_inverse3"]


def _provider(b3):
    if b3 is None:
        from paper_1508_04245_b200 import basis3d as default
        return default
    return b3


def mass_inverse3(mesh):
    """(M^V)^{-1} = 6/|detJ| (Gram I/6 of the tet Dubiner modes)."""
    return 6.0 / np.abs(mesh.affine_det)


def apply_convection3(mesh, k, u_loc, w, inflow=None, b3=None, chunk=4096):
    b3 = _provider(b3)
    from paper_1508_04245_b200 import basis as B2
    nbs = w.shape[1] // 3
    qv = b3.quad_tet(3 * k + 1)
    qf = B2.quad_triangle(3 * k + 1)
    bdm = b3.build_bdm3_basis(k)
    r = np.zeros_like(w, dtype=float)
    W = w.reshape(-1, 3, nbs)
    D, G = b3.dubiner3_values(k, qv.points, with_grads=True)
    phi = bdm.values(qv.points)
    for s in range(0, mesh.n_elements, chunk):
        sl = slice(s, min(mesh.n_elements, s + chunk))
        J, det, Ji = mesh.affine_jac[sl], mesh.affine_det[sl], mesh.affine_inv[sl]
        u = np.einsum("ncd,pjd,nj->npc", J, phi, u_loc[sl]) / det[:, None, None]
        gphys = np.einsum("ndc,pmd->npmc", Ji, G)
        wq = np.einsum("pm,ncm->npc", D, W[sl])
        ugrad = np.einsum("npd,npmd->npm", u, gphys)
        r[sl] -= np.einsum("p,n,npc,npm->ncm", qv.weights, np.abs(det), wq, ugrad).reshape(-1, 3 * nbs)
    fe = mesh.facet_elems
    bnd = np.full(mesh.n_facets, -1, dtype=np.int64)
    bf = np.nonzero(fe[:, 1] < 0)[0]
    bnd[bf] = np.arange(bf.size)
    V = mesh.vertices
    nf = qf.points.shape[0]
    for s in range(0, mesh.n_facets, chunk):
        f = np.arange(s, min(mesh.n_facets, s + chunk))
        a, b, c = (V[mesh.facet_vertices[f, i]] for i in range(3))
        X = a[:, None] + qf.points[None, :, :1] * (b - a)[:, None] + qf.points[None, :, 1:] * (c - a)[:, None]
        cr = np.cross(b - a, c - a)
        area2 = np.linalg.norm(cr, axis=1)
        n = cr / area2[:, None]
        T0 = fe[f, 0]
        # outward for the owner: away from its vertex opposite the face
        opp = V[mesh.tets[T0, mesh.facet_local[f, 0]]]
        flip = np.einsum("nc,nc->n", n, opp - a) > 0
        n[flip] *= -1.0
        ds = area2[:, None] * qf.weights[None, :]          # 2|F| * w (w sums to 1/2)

        def pull(T, Xs):
            return np.einsum("ncd,nqd->nqc", mesh.affine_inv[T], Xs - mesh.affine_origin[T][:, None, :]).reshape(-1, 3)

        x0 = pull(T0, X)
        ph0 = bdm.values(x0).reshape(len(f), nf, -1, 3)
        u0 = np.einsum("ncd,nqjd,nj->nqc", mesh.affine_jac[T0], ph0, u_loc[T0]) / mesh.affine_det[T0][:, None, None]
        un = np.einsum("nqc,nc->nq", u0, n)
        D0 = b3.dubiner3_values(k, x0).reshape(len(f), nf, nbs)
        w0 = np.einsum("nqm,ncm->nqc", D0, W[T0])
        inner = fe[f, 1] >= 0
        wext = np.empty_like(w0)
        T1 = fe[f[inner], 1]
        if T1.size:
            x1 = pull(T1, X[inner])
            D1 = b3.dubiner3_values(k, x1).reshape(T1.size, nf, nbs)
            wext[inner] = np.einsum("nqm,ncm->nqc", D1, W[T1])
        if (~inner).any():
            wext[~inner] = w0[~inner] if inflow is None else inflow[bnd[f[~inner]]]
        what = np.where((un >= 0.0)[..., None], w0, wext)
        flux = (un * ds)[..., None] * what
        np.add.at(r, T0, np.einsum("nqc,nqm->ncm", flux, D0).reshape(len(f), -1))
        if T1.size:
            np.add.at(r, T1, -np.einsum("nqc,nqm->ncm", flux[inner], D1).reshape(T1.size, -1))
    return r


def apply_convection3_flux_form(mesh, k, u_loc, w, inflow=None, b3=None, dtype=np.longdouble, chunk=8192):
    b3 = _provider(b3)
    from paper_1508_04245_b200 import basis as B2
    cast = lambda a: np.asarray(a, dtype=dtype)
    nbs = w.shape[1] // 3
    q = b3.quad_tet(3 * k + 1)
    D, G = b3.dubiner3_values(k, q.points, with_grads=True)
    bdm = b3.build_bdm3_basis(k)
    D, G, coef, wq = cast(D), cast(G), cast(bdm.coef), cast(q.weights)
    qf = B2.quad_triangle(3 * k + 1)
    nf = qf.points.shape[0]
    D2 = B2.dubiner_values(k, qf.points)                        # face modes at face points
    fD = cast(np.stack([b3.dubiner3_values(k, b3.face_points(f, qf.points)) for f in range(4)]))
    nfd = D2.shape[1]
    n_face = 4 * nfd
    sig = np.sign(mesh.affine_det)
    NT = len(u_loc)
    nbr, nbf, bsl = mesh.element_neighbours()
    out = np.empty((NT, 3 * nbs), dtype=dtype)
    for s in range(0, NT, chunk):
        sl = slice(s, min(NT, s + chunk))
        U = cast(u_loc[sl])
        Wl = cast(w[sl]).reshape(-1, 3, nbs)
        uh = (U @ coef.T).reshape(-1, 3, nbs)
        up = np.einsum("ndm,pm->npd", uh, D)
        div = np.einsum("ndm,pmd->np", uh, G)
        wp = np.einsum("ncm,pm->npc", Wl, D)
        gw = np.einsum("ncm,pmd->npcd", Wl, G)
        f_ = np.einsum("npd,npcd->npc", up, gw) + wp * div[:, :, None]
        r = np.einsum("p,npc,pm->ncm", wq, f_, D)
        for fc in range(4):
            # F_hat = 2|f| * u_hat.n_hat = 2|f| * 2 sum_m c_{f,m} D2_m
            cf = U[:, fc * nfd:(fc + 1) * nfd]
            F = cast(2.0 * b3.TET_FACE_AREAS[fc] * 2.0) * np.einsum("nm,qm->nq", cf, cast(D2))
            own = np.einsum("ncm,qm->nqc", Wl, fD[fc])
            ext = own.copy()
            idx = np.arange(sl.start, sl.stop)
            inn = nbr[idx, fc] >= 0
            ext[inn] = np.einsum("ncm,nqm->nqc", cast(w[nbr[idx[inn], fc]]).reshape(-1, 3, nbs),
                                 fD[nbf[idx[inn], fc]])
            if inflow is not None:
                bb = ~inn
                ext[bb] = cast(inflow)[bsl[idx[bb], fc]]
            inflow_pt = (cast(sig[sl])[:, None] * F) < 0
            jump = np.where(inflow_pt[..., None], ext - own, 0)
            r += np.einsum("q,nq,nqc,qm->ncm", cast(qf.weights), F, jump, fD[fc])
        out[sl] = (cast(sig[sl])[:, None, None] * r).reshape(-1, 3 * nbs)
    return out


def substeps3(mesh, k, u_loc, w0, dt, nsteps, inflow=None, b3=None, dtype=np.longdouble):
    minv = np.asarray(mass_inverse3(mesh), dtype=dtype)[:, None]
    w = np.asarray(w0, dtype=dtype).copy()
    for _ in range(nsteps):
        w = w - dt * minv * apply_convection3_flux_form(mesh, k, u_loc, w, inflow, b3, dtype)
    return w.astype(np.float64)
