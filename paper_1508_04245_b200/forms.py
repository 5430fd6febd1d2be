"""Drop-in host interface for the convection path (mirrors ``forms`` in SPEC).

Reference interface (module ``forms``):

* ``apply_convection(u_conv, w, data) -> residual over V_h``
* ``apply_transfer(direction in {I, I_transpose}, vec)``
* ``assemble_mass(spaces, which='M_V')``  (diagonal on affine)

Same argument order and meaning; the arithmetic runs in the CUDA library
``libhdgconv.so`` (include/hdgconv.h) — there is no CPU path.  Inputs may be
torch CUDA fp64 tensors (zero copy, asynchronous on the current stream) or
numpy arrays (copied in, result copied out).  Layouts are element-local
(SURVEY.md A.1): ``u`` (NT, nb) BDM coefficients, ``w``/``r`` (NT, nb) V_h
coefficients with index c*nbs+m.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from . import basis as B

__all__ = ["FESpace", "FEField", "ConvectionData", "ConvectionOperator", "operator_for",
           "apply_convection", "apply_convection_W", "apply_convection_U", "apply_transfer", "assemble_mass",
           "device_tables", "clear_cache"]


# ---------------------------------------------------------------------------
# spaces / fields (the subset of fespace.FESpace / FEField the path needs,
# SPEC.md:177-199)


@dataclass(frozen=True)
class FESpace:
    """kind in {'Hdiv', 'VectorDG'}; element-local layouts of size nb per element."""

    mesh: object
    kind: str
    k: int

    @property
    def nb(self) -> int:
        return B.nb_of(self.k)

    @property
    def ndof(self) -> int:
        """Hdiv(k) #facets (k+1) + #elements (k+1)(k-1) (global,
        2D); VectorDG(k) #elements (k+1)(k+2) (element-local storage)."""
        if self.kind == "Hdiv" and hasattr(self.mesh, "facet_flip"):
            from .fespace import hdiv_ndof
            return hdiv_ndof(self.mesh.n_facets, self.mesh.n_elements, self.k)
        return self.mesh.n_elements * self.nb

    def dofmap(self):
        """Global H(div) dof map (fespace.py), cached per space."""
        from .fespace import build_hdiv_dofmap
        per_mesh = _DOFMAPS.setdefault(self.mesh, {})
        dm = per_mesh.get(self.k)
        if dm is None:
            dm = per_mesh[self.k] = build_hdiv_dofmap(self.mesh, self.k)
        return dm


# mesh -> {k: HdivDofMap}; weak keys: an entry goes away with its mesh
_DOFMAPS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


@dataclass
class FEField:
    space: FESpace
    coeffs: object          # (NT, nb) numpy array or torch CUDA tensor


@dataclass
class ConvectionData:
    """t-dependent data of apply_convection: the exterior (Dirichlet) value
    on boundary facets, (NBF, nf, 2) at quad_interval(3k+1) points
    (SPEC.md:302).  ``inflow=None`` means no inflow data (own trace)."""

    inflow: object = None
    t: float = 0.0


# ---------------------------------------------------------------------------
# tables


def device_tables(k: int) -> dict:
    """Reference tables uploaded once per context."""
    bdm = B.build_bdm_basis(k)
    qv = B.volume_rule(k)
    qf = B.facet_rule(k)
    D, G = B.dubiner_values(k, qv.points, with_grads=True)
    fD = np.stack([B.dubiner_values(k, B.ref_edge_points(e, qf.points)) for e in range(3)])
    return {
        "coef": np.ascontiguousarray(bdm.coef),
        "div_modal": np.ascontiguousarray(B.bdm_divergence_modal(k)),
        "vol_w": np.ascontiguousarray(qv.weights),
        "vol_D": np.ascontiguousarray(D),
        "vol_G": np.ascontiguousarray(G),
        "fac_w": np.ascontiguousarray(qf.weights),
        "fac_L": np.ascontiguousarray(B.legendre_values(k, qf.points)),
        "fac_D": np.ascontiguousarray(fD),
        "fac_len": np.ascontiguousarray(B.REF_EDGE_LENGTHS),
        "nqv": qv.weights.size,
        "nf": qf.weights.size,
    }


def device_tables3(k: int) -> dict:
    """3D (tetrahedra) tables: the same fields as device_tables, with the face
    normal-trace basis fac_L = 2 D2_m(s_q, t_q) (dual of the face moments,
    Gram I/2) and fac_len = 2|f| (the face Jacobian ds_hat / (ds dt))."""
    from . import basis3d as B3
    bdm = B3.build_bdm3_basis(k)
    qv = B3.volume_rule3(k)
    qf = B3.face_rule(k)
    D, G = B3.dubiner3_values(k, qv.points, with_grads=True)
    fD = np.stack([B3.dubiner3_values(k, B3.face_points(f, qf.points)) for f in range(4)])
    c = np.ascontiguousarray
    return {
        "coef": c(bdm.coef), "div_modal": c(B3.bdm3_divergence_modal(k)),
        "vol_w": c(qv.weights), "vol_D": c(D), "vol_G": c(G),
        "fac_w": c(qf.weights), "fac_L": c(2.0 * B.dubiner_values(k, qf.points)),
        "fac_D": c(fD), "fac_len": c(2.0 * B3.TET_FACE_AREAS),
        "nqv": qv.weights.size, "nf": qf.weights.size,
        "col3": _collapsed3(k),
    }


def _collapsed3(k: int) -> dict:
    """Sum-factorisation tables for the 3D kernel (basis3d.collapsed_tables3)
    plus the per-point factors of the flux-form coefficients
    alpha = w (u_x + a (u_y + u_z)) / t1, beta = w (u_y + b u_z) / t2, gamma = w u_z,
    with t1 = (1-b)(1-c), t2 = 1-c (chain rule of the collapsed map)."""
    from . import basis3d as B3
    t = B3.collapsed_tables3(k)
    q = B3.volume_rule3(k)
    n = t["n"]
    C3, B3_, A3 = np.meshgrid(t["c"], t["b"], t["a"], indexing="ij")   # point order c, b, a
    t1 = ((1 - B3_) * (1 - C3)).ravel()
    t2 = (1 - C3).ravel()
    a, b, w = A3.ravel(), B3_.ravel(), q.weights
    pf = np.stack([w / t1, w * a / t1, w / t2, w * b / t2, w], axis=1)
    c = np.ascontiguousarray
    return {"n": n, "A": c(t["A"]), "Ad": c(t["Ad"]), "B": c(t["B"]), "Bd": c(t["Bd"]),
            "C": c(t["C"]), "Cd": c(t["Cd"]), "pf": c(pf)}


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# device context


def _torch():
    import torch
    return torch


class ConvectionOperator:
    """Device context for C^V on one mesh (affine, or with curved boundary
    elements) and order k.

    Owns the uploaded tables, the on-device geometry (Piola factors J/detJ,
    2/detJ) and the element-owned neighbour codes; compute calls allocate
    nothing except their outputs.
    """

    def __init__(self, mesh, k: int, weak_mesh: bool = False, builtin_tables: bool = False):
        lib = _lib.load()
        # operator_for's cache holds contexts by weak mesh reference, so the
        # context (and its device memory) is released together with its mesh
        self._mesh = weakref.ref(mesh) if weak_mesh else mesh
        self.k = int(k)
        self.dim = 3 if hasattr(mesh, "tets") else 2
        if self.dim == 3:
            from . import basis3d as B3
            self.nbs = B3.nbs3_of(k)
            self.nb = 3 * self.nbs
        else:
            self.nb = B.nb_of(k)
            self.nbs = B.nbs_of(k)
        keep = []

        def arr(x, dt=np.float64):
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return _ptr(a)

        md = _lib.MeshDesc(
            dim=self.dim, n_vertices=len(mesh.vertices), n_elements=mesh.n_elements,
            n_facets=mesh.n_facets, vertices=arr(mesh.vertices), elements=arr(mesh.triangles, np.int64),
            facet_elems=arr(mesh.facet_elems, np.int64), facet_local=arr(mesh.facet_local, np.int64),
            facet_perm=None)
        td = None
        if not builtin_tables:
            tab = device_tables3(k) if self.dim == 3 else device_tables(k)
            td = _lib.TablesDesc(
                k=self.k, nqv=tab["nqv"], nf=tab["nf"], coef=arr(tab["coef"]), div_modal=arr(tab["div_modal"]),
                vol_w=arr(tab["vol_w"]), vol_D=arr(tab["vol_D"]), vol_G=arr(tab["vol_G"]),
                fac_w=arr(tab["fac_w"]), fac_L=arr(tab["fac_L"]), fac_D=arr(tab["fac_D"]),
                fac_len=arr(tab["fac_len"]))
            if self.k >= 3 and self.dim == 2:
                ct = B.collapsed_tables(self.k)
                td.col_n = ct["n"]
                for name in ("A", "Ad", "B", "Bd", "xi", "wa", "wy", "inv1my"):
                    setattr(td, "col_" + name, arr(ct[name]))
            if self.dim == 3:
                ct = tab["col3"]
                td.col_n = ct["n"]
                for name in ("A", "Ad", "B", "Bd", "C", "Cd", "pf"):
                    setattr(td, "col_" + name, arr(ct[name]))
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("ConvectionOperator needs a CUDA device (no CPU fallback)")
        torch.cuda.init()
        h = C.c_void_p()
        if builtin_tables:
            # the library's own build-time tables (hdgc_create_k): what a non-Python caller uses
            _lib.check(lib.hdgc_create_k(C.byref(md), C.c_int32(self.k), C.byref(h)), "hdgc_create_k")
        else:
            _lib.check(lib.hdgc_create(C.byref(md), C.byref(td), C.byref(h)), "hdgc_create")
        self._h = h
        self._fin = weakref.finalize(self, lib.hdgc_destroy, h)
        info = _lib.Info()
        _lib.check(lib.hdgc_get_info(h, C.byref(info)), "hdgc_get_info")
        self.info = info
        self.nf = info.nf
        self.nqv = info.nqv
        self.n_elements = info.n_elements
        self.n_boundary_facets = info.n_boundary_facets
        self.curved = None
        if self.dim == 2 and getattr(mesh, "curved_maps", None):
            # isoparametric elements along curved boundaries (MESH:555-615): block
            # mass inverse, L2-projection transfer, per-point Piola
            from .curved import curved_tables
            ctab = curved_tables(mesh, self.k)
            self.curved = ctab
            n = int(ctab["elems"].size)
            _lib.check(lib.hdgc_set_curved(h, n, arr(ctab["elems"], np.int32), arr(ctab["minv"]),
                                           arr(ctab["itrans"]), arr(ctab["piola"])), "hdgc_set_curved")

    # -- helpers ---------------------------------------------------------------

    @property
    def mesh(self):
        return self._mesh() if isinstance(self._mesh, weakref.ref) else self._mesh

    def close(self):
        """Release the device context now (otherwise at garbage collection)."""
        self._fin()

    @property
    def handle(self):
        return self._h

    @staticmethod
    def _stream():
        return C.c_void_p(_torch().cuda.current_stream().cuda_stream)

    def _dev(self, x, shape, name):
        torch = _torch()
        if isinstance(x, torch.Tensor):
            if not x.is_cuda or x.dtype != torch.float64:
                raise TypeError(f"{name}: expected a CUDA float64 tensor")
            t = x.contiguous()
            if t.data_ptr() % 16:
                # the kernels move rows with 16-byte vector loads and TMA bulk
                # copies (include/hdgconv.h: pointers must be 16-byte aligned)
                t = t.clone()
            host = False
        else:
            a = np.ascontiguousarray(x, dtype=np.float64)
            t = torch.from_numpy(a).cuda()
            host = True
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
        return t, host

    def _vec_shape(self):
        return (self.n_elements, self.nb)

    def _inflow(self, inflow):
        if inflow is None:
            return None, None
        t, _ = self._dev(inflow, (self.n_boundary_facets, self.nf, self.dim), "inflow")
        return t, C.c_void_p(t.data_ptr())

    # -- operators -------------------------------------------------------------

    def apply(self, u, w, inflow=None, out=None):
        """r = C^V(u; w)."""
        torch = _torch()
        lib = _lib.load()
        ut, host = self._dev(u, self._vec_shape(), "u_conv")
        wt, host2 = self._dev(w, self._vec_shape(), "w")
        it, ip = self._inflow(inflow)
        r = out if out is not None else torch.empty_like(wt)
        _lib.check(lib.hdgc_apply_v(self._h, C.c_void_p(ut.data_ptr()), C.c_void_p(wt.data_ptr()), ip,
                                    C.c_void_p(r.data_ptr()), self._stream()), "hdgc_apply_v")
        return r.cpu().numpy() if (host and host2 and out is None) else r

    def apply_host(self, u: np.ndarray, w: np.ndarray, inflow: Optional[np.ndarray] = None) -> np.ndarray:
        """End-to-end apply on host arrays through hdgc_apply_v_host (H2D,
        kernel, D2H inside the library)."""
        lib = _lib.load()
        u = np.ascontiguousarray(u, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        r = np.empty_like(w)
        ip = None
        if inflow is not None:
            inflow = np.ascontiguousarray(inflow, dtype=np.float64)
            ip = _ptr(inflow)
        _lib.check(lib.hdgc_apply_v_host(self._h, _ptr(u), _ptr(w), ip, _ptr(r), self._stream()),
                   "hdgc_apply_v_host")
        return r

    def apply_w(self, u, inflow=None, out=None):
        """r_W = I^T C^V(u; I u) in BDM-test layout."""
        torch = _torch()
        lib = _lib.load()
        ut, host = self._dev(u, self._vec_shape(), "u_conv")
        it, ip = self._inflow(inflow)
        r = out if out is not None else torch.empty_like(ut)
        _lib.check(lib.hdgc_apply_w(self._h, C.c_void_p(ut.data_ptr()), ip, C.c_void_p(r.data_ptr()),
                                    self._stream()), "hdgc_apply_w")
        return r.cpu().numpy() if (host and out is None) else r

    def transfer(self, vec, transpose: bool = False):
        """I vec (BDM -> V_h) or I^T vec."""
        torch = _torch()
        lib = _lib.load()
        xt, host = self._dev(vec, self._vec_shape(), "vec")
        y = torch.empty_like(xt)
        _lib.check(lib.hdgc_transfer(self._h, 1 if transpose else 0, C.c_void_p(xt.data_ptr()),
                                     C.c_void_p(y.data_ptr()), self._stream()), "hdgc_transfer")
        return y.cpu().numpy() if host else y

    def substeps(self, u, w, dt: float, nsteps: int, inflow=None):
        """nsteps forward-Euler substeps of dw/ds = -(M^V)^{-1} C^V(u) w, u frozen,
        device-resident.  Torch input is updated in place."""
        lib = _lib.load()
        ut, _ = self._dev(u, self._vec_shape(), "u_conv")
        wt, host = self._dev(w, self._vec_shape(), "w")
        it, ip = self._inflow(inflow)
        if not host and wt.data_ptr() != w.data_ptr():
            raise ValueError("w must be contiguous and 16-byte aligned for the in-place substep loop")
        _lib.check(lib.hdgc_substeps(self._h, C.c_void_p(ut.data_ptr()), C.c_void_p(wt.data_ptr()), ip,
                                     C.c_double(dt), C.c_int32(nsteps), self._stream()), "hdgc_substeps")
        if host:
            self.check_finite()
            return wt.cpu().numpy()
        return wt

    def check_finite(self):
        """Norm-blowup guard: synchronise the current stream and
        raise NormBlowupError if any update since the last check wrote a
        non-finite value (hdgc_check_finite)."""
        _lib.check(_lib.load().hdgc_check_finite(self._h, self._stream()), "norm-blowup guard")

    def substeps_host(self, u: np.ndarray, w: np.ndarray, dt: float, nsteps: int,
                      inflow: Optional[np.ndarray] = None, inplace: bool = False) -> np.ndarray:
        """End-to-end substep batch on host arrays (hdgc_substeps_host).
        ``inplace=True`` updates ``w`` itself (C-contiguous fp64, ideally
        pinned): no host-side copy, the device reads and writes the caller's
        buffer directly."""
        lib = _lib.load()
        u = np.ascontiguousarray(u, dtype=np.float64)
        if inplace:
            if not (isinstance(w, np.ndarray) and w.dtype == np.float64 and w.flags.c_contiguous
                    and w.flags.writeable):
                raise ValueError("inplace substeps_host needs a writeable C-contiguous float64 array")
            out = w
        else:
            out = np.array(w, dtype=np.float64, copy=True, order="C")
        ip = None
        if inflow is not None:
            inflow = np.ascontiguousarray(inflow, dtype=np.float64)
            ip = _ptr(inflow)
        _lib.check(lib.hdgc_substeps_host(self._h, _ptr(u), _ptr(out), ip, C.c_double(dt),
                                          C.c_int32(nsteps), self._stream()), "hdgc_substeps_host")
        return out

    def propagate(self, u_cur, w, ds: float, nsteps: int, inflow=None, scheme: str = "euler",
                  u_prev=None, t_prev: float = 0.0, t_cur: float = 0.0, t1: float = 0.0):
        """nsteps explicit substeps of dv/ds = -(M^V)^{-1} C^V(u(s)) v from pseudo
        time t1: scheme "euler" or "ssprk2" (Heun).  u(s) =
        u_cur if u_prev is None, else the linear extrapolation through
        (t_prev, u_prev), (t_cur, u_cur).  Torch input is updated in place."""
        lib = _lib.load()
        if scheme not in ("euler", "ssprk2"):
            raise ValueError("scheme must be 'euler' or 'ssprk2'")
        ut, _ = self._dev(u_cur, self._vec_shape(), "u_cur")
        pp = None
        if u_prev is not None:
            pt, _ = self._dev(u_prev, self._vec_shape(), "u_prev")
            pp = C.c_void_p(pt.data_ptr())
        wt, host = self._dev(w, self._vec_shape(), "w")
        it, ip = self._inflow(inflow)
        if not host and wt.data_ptr() != w.data_ptr():
            raise ValueError("w must be contiguous and 16-byte aligned for the in-place propagation")
        _lib.check(lib.hdgc_propagate(self._h, pp, C.c_void_p(ut.data_ptr()), C.c_double(t_prev),
                                      C.c_double(t_cur), C.c_double(t1), C.c_double(ds), C.c_int32(nsteps),
                                      C.c_int32(0 if scheme == "euler" else 1), ip, C.c_void_p(wt.data_ptr()),
                                      self._stream()), "hdgc_propagate")
        if host:
            self.check_finite()
            return wt.cpu().numpy()
        return wt

    def richardson(self, u, g, v0, tau: float, ds: float, rho: float = 1e-3, max_iter: int = 500,
                   inflow=None):
        """Richardson / pseudo-time solve of v + tau (M^V)^{-1} C^V v = g
        (PAPER.md:671-687).  Returns (v, iterations, converged, res0, res)."""
        lib = _lib.load()
        ut, _ = self._dev(u, self._vec_shape(), "u_conv")
        gt, _ = self._dev(g, self._vec_shape(), "g")
        vt, host = self._dev(v0, self._vec_shape(), "v0")
        if vt.data_ptr() == getattr(v0, "data_ptr", lambda: None)():
            vt = vt.clone()
        it, ip = self._inflow(inflow)
        iters, r0, r1 = C.c_int32(0), C.c_double(0.0), C.c_double(0.0)
        rc = lib.hdgc_richardson(self._h, C.c_void_p(ut.data_ptr()), C.c_void_p(gt.data_ptr()), ip,
                                 C.c_double(tau), C.c_double(ds), C.c_double(rho), C.c_int32(max_iter),
                                 C.c_void_p(vt.data_ptr()), C.byref(iters), C.byref(r0), C.byref(r1),
                                 self._stream())
        if rc not in (0, _lib.HDGC_ENOCONV):
            _lib.check(rc, "hdgc_richardson")
        v = vt.cpu().numpy() if host else vt
        return v, int(iters.value), rc == 0, float(r0.value), float(r1.value)

    # -- global H(div) numbering ---------------------------------------------------

    def set_dofmap(self, dm):
        """Install a fespace.HdivDofMap on the device (hdgc_set_dofmap)."""
        lib = _lib.load()
        d = np.ascontiguousarray(dm.element_dofs, dtype=np.int64)
        f = np.ascontiguousarray(dm.factors, dtype=np.float64)
        if d.shape != self._vec_shape() or f.shape != self._vec_shape():
            raise ValueError("dof map shape does not match the context")
        _lib.check(lib.hdgc_set_dofmap(self._h, C.c_int64(dm.ndof), d.ctypes.data_as(C.c_void_p), _ptr(f)),
                   "hdgc_set_dofmap")
        self._ndof = int(dm.ndof)

    def _need_dofmap(self):
        if getattr(self, "_ndof", None) is None:
            from .fespace import build_hdiv_dofmap
            self.set_dofmap(build_hdiv_dofmap(self.mesh, self.k))
        return self._ndof

    def gather(self, u_glob):
        """u_loc (NT, nb) = factors * u_glob[element_dofs]."""
        torch = _torch()
        lib = _lib.load()
        nd = self._need_dofmap()
        gt, host = self._dev(u_glob, (nd,), "u_glob")
        out = torch.empty(self._vec_shape(), dtype=torch.float64, device="cuda")
        _lib.check(lib.hdgc_gather(self._h, C.c_void_p(gt.data_ptr()), C.c_void_p(out.data_ptr()), self._stream()),
                   "hdgc_gather")
        return out.cpu().numpy() if host else out

    def scatter(self, r_loc):
        """r_glob (ndof,) = global I^T assembly of element-local r_loc (NT, nb)."""
        torch = _torch()
        lib = _lib.load()
        nd = self._need_dofmap()
        rt, host = self._dev(r_loc, self._vec_shape(), "r_loc")
        out = torch.empty(nd, dtype=torch.float64, device="cuda")
        _lib.check(lib.hdgc_scatter(self._h, C.c_void_p(rt.data_ptr()), C.c_void_p(out.data_ptr()), self._stream()),
                   "hdgc_scatter")
        return out.cpu().numpy() if host else out

    def apply_u(self, u_glob, inflow=None):
        """C^U u in global numbering: scatter(I^T C^V(I u_loc; I u_loc)), u_loc = gather(u_glob)."""
        torch = _torch()
        lib = _lib.load()
        nd = self._need_dofmap()
        gt, host = self._dev(u_glob, (nd,), "u_glob")
        it, ip = self._inflow(inflow)
        out = torch.empty(nd, dtype=torch.float64, device="cuda")
        _lib.check(lib.hdgc_apply_u(self._h, C.c_void_p(gt.data_ptr()), ip, C.c_void_p(out.data_ptr()),
                                    self._stream()), "hdgc_apply_u")
        return out.cpu().numpy() if host else out

    def mass_inverse(self):
        """(M^V)^{-1} diagonal: 2/detJ per element.  On a
        curved mesh the curved rows hold -(slot + 1); their full blocks are
        ``self.curved["minv"][slot]``."""
        torch = _torch()
        lib = _lib.load()
        out = torch.empty(self.n_elements, dtype=torch.float64, device="cuda")
        _lib.check(lib.hdgc_mass_inverse(self._h, C.c_void_p(out.data_ptr()), self._stream()),
                   "hdgc_mass_inverse")
        return out

    def max_speed(self, u) -> float:
        """max |u| over elements x volume points (for the CFL substep)."""
        torch = _torch()
        lib = _lib.load()
        ut, _ = self._dev(u, self._vec_shape(), "u_conv")
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.check(lib.hdgc_max_speed(self._h, C.c_void_p(ut.data_ptr()), C.c_void_p(out.data_ptr()),
                                      self._stream()), "hdgc_max_speed")
        return float(out.item())


# mesh -> {k: ConvectionOperator}.  Weak keys and weak mesh references inside
# the cached operators: when the caller drops a mesh, its contexts are
# destroyed (hdgc_destroy via the operator's finalizer) and the device memory
# is returned, so loops that build many meshes do not accumulate contexts.
_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def operator_for(mesh, k: int) -> ConvectionOperator:
    """Context cache keyed by (mesh, k): building a context uploads tables and
    runs the geometry precompute, so do it once per mesh and order."""
    per_mesh = _CACHE.setdefault(mesh, {})
    op = per_mesh.get(int(k))
    if op is None:
        op = per_mesh[int(k)] = ConvectionOperator(mesh, k, weak_mesh=True)
    return op


def clear_cache() -> None:
    """Destroy every cached context now (operator_for / FESpace.dofmap)."""
    for per_mesh in list(_CACHE.values()):
        for op in per_mesh.values():
            op.close()
    _CACHE.clear()
    _DOFMAPS.clear()


# ---------------------------------------------------------------------------
# reference-named entry points


def apply_convection(u_conv: FEField, w, data: Optional[ConvectionData] = None):
    """``forms.apply_convection(u_conv, w, data)``.

    u_conv: FEField over Hdiv(k) (element-local BDM coefficients);
    w: V_h coefficients (NT, nb) (array/tensor or FEField over VectorDG(k));
    data: ConvectionData (inflow values).  Returns the residual r over V_h.
    Pure: inputs are not modified.  Errors: none beyond argument checks.
    """
    sp = u_conv.space
    op = operator_for(sp.mesh, sp.k)
    wc = w.coeffs if isinstance(w, FEField) else w
    inflow = None if data is None else data.inflow
    return op.apply(u_conv.coeffs, wc, inflow)


def apply_convection_W(u_conv: FEField, data: Optional[ConvectionData] = None):
    """C^U u = I^T C^V(u; I u) in the BDM-test layout."""
    sp = u_conv.space
    op = operator_for(sp.mesh, sp.k)
    return op.apply_w(u_conv.coeffs, None if data is None else data.inflow)


def apply_convection_U(u_glob, space: FESpace, data: Optional[ConvectionData] = None):
    """C^U u in the global H(div) numbering (fespace dof map): the convection
    right-hand side of the Stokes solve."""
    op = operator_for(space.mesh, space.k)
    if getattr(op, "_ndof", None) is None:
        op.set_dofmap(space.dofmap())
    return op.apply_u(u_glob, None if data is None else data.inflow)


def apply_transfer(direction: str, vec, space: FESpace):
    """``forms.apply_transfer``: direction 'I' maps BDM
    coefficients to V_h, 'I_transpose' maps V_h functionals to BDM-test."""
    if direction not in ("I", "I_transpose"):
        raise ValueError(f"unknown transfer direction {direction!r}")
    return operator_for(space.mesh, space.k).transfer(vec, transpose=direction == "I_transpose")


def assemble_mass(space: FESpace, which: str = "M_V"):
    """Diagonal M^V on affine meshes: detJ/2 per element and mode
    (SPEC.md:280-289), returned as its (NT,) inverse
    scale 2/detJ as a CUDA tensor."""
    if which != "M_V":
        raise ValueError("only the V_h mass (M_V) is part of the convection path")
    return operator_for(space.mesh, space.k).mass_inverse()
