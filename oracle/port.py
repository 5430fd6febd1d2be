"""ORACLE — test infrastructure only.  ctypes wrapper of oracle/conv_port.c
(the OpenMP C restatement), used as the fast full-size checker and as the
CPU baseline ("kind": "port") in bench.py.  Never imported by the product.

Tables come from a basis provider with the ``hdgflow.polybasis`` API
(default: the package's host basis module, itself pinned against the
reference's tables by tests/test_basis.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "conv_port.c")
SRC3 = os.path.join(HERE, "conv3d_port.c")
LIB = os.path.join(HERE, "build", "liboracle_port.so")

_lib = None


def build(force: bool = False) -> str:
    """gcc -O3 -fopenmp -shared (CPU only; no reference sources involved)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(SRC3)):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-shared", "-fPIC",
                               "-o", LIB + ".tmp", SRC, SRC3])
        os.replace(LIB + ".tmp", LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        vp, i32 = C.c_void_p, C.c_int
        common = [i32, i32, i32, i32] + [vp] * 9 + [vp] * 3 + [vp, vp, vp]
        _lib.port_apply.argtypes = common + [vp, i32]
        _lib.port_apply.restype = C.c_int
        _lib.port_substeps.argtypes = common + [vp, C.c_double, i32, vp, i32]
        _lib.port_substeps.restype = C.c_int
        common3 = [i32, i32, i32, i32] + [vp] * 9 + [vp] * 3 + [vp, vp, vp]
        _lib.port3_apply.argtypes = common3 + [vp, i32]
        _lib.port3_apply.restype = C.c_int
        _lib.port3_substeps.argtypes = common3 + [vp, C.c_double, i32, vp, i32]
        _lib.port3_substeps.restype = C.c_int
    return _lib


def _divergence_modal(basis, k):
    """div of each BDM member in the Dubiner P_{k-1} basis, by exact L2
    projection (Gram I/2, PB:8-9), from the provider's own tables."""
    q = basis.quad_triangle(2 * k)
    D = basis.dubiner_values(k - 1, q.points)
    return 2.0 * (D * q.weights[:, None]).T @ basis.build_bdm_basis(k).divergence(q.points)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class PortOperator:
    """C^V(u; w) on the CPU with `threads` OpenMP threads."""

    def __init__(self, mesh, k, basis=None, threads=None):
        if basis is None:
            from paper_1508_04245_b200 import basis as basis_mod   # tables only
            basis = basis_mod
        self.k = k
        self.threads = int(threads or os.cpu_count() or 1)
        nbs = (k + 1) * (k + 2) // 2
        qv = basis.quad_triangle(3 * k - 1)
        qf = basis.quad_interval(3 * k + 1)
        D, G = basis.dubiner_values(k, qv.points, with_grads=True)
        fD = np.stack([basis.dubiner_values(k, basis.ref_edge_points(e, qf.points)) for e in range(3)])
        c = np.ascontiguousarray
        self.tabs = [c(basis.build_bdm_basis(k).coef), c(_divergence_modal(basis, k)), c(qv.weights), c(D), c(G), c(qf.weights),
                     c(basis.legendre_values(k, qf.points)), c(fD), c(np.asarray(basis.REF_EDGE_LENGTHS))]
        self.nqv, self.nf, self.nbs = qv.weights.size, qf.weights.size, nbs
        nt = mesh.n_elements
        self.nt = nt
        nbr = np.full((nt, 3), -1, dtype=np.int32)
        nbe = np.full((nt, 3), -1, dtype=np.int32)
        bsl = np.full((nt, 3), -1, dtype=np.int32)
        fe, fl = mesh.facet_elems, mesh.facet_local
        inner = fe[:, 1] >= 0
        for s, o in ((0, 1), (1, 0)):
            nbr[fe[inner, s], fl[inner, s]] = fe[inner, o]
            nbe[fe[inner, s], fl[inner, s]] = fl[inner, o]
        bf = np.nonzero(~inner)[0]
        bsl[fe[bf, 0], fl[bf, 0]] = np.arange(bf.size)
        self.adj = [nbr, nbe, bsl]
        self.minv = c(2.0 / mesh.affine_det)

    def _args(self):
        return [self.k, self.nt, self.nqv, self.nf] + [_p(t) for t in self.tabs] + [_p(a) for a in self.adj]

    def apply(self, u, w, inflow=None):
        lib = _load()
        u = np.ascontiguousarray(u, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        inflow = None if inflow is None else np.ascontiguousarray(inflow, dtype=np.float64)
        r = np.empty_like(w)
        lib.port_apply(*self._args(), _p(u), _p(w), _p(inflow), _p(r), self.threads)
        return r

    def substeps(self, u, w, dt, nsteps, inflow=None):
        lib = _load()
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.array(w, dtype=np.float64, copy=True, order="C")
        inflow = None if inflow is None else np.ascontiguousarray(inflow, dtype=np.float64)
        work = np.empty_like(out)
        lib.port_substeps(*self._args(), _p(u), _p(out), _p(inflow), _p(self.minv), C.c_double(dt),
                          int(nsteps), _p(work), self.threads)
        return out


class Port3Operator:
    """3D (tets) C^V(u; w) on the CPU with `threads` OpenMP threads
    (oracle/conv3d_port.c; restates oracle/convection3d.py's flux form)."""

    def __init__(self, mesh, k, b3=None, threads=None):
        from paper_1508_04245_b200 import basis as B2
        if b3 is None:
            from paper_1508_04245_b200 import basis3d as b3   # tables only
        self.k = k
        self.threads = int(threads or os.cpu_count() or 1)
        qv = b3.quad_tet(3 * k + 1)
        qf = B2.quad_triangle(3 * k + 1)
        D, G = b3.dubiner3_values(k, qv.points, with_grads=True)
        fD = np.stack([b3.dubiner3_values(k, b3.face_points(f, qf.points)) for f in range(4)])
        c = np.ascontiguousarray
        self.tabs = [c(b3.build_bdm3_basis(k).coef), c(qv.weights), c(D), c(G), c(qf.weights),
                     c(B2.dubiner_values(k, qf.points)), c(fD), c(np.asarray(b3.TET_FACE_AREAS, dtype=float)),
                     c(np.sign(mesh.affine_det))]
        self.nqv, self.nf = qv.weights.size, qf.weights.size
        self.nt = mesh.n_elements
        nbr, nbf, bsl = mesh.element_neighbours()
        self.adj = [c(nbr, dtype=np.int32), c(nbf, dtype=np.int32), c(bsl, dtype=np.int32)]
        self.minv = c(6.0 / np.abs(mesh.affine_det))

    def _args(self):
        return [self.k, self.nt, self.nqv, self.nf] + [_p(t) for t in self.tabs] + [_p(a) for a in self.adj]

    def apply(self, u, w, inflow=None):
        lib = _load()
        u = np.ascontiguousarray(u, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        inflow = None if inflow is None else np.ascontiguousarray(inflow, dtype=np.float64)
        r = np.empty_like(w)
        if lib.port3_apply(*self._args(), _p(u), _p(w), _p(inflow), _p(r), self.threads) != 0:
            raise ValueError("port3_apply: order too large")
        return r

    def substeps(self, u, w, dt, nsteps, inflow=None):
        lib = _load()
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.array(w, dtype=np.float64, copy=True, order="C")
        inflow = None if inflow is None else np.ascontiguousarray(inflow, dtype=np.float64)
        work = np.empty_like(out)
        if lib.port3_substeps(*self._args(), _p(u), _p(out), _p(inflow), _p(self.minv), C.c_double(dt),
                              int(nsteps), _p(work), self.threads) != 0:
            raise ValueError("port3_substeps: order too large")
        return out
