"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE.

Run in the build container, where the read-only reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything table- or mesh-shaped comes from the reference's own modules
(``hdgflow.polybasis`` PB:47-378, ``hdgflow.mesh2d`` MESH:86-378), imported
unchanged.  The operator outputs come from the oracle restatement
(``oracle/convection.py``) evaluated ON the reference's basis and mesh
objects, because the reference has no convection apply of its own
(SURVEY §0 fact 1).  Inputs (u, w, inflow) are stored bit-exactly so the GPU
tests never regenerate them.

The fixtures travel to the GPU box with the repo; /root/reference does not.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from hdgflow import mesh2d as rmesh          # noqa: E402  (reference)
from hdgflow import polybasis as rpb         # noqa: E402  (reference)

from oracle import convection as O          # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402  (input synthesis only)


def tables():
    out = {}
    for d in range(0, 26):
        qi = rpb.quad_interval(d)
        qt = rpb.quad_triangle(d)
        out[f"qi{d}_p"], out[f"qi{d}_w"] = qi.points, qi.weights
        out[f"qt{d}_p"], out[f"qt{d}_w"] = qt.points, qt.weights
    rng = np.random.default_rng(1508)
    pts = rng.random((40, 2))
    pts = pts[pts.sum(1) < 1.0][:24]
    out["rand_pts"] = pts
    t = np.linspace(0.0, 1.0, 11)
    out["leg_t"] = t
    out["leg_v"] = rpb.legendre_values(10, t)
    out["leg_d"] = rpb.legendre_derivs(10, t)
    for k in range(1, 9):
        q = rpb.quad_triangle(3 * k + 1)
        v, g = rpb.dubiner_values(k, np.vstack([q.points, pts]), with_grads=True)
        out[f"dub{k}_v"], out[f"dub{k}_g"] = v, g
        b = rpb.build_bdm_basis(k)
        out[f"bdm{k}_coef"], out[f"bdm{k}_V"] = b.coef, b.vandermonde
        out[f"bdm{k}_cond"] = np.array(b.cond)
        out[f"bdm{k}_vals"] = b.values(pts)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def _mesh_arrays(m, prefix, out):
    for a in ("vertices", "triangles", "facet_vertices", "facet_elems", "facet_local",
              "facet_flip", "elem_facets", "affine_det"):
        out[f"{prefix}_{a}"] = getattr(m, a)


def meshes():
    out = {}
    m = rmesh.generate_structured((0.0, 0.0, 2.0, 1.0), 6, 5)
    _mesh_arrays(m, "rect", out)
    # jittered 12x12 through Mesh.build (cfg3 construction, small)
    base = rmesh.generate_structured((0.0, 0.0, 1.0, 1.0), 12, 12)
    rng = np.random.default_rng(77)
    v = base.vertices.copy()
    inner = (v[:, 0] > 0) & (v[:, 0] < 1) & (v[:, 1] > 0) & (v[:, 1] < 1)
    v[inner] += rng.uniform(-0.2 / 12, 0.2 / 12, size=v.shape)[inner]
    mj = rmesh.Mesh.build(v, base.triangles, {tuple(base.facet_vertices[f]): lab
                                              for f, lab in base.facet_labels.items()})
    _mesh_arrays(mj, "jit", out)
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **out)
    return m, mj


def conv_case(name, mesh, k, sf, with_inflow, nsub=0, dt=None):
    u = F.interpolate_curl(mesh, k, sf)
    w = O.transfer_I(mesh, k, u, basis=rpb)
    inflow = F.inflow_values(mesh, k, sf) if with_inflow else None
    r = O.apply_convection(mesh, k, u, w, inflow, basis=rpb)
    rng = np.random.default_rng(k)
    wr = rng.standard_normal(w.shape)
    rr = O.apply_convection(mesh, k, u, wr, inflow, basis=rpb)
    # extended-precision flux-difference form on the same reference tables: the
    # accuracy anchor (the textbook form above loses digits to cancellation)
    r_ld = O.apply_convection_flux_form(mesh, k, u, w, inflow, basis=rpb).astype(np.float64)
    rr_ld = O.apply_convection_flux_form(mesh, k, u, wr, inflow, basis=rpb).astype(np.float64)
    rec = dict(k=np.array(k), u=u, w=w, r=r, w_rand=wr, r_rand=rr, r_ld=r_ld, r_rand_ld=rr_ld,
               r_w=O.transfer_IT(mesh, k, r, basis=rpb),
               vertices=mesh.vertices, triangles=mesh.triangles,
               facet_vertices=mesh.facet_vertices, facet_elems=mesh.facet_elems,
               facet_local=mesh.facet_local, facet_flip=mesh.facet_flip)
    if inflow is not None:
        rec["inflow"] = inflow
    if nsub:
        rec["dt"] = np.array(dt)
        rec["nsub"] = np.array(nsub)
        rec["w_sub"] = O.substeps(mesh, k, u, w, dt, nsub, inflow, basis=rpb)
        wl = w.astype(np.longdouble)
        minv = 2.0 / mesh.affine_det.astype(np.longdouble)
        for _ in range(nsub):
            wl = wl - dt * minv[:, None] * O.apply_convection_flux_form(mesh, k, u, wl, inflow, basis=rpb)
        rec["w_sub_ld"] = wl.astype(np.float64)
    np.savez_compressed(os.path.join(HERE, f"conv_{name}.npz"), **rec)
    print(name, "k", k, "NT", mesh.n_elements, "|r|", float(np.abs(r).max()))


def main():
    tables()
    rect, jit = meshes()
    # cfg1 exactly: 32x32 unit square, k=2, modes<=4
    cfg1 = rmesh.generate_structured((0.0, 0.0, 1.0, 1.0), 32, 32)
    conv_case("cfg1", cfg1, 2, F.StreamFunction(4, 1), with_inflow=False)
    # order sweep on a small structured mesh, modes<=4 (cfg4 shape, small)
    small = rmesh.generate_structured((0.0, 0.0, 1.0, 1.0), 6, 6)
    for k in range(1, 9):
        conv_case(f"sweep_k{k}", small, k, F.StreamFunction(4, 4), with_inflow=True)
    # jittered + wind + inflow (cfg3 shape, small), with a substep run
    sfw = F.StreamFunction(4, 3, (1.0, 0.3))
    for k in (3, 6):
        conv_case(f"jit_k{k}", jit, k, sfw, with_inflow=True, nsub=10,
                  dt=0.1 * jit.h_min() / (k * k * 12.0))
    # k=4 substeps on a structured mesh (cfg2 shape, small)
    conv_case("sub_k4", rmesh.generate_structured((0.0, 0.0, 1.0, 1.0), 10, 10), 4,
              F.StreamFunction(6, 2), with_inflow=True, nsub=20, dt=2e-4)


if __name__ == "__main__":
    main()
