"""Golden fixtures for CURVED meshes FROM THE REFERENCE:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_curved.py

* ring meshes from the reference's own ``generate_ring`` + ``curve_boundary``
  (MESH:381-443, 555-615) at geometry orders g = 2, 3: mesh arrays, the
  curved maps (element ids + monomial coefficients), ``geometry_map`` at a
  few reference points of every curved element (MESH:254-278) and the
  reference's ``total_area``;
* the curved-mesh oracle (``oracle/curved.py``) evaluated ON the reference's
  mesh object and ``hdgflow.polybasis`` (the reference has no convection
  apply): r = C^V(u; w) with inflow, 5 forward-Euler substeps with
  the block-diagonal V_h mass, I u (element L2 projection) and I^T r.
  Inputs u / w / inflow are synthesised by this package on the reference mesh
  and stored bit-exactly.

Writes tests/golden/curved.npz.  /root/reference does not travel to the GPU
box; the fixture does.
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

from oracle import curved as OC              # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402  (input synthesis only)
from paper_1508_04245_b200 import mesh as M    # noqa: E402

CIRCLE = ((0.5, 0.5), 0.15)
RING = dict(rect=(0.0, 0.0, 1.0, 1.0), n_theta=16, n_layers=3)
PTS = np.array([[0.2, 0.3], [0.5, 0.25], [0.1, 0.8], [1.0 / 3.0, 1.0 / 3.0]])


def ring_ref(g):
    c = rmesh.Circle(*CIRCLE)
    m = rmesh.generate_ring(c, RING["rect"], RING["n_theta"], RING["n_layers"])
    return rmesh.curve_boundary(m, "obstacle", c, g)


def ring_ours(g):
    c = M.Circle(*CIRCLE)
    m = M.generate_ring(c, RING["rect"], RING["n_theta"], RING["n_layers"])
    return M.curve_boundary(m, "obstacle", c, g)


def main():
    out = {}
    for g in (2, 3):
        m = ring_ref(g)
        for a in ("vertices", "triangles", "facet_vertices", "facet_elems", "facet_local", "facet_flip"):
            out[f"g{g}_{a}"] = np.asarray(getattr(m, a))
        ce = np.array(sorted(m.curved_maps), dtype=np.int64)
        out[f"g{g}_curved_elems"] = ce
        out[f"g{g}_curved_coeffs"] = np.stack([m.curved_maps[e] for e in ce])
        xs, Js, ds = zip(*(m.geometry_map(int(e), PTS) for e in ce))
        out[f"g{g}_geo_x"], out[f"g{g}_geo_J"], out[f"g{g}_geo_det"] = np.array(xs), np.array(Js), np.array(ds)
        out[f"g{g}_total_area"] = np.array(m.total_area())
        out[f"g{g}_labels_f"] = np.array(sorted(m.facet_labels), dtype=np.int64)
        out[f"g{g}_labels_n"] = np.array([m.facet_labels[f] for f in sorted(m.facet_labels)])
    out["pts"] = PTS
    # operator on the reference's g=3 ring mesh and polybasis, k = 3
    m = ring_ref(3)
    ours = ring_ours(3)
    assert np.array_equal(ours.triangles, m.triangles) and np.allclose(ours.vertices, m.vertices, 0, 0)
    k = 3
    sf = F.StreamFunction(4, 5, (1.0, 0.3))
    u = F.interpolate_curl(ours, k, sf)
    w = OC.transfer_I(m, k, u, basis=rpb)
    inflow = F.inflow_values(ours, k, sf)
    r = OC.apply_convection(m, k, u, w, inflow, basis=rpb)
    dt = 2e-4
    out.update(k=np.array(k), u=u, w=w, inflow=inflow, r=r, dt=np.array(dt), nsub=np.array(5),
               w_sub=OC.substeps(m, k, u, w, dt, 5, inflow, basis=rpb),
               r_w=OC.transfer_IT(m, k, r, basis=rpb))
    np.savez_compressed(os.path.join(HERE, "curved.npz"), **out)
    print("curved.npz:", {kk: v.shape for kk, v in out.items() if kk.startswith("g3_") or kk in ("u", "r")})


if __name__ == "__main__":
    main()
