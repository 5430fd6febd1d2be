"""Generate 3D (tetrahedra, BASELINE cfg5 shape) regression fixtures.

The reference has no 3D code, so these are outputs of
the 3D oracle restatement (oracle/convection3d.py) on this package's 3D
basis (itself checked by tests/test_basis3d.py): the textbook form in
physical coordinates and the long-double flux-difference form.  Run:

    python tests/golden/make_golden3d.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import convection3d as O3                      # noqa: E402
from paper_1508_04245_b200 import fields3d as F3           # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3             # noqa: E402


def case(name, n, k, modes, seed, nsub=0, wind=(0.0, 0.0, 0.0)):
    m = M3.generate_cube(n)
    vp = F3.VectorPotential(modes, seed, wind)
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    rng = np.random.default_rng(100 + k)
    nf = O3._provider(None).face_rule(k).weights.size
    # a uniform wind makes part of the cube boundary an inflow boundary; the
    # exterior state is random so the inflow branch is exercised
    inflow = rng.standard_normal((m.boundary_facets.size, nf, 3))
    wr = rng.standard_normal(w.shape)
    rec = dict(k=np.array(k), n=np.array(n), u=u, w=w, w_rand=wr, inflow=inflow,
               r=O3.apply_convection3(m, k, u, w, inflow),
               r_ld=O3.apply_convection3_flux_form(m, k, u, w, inflow).astype(np.float64),
               r_rand=O3.apply_convection3(m, k, u, wr, inflow),
               r_rand_ld=O3.apply_convection3_flux_form(m, k, u, wr, inflow).astype(np.float64))
    if nsub:
        dt = 0.1 * m.h_min() / (k * k * F3.max_speed3_host(m, k, u))
        rec["dt"] = np.array(dt)
        rec["nsub"] = np.array(nsub)
        rec["w_sub_ld"] = O3.substeps3(m, k, u, w, dt, nsub, inflow)
    np.savez_compressed(os.path.join(HERE, f"conv3d_{name}.npz"), **rec)
    print(name, m.n_elements, float(np.abs(rec["r"]).max()))


if __name__ == "__main__":
    case("k1", 3, 1, 3, 11)
    case("k2", 3, 2, 3, 12, wind=(1.0, 0.3, 0.2))
    case("k3", 3, 3, 4, 13, nsub=10, wind=(1.0, -0.4, 0.3))
    case("k4", 2, 4, 2, 14, wind=(0.2, 0.5, -1.0))
