"""Field dumps and step logs consumed by adjacent tooling.

* ``dump_field`` — SPEC.md:240 "Field dump: element index, ref-point grid,
  value columns as CSV (for plotting)": one row per (element, reference
  lattice point), columns ``element,xi,eta,x,y,v0,v1``.  V_h fields (w, r)
  are evaluated as sum_m w[c*nbs+m] D_m(x_hat); W_h (BDM) fields by the
  contravariant Piola map u = J u_hat / detJ.
* ``max_divergence`` — max over elements and points of |div u| for an
  element-local BDM field, div u = div_hat u_hat / detJ (div BDM_k in P_{k-1}).
* ``StepLog`` — SPEC.md:490 "Step log (CSV): t, scheme, stage timings,
  Richardson iterations, max divergence".

Host-side I/O helpers (numpy); they are not on the device hot path.
"""

from __future__ import annotations

import csv
import io
import os

import numpy as np

from . import basis as B

__all__ = ["reference_lattice", "dump_field", "max_divergence", "StepLog"]


def reference_lattice(n: int) -> np.ndarray:
    """Points (i/n, j/n), i + j <= n, of the reference triangle, row-major in j then i."""
    return np.array([(i / n, j / n) for j in range(n + 1) for i in range(n + 1 - j)], dtype=float)


def _values(mesh, k: int, coeffs: np.ndarray, kind: str, pts: np.ndarray) -> np.ndarray:
    """(NT, npts, 2) values of an element-local field at reference points."""
    if kind == "VectorDG":
        D = B.dubiner_values(k, pts)                         # (np, nbs)
        nbs = D.shape[1]
        return np.stack([coeffs[:, :nbs] @ D.T, coeffs[:, nbs:] @ D.T], axis=-1)
    if kind == "Hdiv":
        phi = B.build_bdm_basis(k).values(pts)                # (np, nb, 2)
        uh = np.einsum("tj,pjd->tpd", coeffs, phi)
        J = mesh.affine_jac
        det = mesh.affine_det
        return np.einsum("tcd,tpd->tpc", J, uh) / det[:, None, None]
    raise ValueError("kind must be 'VectorDG' or 'Hdiv'")


def dump_field(path_or_buf, mesh, k: int, coeffs, kind: str = "VectorDG", n: int = None) -> None:
    """Write the CSV field dump to a path or text buffer."""
    coeffs = np.asarray(coeffs.detach().cpu().numpy() if hasattr(coeffs, "detach") else coeffs, dtype=float)
    n = n or max(1, k)
    pts = reference_lattice(n)
    vals = _values(mesh, k, coeffs, kind, pts)
    X = mesh.affine_origin[:, None, :] + np.einsum("tcd,pd->tpc", mesh.affine_jac, pts)
    NT, P = vals.shape[:2]
    table = np.column_stack([np.repeat(np.arange(NT), P), np.tile(pts, (NT, 1)), X.reshape(-1, 2),
                             vals.reshape(-1, 2)])
    own = isinstance(path_or_buf, (str, os.PathLike))
    fh = open(path_or_buf, "w", newline="") if own else path_or_buf
    try:
        fh.write("element,xi,eta,x,y,v0,v1\n")
        for row in table:
            fh.write(f"{int(row[0])}," + ",".join(f"{v:.17g}" for v in row[1:]) + "\n")
    finally:
        if own:
            fh.close()


def max_divergence(mesh, k: int, u_loc) -> float:
    """max |div u| over elements x quad_triangle(2k) points of a BDM_k field."""
    u = np.asarray(u_loc.detach().cpu().numpy() if hasattr(u_loc, "detach") else u_loc, dtype=float)
    q = B.quad_triangle(2 * k)
    div_hat = B.build_bdm_basis(k).divergence(q.points)      # (np, nb)
    d = (u @ div_hat.T) / mesh.affine_det[:, None]
    return float(np.abs(d).max()) if d.size else 0.0


class StepLog:
    """CSV step log: t, scheme, stage timings (ms, ';'-joined),
    Richardson iterations, max divergence.  ``path=None`` keeps it in memory."""

    HEADER = ("t", "scheme", "stage_ms", "richardson_iterations", "max_divergence")

    def __init__(self, path=None):
        self.path = path
        self.rows = []

    def log(self, t: float, scheme: str, stage_ms=(), richardson_iterations: int = 0,
            max_divergence: float = float("nan")) -> None:
        self.rows.append((float(t), str(scheme), ";".join(f"{x:.6g}" for x in stage_ms),
                          int(richardson_iterations), float(max_divergence)))
        if self.path is not None:
            new = not os.path.exists(self.path)
            with open(self.path, "a", newline="") as fh:
                w = csv.writer(fh)
                if new:
                    w.writerow(self.HEADER)
                w.writerow(self.rows[-1])

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf)
        w.writerow(self.HEADER)
        w.writerows(self.rows)
        return buf.getvalue()
