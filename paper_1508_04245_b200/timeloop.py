"""Explicit convection substeps (mirrors ``timeloop`` in SPEC.md:396-496).

* ``cfl_substep(u_max, h_min, k, safety)`` — SPEC.md:438-446, with the
  BASELINE rule dt = safety * h / (k^2 u_max), safety 0.1.
* ``propagate_convection(v0, t1, t2, u_conv, data)`` — SPEC.md:429-437,
  PAPER.md:588-594: integrates dv/ds + (M^V)^{-1} C^V(u) v = 0 over
  [t1, t2] with frozen u.  BASELINE replaces the SPEC's SSP-RK2 by forward
  Euler, which is what the device loop (hdgc_substeps) implements; the whole
  loop runs on the device, one fused apply+update kernel per substep.
"""

from __future__ import annotations

import math

from .forms import ConvectionData, FEField, operator_for

__all__ = ["cfl_substep", "propagate_convection"]


def cfl_substep(u_max: float, h_min: float, k: int, safety: float = 0.1, interval: float = math.inf) -> float:
    """Substep size (SPEC.md:438-446 with the BASELINE k^2 rule)."""
    if u_max <= 0.0:
        return interval
    return safety * h_min / (k * k * u_max)


def propagate_convection(v0, t1: float, t2: float, u_conv: FEField, data: ConvectionData = None,
                         dt: float = None, safety: float = 0.1):
    """Q^{t1->t2} v0 by nsub = ceil((t2-t1)/dt) forward-Euler substeps.

    Returns (v, nsub, dt_used).  ``dt`` defaults to the CFL rule with max|u|
    measured on the device; the last substep is shortened so the loop ends
    exactly at t2 (each substep size is uniform: (t2-t1)/nsub)."""
    sp = u_conv.space
    op = operator_for(sp.mesh, sp.k)
    span = float(t2 - t1)
    if span <= 0.0:
        return v0, 0, 0.0
    if dt is None:
        dt = cfl_substep(op.max_speed(u_conv.coeffs), sp.mesh.h_min(), sp.k, safety, span)
    nsub = max(1, math.ceil(span / dt - 1e-12))
    ds = span / nsub
    inflow = None if data is None else data.inflow
    v = op.substeps(u_conv.coeffs, v0, ds, nsub, inflow)
    return v, nsub, ds
