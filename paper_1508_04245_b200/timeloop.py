"""Explicit convection time integration (mirrors ``timeloop`` in SPEC.md:396-496).

* ``cfl_substep(u_max, h_min, k, safety)`` — SPEC.md:438-446:
  ds = safety * h_min / ((2k+1) u_max).  (BASELINE cfg2's benchmark rule
  dt = 0.1 h / (k^2 u_max) is ``fields.cfl_dt``; bench.py passes it explicitly.)
* ``propagate_convection(v0, t1, t2, u_conv, data, scheme, u_prev, ...)`` —
  SPEC.md:429-437: integrates dv/ds + (M^V)^{-1} C^V(u(s)) v = 0
  over [t1, t2].  scheme "ssprk2" (the SPEC's SSP-RK2, the default) or "euler"
  (BASELINE cfg2's forward Euler); u frozen, or linearly extrapolated from a
  previous field (u_prev at t_prev, u_conv at t_cur).  The whole loop runs on
  the device (hdgc_propagate / hdgc_substeps): one fused apply+update kernel
  per stage, the frozen-velocity prep redone only when u(s) changes.
* ``pseudo_time_solve(g, tau, u_conv, data, ...)`` — SPEC.md:456-464,
  PAPER.md:671-687: Richardson iteration for v + tau (M^V)^{-1} C^V v = g
  (hdgc_richardson: fused residual + update kernel and a deterministic norm).
"""

from __future__ import annotations

import math

from .forms import ConvectionData, FEField, operator_for

__all__ = ["cfl_substep", "propagate_convection", "pseudo_time_solve", "richardson_ds"]


def cfl_substep(u_max: float, h_min: float, k: int, safety: float = 0.1, interval: float = math.inf) -> float:
    """Substep size ds = safety * h_min / ((2k+1) u_max);
    u_max <= 0 returns the requested interval."""
    if u_max <= 0.0:
        return interval
    return safety * h_min / ((2 * k + 1) * u_max)


def propagate_convection(v0, t1: float, t2: float, u_conv: FEField, data: ConvectionData = None,
                         dt: float = None, safety: float = 0.1, scheme: str = "ssprk2",
                         u_prev: FEField = None, t_prev: float = None, t_cur: float = None,
                         guard: bool = True):
    """Q^{t1->t2} v0 by nsub = ceil((t2-t1)/dt) explicit substeps.

    ``guard``: after the loop, synchronise and raise
    ``NormBlowupError`` if any substep produced non-finite values.

    Returns (v, nsub, ds_used).  ``dt`` defaults to the CFL rule with max|u|
    measured on the device (max over u_prev and u_conv when extrapolating);
    the substep size is uniform, (t2-t1)/nsub, so the loop ends exactly at t2.
    With ``u_prev`` the convecting velocity is the linear extrapolation
    u(s) = u_conv + (s - t_cur)/(t_cur - t_prev) (u_conv - u_prev)."""
    sp = u_conv.space
    op = operator_for(sp.mesh, sp.k)
    span = float(t2 - t1)
    if span <= 0.0:
        return v0, 0, 0.0
    if dt is None:
        umax = op.max_speed(u_conv.coeffs)
        if u_prev is not None:
            umax = max(umax, op.max_speed(u_prev.coeffs))
        dt = cfl_substep(umax, sp.mesh.h_min(), sp.k, safety, span)
    nsub = max(1, math.ceil(span / dt - 1e-12))
    ds = span / nsub
    inflow = None if data is None else data.inflow
    if scheme == "euler" and u_prev is None:
        v = op.substeps(u_conv.coeffs, v0, ds, nsub, inflow)
    else:
        if u_prev is not None and (t_prev is None or t_cur is None):
            raise ValueError("extrapolation needs t_prev and t_cur")
        v = op.propagate(u_conv.coeffs, v0, ds, nsub, inflow, scheme,
                         None if u_prev is None else u_prev.coeffs,
                         0.0 if t_prev is None else t_prev, 0.0 if t_cur is None else t_cur, t1)
    if guard:
        op.check_finite()
    return v, nsub, ds


def richardson_ds(tau: float, u_max: float, h_min: float, k: int, safety: float = 0.1) -> float:
    """Pseudo-time step for the Richardson iteration: the explicit-Euler CFL of
    the operator Id + tau (M^V)^{-1} C^V, ds = 1 / (1 + tau / dt_c) with dt_c the
    convection substep (cfl_substep): ds = 1 for tau = 0 (one exact step),
    tau ds -> dt_c for large tau (SPEC.md DESIGN DECISIONS, Richardson defaults)."""
    dt_c = cfl_substep(u_max, h_min, k, safety)
    if not math.isfinite(dt_c):
        return 1.0
    return 1.0 / (1.0 + tau / dt_c)


def pseudo_time_solve(g, tau: float, u_conv: FEField, data: ConvectionData = None, rho: float = 1e-3,
                      max_iter: int = 500, ds: float = None, v0=None, safety: float = 0.1):
    """Solve v + tau (M^V)^{-1} C^V(u) v = g by the Richardson / pseudo-time
    iteration until ||res|| <= rho ||res_0||.

    Returns (v, iterations, converged).  v0 defaults to zero; non-convergence
    within max_iter is flagged (converged False), not raised."""
    sp = u_conv.space
    op = operator_for(sp.mesh, sp.k)
    if ds is None:
        ds = richardson_ds(tau, op.max_speed(u_conv.coeffs), sp.mesh.h_min(), sp.k, safety)
    if v0 is None:
        import numpy as np
        torch = None
        try:
            import torch
        except Exception:  # pragma: no cover
            pass
        if torch is not None and isinstance(g, torch.Tensor):
            v0 = torch.zeros_like(g)
        else:
            v0 = np.zeros_like(np.asarray(g, dtype=np.float64))
    inflow = None if data is None else data.inflow
    v, it, conv, _, _ = op.richardson(u_conv.coeffs, g, v0, tau, ds, rho, max_iter, inflow)
    return v, it, conv
