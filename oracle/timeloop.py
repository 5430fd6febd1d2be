"""ORACLE — test infrastructure only.  CPU restatement of the explicit
convection time integration built on the apply (SPEC.md ``timeloop``):

* ``propagate`` — propagate_convection, SPEC:429-437 / PAPER:588-594:
  forward Euler or SSP-RK2 (Heun) substeps of  dv/ds = -(M^V)^{-1} C^V(u(s)) v,
  with u(s) frozen or linearly extrapolated from two stored fields
  ("extrapolation data u(s) built from stored divergence-free
  fields"; "linear two-point for BDF2").
* ``richardson`` — pseudo_time_solve, SPEC:456-464 / PAPER:671-687:
  explicit-Euler pseudo-time iteration for  v + tau (M^V)^{-1} C^V v = g,
      res_i = g - v_i - tau M^-1 C v_i,   v_{i+1} = v_i + ds res_i,
  stopped at the first i with ||res_i||_2 <= rho ||res_0||_2.
  PAPER.md:681 prints "+ tau (M^V)^{-1} C^V v_i" inside the bracket; that
  sign contradicts the pseudo-time ODE two lines above it (PAPER.md:678,
  d/ds v + v + tau C v = g) and the equation being solved, whose
  stationary point is the solution only with the minus sign, which is what
  is restated here.

Both are generic over ``apply(u, v) -> r`` (C^V(u; v) in V_h layout) and the
mass inverse ``minv``: a per-element diagonal (NT,), or a callable applying
the block-diagonal (M^V)^{-1} of a curved mesh, so the same
restatement checks the 2D, curved and 3D device paths.  Only tests/ may import this module.
"""
from __future__ import annotations

import numpy as np


def velocity_at(s, u_cur, u_prev=None, t_prev=0.0, t_cur=0.0):
    """u(s): frozen u_cur, or u_cur + (s - t_cur)/(t_cur - t_prev) (u_cur - u_prev)."""
    if u_prev is None:
        return u_cur
    th = (s - t_cur) / (t_cur - t_prev)
    return (1.0 + th) * u_cur - th * u_prev


def _mass_inv(minv):
    if callable(minv):
        return minv
    mi = np.asarray(minv, dtype=float)[:, None]
    return lambda r: mi * r


def propagate(apply, minv, u_cur, w0, ds, nsteps, scheme="euler", u_prev=None, t_prev=0.0, t_cur=0.0,
              t1=0.0):
    """nsteps substeps from pseudo time t1; scheme "euler" or "ssprk2" (Heun:
    v1 = v - ds M^-1 C(s) v, v' = (v + v1 - ds M^-1 C(s+ds) v1) / 2)."""
    mi = _mass_inv(minv)
    v = np.array(w0, dtype=float, copy=True)
    for i in range(nsteps):
        s0, s1 = t1 + i * ds, t1 + (i + 1) * ds
        v1 = v - ds * mi(apply(velocity_at(s0, u_cur, u_prev, t_prev, t_cur), v))
        if scheme == "euler":
            v = v1
            continue
        v2 = v1 - ds * mi(apply(velocity_at(s1, u_cur, u_prev, t_prev, t_cur), v1))
        v = 0.5 * v + 0.5 * v2
    return v


def richardson(apply, minv, u, g, tau, ds, rho=1e-3, max_iter=500, v0=None):
    """Returns (v, iterations, converged, res0, res)."""
    mi = _mass_inv(minv)
    v = np.zeros_like(g, dtype=float) if v0 is None else np.array(v0, dtype=float, copy=True)
    r0 = None
    for it in range(max_iter + 1):
        res = g - v - tau * mi(apply(u, v))
        rn = float(np.sqrt(np.sum(res * res)))
        if r0 is None:
            r0 = rn
        if rn <= rho * r0:
            return v, it, True, r0, rn
        if it == max_iter:
            return v, it, False, r0, rn
        v = v + ds * res
    raise AssertionError("unreachable")
