/*
 * ORACLE — test infrastructure only (never linked into the product).
 *
 * Plain-C OpenMP restatement of the 3D (tetrahedral) convection apply, the
 * fast full-size checker for BASELINE cfg5 (196,608 tets, BDM_3, 20
 * substeps): the numpy/long-double oracle (oracle/convection3d.py) needs
 * minutes per apply at that size, this port ~0.3 s on 16 cores.
 *
 * It restates oracle/convection3d.py::apply_convection3_flux_form (same
 * algorithm, fp64, element-owned), which tests/test_oracle3d_port.py checks
 * against both that long-double flux form and the physical-coordinate
 * textbook form apply_convection3 on small meshes.  Operator: the upwind-DG
 * trilinear form of PAPER.md:424-436 / SPEC.md:299-307 on tets, in the
 * geometry-free flux-difference form:
 *   r = sign(detJ) [ sum_p w_p (u_hat . grad_hat w_c + w_c div_hat u_hat) D_m
 *                  + sum_faces sum_{q: sign(detJ) F_q < 0} w_q F_q (w_ext - w_own)_c D_m ],
 *   F_q = 2|f| * 2 sum_n u[f*nfd + n] D2_n(q)   (u_hat . n_hat dS_hat from the face dofs),
 * with direct (not sum-factorised) quadrature: volume rule quad_tet(3k+1),
 * face rule quad_triangle(3k+1); neighbours share face point q (every tet's
 * vertex ids sorted, mesh3d.py).
 *
 * Layouts: u, w, r (NT, nb) row-major, nb = 3 nbs, w index c*nbs+m; tables:
 * coef (nb, nb), vw (nqv), vD (nqv, nbs), vG (nqv, nbs, 3), fw (nf),
 * D2 (nf, nfd), fD (4, nf, nbs), farea (4); per element sign (NT);
 * neighbours nbr (NT, 4) element or -1, nbf (NT, 4) neighbour face,
 * bslot (NT, 4) boundary-face row or -1; inflow (NBF, nf, 3) or NULL.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int k, nt, nqv, nf;
  const double *coef, *vw, *vD, *vG, *fw, *D2, *fD, *farea, *sgn;
  const int32_t *nbr, *nbf, *bslot;
} port3_mesh;

enum { MAXNB = 3 * 35, MAXNF = 64 };

static void apply3_elem(const port3_mesh* m, int T, const double* u, const double* w, const double* inflow,
                        double* r) {
  const int k = m->k, nbs = (k + 1) * (k + 2) * (k + 3) / 6, nb = 3 * nbs, nfd = (k + 1) * (k + 2) / 2;
  const int nqv = m->nqv, nf = m->nf;
  const double* ut = u + (size_t)T * nb;
  const double* wt = w + (size_t)T * nb;
  double uh[MAXNB];
  for (int i = 0; i < nb; ++i) {
    double a = 0.0;
    for (int j = 0; j < nb; ++j) a += m->coef[i * nb + j] * ut[j];
    uh[i] = a;
  }
  for (int j = 0; j < nb; ++j) r[j] = 0.0;
  /* volume: r[c,m] += sum_p w_p (u_hat . grad w_c + w_c div u_hat)(p) D_m(p) */
  for (int p = 0; p < nqv; ++p) {
    const double* D = m->vD + (size_t)p * nbs;
    const double* G = m->vG + (size_t)p * nbs * 3;
    double up[3] = {0, 0, 0}, div = 0.0, wp[3] = {0, 0, 0}, gw[3][3] = {{0}};
    for (int i = 0; i < nbs; ++i) {
      for (int d = 0; d < 3; ++d) {
        up[d] += uh[d * nbs + i] * D[i];
        div += uh[d * nbs + i] * G[3 * i + d];
      }
      for (int c = 0; c < 3; ++c) {
        const double wc = wt[c * nbs + i];
        wp[c] += wc * D[i];
        for (int d = 0; d < 3; ++d) gw[c][d] += wc * G[3 * i + d];
      }
    }
    for (int c = 0; c < 3; ++c) {
      const double f = m->vw[p] * (up[0] * gw[c][0] + up[1] * gw[c][1] + up[2] * gw[c][2] + wp[c] * div);
      for (int i = 0; i < nbs; ++i) r[c * nbs + i] += f * D[i];
    }
  }
  /* faces: upwind per point on sign(detJ) F; only inflow
   * points contribute F (w_ext - w_own) in the flux-difference form */
  const double sg = m->sgn[T];
  for (int f = 0; f < 4; ++f) {
    const int nT = m->nbr[T * 4 + f], nF = m->nbf[T * 4 + f], slot = m->bslot[T * 4 + f];
    const double* wn = nT >= 0 ? w + (size_t)nT * nb : NULL;
    if (!wn && !(inflow && slot >= 0)) continue;      /* exterior value = own trace: no jump */
    for (int q = 0; q < nf; ++q) {
      double F = 0.0;
      for (int n = 0; n < nfd; ++n) F += ut[f * nfd + n] * m->D2[q * nfd + n];
      F *= 2.0 * m->farea[f] * 2.0;
      if (!(sg * F < 0.0)) continue;
      const double* De = m->fD + ((size_t)f * nf + q) * nbs;
      double own[3] = {0, 0, 0}, ext[3] = {0, 0, 0};
      for (int i = 0; i < nbs; ++i)
        for (int c = 0; c < 3; ++c) own[c] += wt[c * nbs + i] * De[i];
      if (wn) {
        const double* Dn = m->fD + ((size_t)nF * nf + q) * nbs;   /* same point q: sorted vertices */
        for (int i = 0; i < nbs; ++i)
          for (int c = 0; c < 3; ++c) ext[c] += wn[c * nbs + i] * Dn[i];
      } else {
        for (int c = 0; c < 3; ++c) ext[c] = inflow[((size_t)slot * nf + q) * 3 + c];
      }
      const double s = m->fw[q] * F;
      for (int c = 0; c < 3; ++c) {
        const double j = s * (ext[c] - own[c]);
        for (int i = 0; i < nbs; ++i) r[c * nbs + i] += j * De[i];
      }
    }
  }
  for (int j = 0; j < nb; ++j) r[j] *= sg;
}

#define PORT3_ARGS                                                                                             \
  int k, int nt, int nqv, int nf, const double *coef, const double *vw, const double *vD, const double *vG,    \
      const double *fw, const double *D2, const double *fD, const double *farea, const double *sgn,           \
      const int32_t *nbr, const int32_t *nbf, const int32_t *bslot
#define PORT3_INIT \
  port3_mesh m = {k, nt, nqv, nf, coef, vw, vD, vG, fw, D2, fD, farea, sgn, nbr, nbf, bslot}

int port3_apply(PORT3_ARGS, const double* u, const double* w, const double* inflow, double* r, int nthreads) {
  PORT3_INIT;
  const int nb = (k + 1) * (k + 2) * (k + 3) / 2;
  if (nb > MAXNB || nf > MAXNF) return -1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int T = 0; T < nt; ++T) apply3_elem(&m, T, u, w, inflow, r + (size_t)T * nb);
  return 0;
}

/* forward Euler: w <- w - dt * minv * C(u; w), nsteps times */
int port3_substeps(PORT3_ARGS, const double* u, double* w, const double* inflow, const double* minv, double dt,
                   int nsteps, double* work, int nthreads) {
  PORT3_INIT;
  const int nb = (k + 1) * (k + 2) * (k + 3) / 2;
  if (nb > MAXNB || nf > MAXNF) return -1;
  double* a = w;
  double* b = work;
  for (int s = 0; s < nsteps; ++s) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int T = 0; T < nt; ++T) {
      double r[MAXNB];
      apply3_elem(&m, T, u, a, inflow, r);
      const double sc = dt * minv[T];
      for (int j = 0; j < nb; ++j) b[(size_t)T * nb + j] = a[(size_t)T * nb + j] - sc * r[j];
    }
    double* t = a; a = b; b = t;
  }
  if (a != w) memcpy(w, a, sizeof(double) * (size_t)nt * nb);
  return 0;
}
