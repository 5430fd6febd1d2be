/*
 * ORACLE — test infrastructure only (never linked into the product).
 *
 * Plain-C OpenMP restatement of the reference convection apply, used
 *  (1) as the fast checker at BASELINE's full sizes (100 substeps at 131k
 *      triangles would take the numpy oracle ~7 minutes), and
 *  (2) as the CPU baseline ("port") that bench.py times on the GPU box's
 *      host cores (the reference itself has no implementation of this path,
 *      SURVEY.md §0 fact 1).
 *
 * Algorithm: the upwind-DG trilinear form of PAPER.md:424-436 /
 * SPEC.md:299-307 in the geometry-free reference form that holds on affine
 * elements, element-owned (each interior facet
 * evaluated from both sides; SPEC.md:326 visits it once — identical values up
 * to summation order), written in the flux-difference form
 *   r = int (u.grad w + w div u) z + sum_{inflow pts} F (w_ext - w_own) z,
 * which equals the textbook form exactly (divergence theorem with exact
 * quadrature) but keeps ~15 digits where the textbook form cancels two large
 * terms (tests/test_oracle.py measures both against a
 * long-double evaluation).  The physical-coordinate, facet-wise restatement in
 * oracle/convection.py checks this file on small meshes (tests/test_oracle.py).
 *
 * Layouts: u, w, r (NT, nb) row-major; tables as produced by
 * the basis provider: coef (nb, nb), divm (nbs(k-1), nb), vw (nqv), vD (nqv, nbs), vG (nqv, nbs, 2),
 * fw (nf), fL (nf, k+1), fD (3, nf, nbs), flen (3).  Neighbours: nbr (NT, 3)
 * element or -1, nbr_edge (NT, 3), bslot (NT, 3) boundary-facet row or -1.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int k, nt, nqv, nf;
  const double *coef, *divm, *vw, *vD, *vG, *fw, *fL, *fD, *flen;
  const int32_t *nbr, *nbr_edge, *bslot;
} port_mesh;

static void apply_elem(const port_mesh* m, int T, const double* u, const double* w,
                       const double* inflow, double* r, double* scratch) {
  const int k = m->k, nbs = (k + 1) * (k + 2) / 2, nb = 2 * nbs, ne = k + 1;
  const int nqv = m->nqv, nf = m->nf;
  double* uh = scratch;  /* nb */
  const double* ut = u + (size_t)T * nb;
  const double* wt = w + (size_t)T * nb;
  for (int i = 0; i < nb; ++i) {
    double a = 0.0;
    for (int j = 0; j < nb; ++j) a += m->coef[i * nb + j] * ut[j];
    uh[i] = a;
  }
  /* modal divergence of u_hat (P_{k-1} Dubiner coefficients) */
  const int nbs1 = k * (k + 1) / 2;
  double dv[64];
  for (int i = 0; i < nbs1; ++i) {
    double a = 0.0;
    for (int j = 0; j < nb; ++j) a += m->divm[i * nb + j] * ut[j];
    dv[i] = a;
  }
  for (int j = 0; j < nb; ++j) r[j] = 0.0;
  /* volume, flux-difference form: r[c,m] += sum_p wp (u.grad w_c + w_c div u)(p) D_m(p)
   * == -int w (x) u : grad z + int_dT (u.n) w_own z  (divergence theorem, exact rules) */
  for (int q = 0; q < nqv; ++q) {
    const double* D = m->vD + (size_t)q * nbs;
    const double* G = m->vG + (size_t)q * nbs * 2;
    double w0 = 0, w1 = 0, u0 = 0, u1 = 0, dq = 0, w0x = 0, w0y = 0, w1x = 0, w1y = 0;
    for (int i = 0; i < nbs; ++i) {
      w0 += wt[i] * D[i];
      w1 += wt[nbs + i] * D[i];
      u0 += uh[i] * D[i];
      u1 += uh[nbs + i] * D[i];
      w0x += wt[i] * G[2 * i];
      w0y += wt[i] * G[2 * i + 1];
      w1x += wt[nbs + i] * G[2 * i];
      w1y += wt[nbs + i] * G[2 * i + 1];
      if (i < nbs1) dq += dv[i] * D[i];
    }
    const double wp = m->vw[q];
    const double f0 = wp * (u0 * w0x + u1 * w0y + w0 * dq);
    const double f1 = wp * (u0 * w1x + u1 * w1y + w1 * dq);
    for (int i = 0; i < nbs; ++i) {
      r[i] += f0 * D[i];
      r[nbs + i] += f1 * D[i];
    }
  }
  /* facets: upwind on sign(u.n) per point; in the flux-difference
   * form only inflow points (F < 0) contribute F (w_ext - w_own) */
  for (int e = 0; e < 3; ++e) {
    const int nbT = m->nbr[T * 3 + e];
    const int e2 = m->nbr_edge[T * 3 + e];
    const int slot = m->bslot[T * 3 + e];
    const double* wn = nbT >= 0 ? w + (size_t)nbT * nb : NULL;
    if (!wn && !(inflow && slot >= 0)) continue;  /* exterior value = own trace */
    for (int q = 0; q < nf; ++q) {
      double F = 0.0;
      for (int l = 0; l < ne; ++l) F += ut[e * ne + l] * m->fL[q * ne + l];
      F *= m->flen[e];
      if (!(F < 0.0)) continue;
      const double* De = m->fD + ((size_t)e * nf + q) * nbs;
      double o0 = 0, o1 = 0, h0 = 0, h1 = 0;
      for (int i = 0; i < nbs; ++i) {
        o0 += wt[i] * De[i];
        o1 += wt[nbs + i] * De[i];
      }
      if (wn) {
        /* neighbour traverses the shared edge backwards: t' = 1 - t (mesh2d.py:201) */
        const double* Dn = m->fD + ((size_t)e2 * nf + (nf - 1 - q)) * nbs;
        for (int i = 0; i < nbs; ++i) {
          h0 += wn[i] * Dn[i];
          h1 += wn[nbs + i] * Dn[i];
        }
      } else {
        h0 = inflow[((size_t)slot * nf + q) * 2];
        h1 = inflow[((size_t)slot * nf + q) * 2 + 1];
      }
      const double s = m->fw[q] * F;
      for (int i = 0; i < nbs; ++i) {
        r[i] += s * (h0 - o0) * De[i];
        r[nbs + i] += s * (h1 - o1) * De[i];
      }
    }
  }
}

int port_apply(int k, int nt, int nqv, int nf, const double* coef, const double* divm, const double* vw, const double* vD,
               const double* vG, const double* fw, const double* fL, const double* fD, const double* flen,
               const int32_t* nbr, const int32_t* nbr_edge, const int32_t* bslot, const double* u,
               const double* w, const double* inflow, double* r, int nthreads) {
  port_mesh m = {k, nt, nqv, nf, coef, divm, vw, vD, vG, fw, fL, fD, flen, nbr, nbr_edge, bslot};
  const int nb = (k + 1) * (k + 2);
#pragma omp parallel num_threads(nthreads)
  {
    double scratch[128];
#pragma omp for schedule(static)
    for (int T = 0; T < nt; ++T) apply_elem(&m, T, u, w, inflow, r + (size_t)T * nb, scratch);
  }
  return 0;
}

/* forward Euler: w <- w - dt * minv * C(u; w), nsteps times */
int port_substeps(int k, int nt, int nqv, int nf, const double* coef, const double* divm, const double* vw, const double* vD,
                  const double* vG, const double* fw, const double* fL, const double* fD, const double* flen,
                  const int32_t* nbr, const int32_t* nbr_edge, const int32_t* bslot, const double* u,
                  double* w, const double* inflow, const double* minv, double dt, int nsteps,
                  double* work, int nthreads) {
  port_mesh m = {k, nt, nqv, nf, coef, divm, vw, vD, vG, fw, fL, fD, flen, nbr, nbr_edge, bslot};
  const int nb = (k + 1) * (k + 2);
  double* a = w;
  double* b = work;
  for (int s = 0; s < nsteps; ++s) {
#pragma omp parallel num_threads(nthreads)
    {
      double scratch[128];
      double r[128];
#pragma omp for schedule(static)
      for (int T = 0; T < nt; ++T) {
        apply_elem(&m, T, u, a, inflow, r, scratch);
        const double sc = dt * minv[T];
        for (int j = 0; j < nb; ++j) b[(size_t)T * nb + j] = a[(size_t)T * nb + j] - sc * r[j];
      }
    }
    double* t = a; a = b; b = t;
  }
  if (a != w) memcpy(w, a, sizeof(double) * (size_t)nt * nb);
  return 0;
}
