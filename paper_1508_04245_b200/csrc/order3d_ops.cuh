// order3d_ops.cuh — per-order launchers of the 3D kernels (included by order3d_k<K>.cu).
#pragma once
#include <cstdlib>
#include <cstring>
#include <vector>

#include "context.cuh"
#include "conv3d.cuh"

namespace hdgc {

static inline unsigned grid3_for(long long work, int threads) { return (unsigned)((work + threads - 1) / threads); }

// upload the sum-factorisation tables of this order (constant bank)
template <int K>
int launch3_setup(hdgc_ctx* c, const hdgc_tables_desc* t) {
  using S = SF3<K>;
  if (t->col_n != S::N || !t->col_A || !t->col_Ad || !t->col_B || !t->col_Bd || !t->col_C || !t->col_Cd ||
      !t->col_pf)
    return hdgc_set_err(HDGC_EINVAL, "3D collapsed tables missing or n=%d != %d", t->col_n, S::N);
  std::vector<double> h(S::C_TOTAL);
  memcpy(&h[S::C_A], t->col_A, sizeof(double) * S::N * S::NE);
  memcpy(&h[S::C_AD], t->col_Ad, sizeof(double) * S::N * S::NE);
  memcpy(&h[S::C_B], t->col_B, sizeof(double) * S::N * S::NPAIR);
  memcpy(&h[S::C_BD], t->col_Bd, sizeof(double) * S::N * S::NPAIR);
  memcpy(&h[S::C_C], t->col_C, sizeof(double) * S::N * S::NBS);
  memcpy(&h[S::C_CD], t->col_Cd, sizeof(double) * S::N * S::NBS);
  memcpy(&h[S::C_PF], t->col_pf, sizeof(double) * S::NQ * 5);
  // face modes at the face points: D2 = fac_L / 2 (fac_L is the normal-trace basis 2 D2)
  for (int i = 0; i < S::NF * S::NFD; ++i) h[S::C_D2 + i] = 0.5 * t->fac_L[i];
#if HDGC_3D_SYM
  {
    // mirror symmetry of the a rule, used by the volume term of conv3d_kernel
    double bad = 0.0;
    for (int a = 0; a < S::N; ++a)
      for (int i = 0; i <= K; ++i) {
        const double sg = (i & 1) ? -1.0 : 1.0;
        bad = fmax(bad, fabs(t->col_A[(S::N - 1 - a) * S::NE + i] - sg * t->col_A[a * S::NE + i]));
        bad = fmax(bad, fabs(t->col_Ad[(S::N - 1 - a) * S::NE + i] + sg * t->col_Ad[a * S::NE + i]));
      }
    if (bad > 1e-12) return hdgc_set_err(HDGC_EINVAL, "3D collapsed tables are not mirror-symmetric in a (defect %.3e)", bad);
  }
#endif
  CUDA_TRY(cudaMemcpyToSymbol(c_sf3d, h.data(), sizeof(double) * S::C_TOTAL));
  // face trace maps R_f[n][m] = 2 sum_q w_q D_m(x_f(q)) D2_n(q)  (exact: degree 2k <= 3k+1)
  std::vector<double> R((size_t)4 * S::NFD * S::NBS, 0.0);
  for (int f = 0; f < 4; ++f)
    for (int n = 0; n < S::NFD; ++n)
      for (int m = 0; m < S::NBS; ++m) {
        double a = 0.0;
        for (int q = 0; q < S::NF; ++q)
          a += t->fac_w[q] * t->fac_D[((size_t)f * S::NF + q) * S::NBS + m] * t->fac_L[q * S::NFD + n];
        R[((size_t)f * S::NFD + n) * S::NBS + m] = a;   // 2 * w * D * D2 = w * D * fac_L
      }
  int rc = hdgc_dev_alloc(c, (void**)&c->d_ftab, sizeof(double) * R.size());
  if (rc) return rc;
  {
    // A fragments of prep_tile3d_kernel's DMMA stage: M = [coef ; divm] ((NB + NBS1) x NB)
    using P = Prep3Mma<K>;
    std::vector<double> M((size_t)P::NR * P::NB), af(P::AFRAG);
    memcpy(M.data(), t->coef, sizeof(double) * P::NB * P::NB);
    memcpy(M.data() + (size_t)P::NB * P::NB, t->div_modal, sizeof(double) * (P::NR - P::NB) * P::NB);
    dmma_a_fragments(M.data(), P::NR, P::NB, af.data());
    if ((rc = hdgc_dev_alloc(c, (void**)&c->d_afrag, sizeof(double) * af.size()))) return rc;
    CUDA_TRY(cudaMemcpy(c->d_afrag, af.data(), sizeof(double) * af.size(), cudaMemcpyHostToDevice));
  }
  CUDA_TRY(cudaMemcpy(c->d_ftab, R.data(), sizeof(double) * R.size(), cudaMemcpyHostToDevice));
  return HDGC_OK;
}

template <int K>
int launch3_prep(hdgc_ctx* c, const double* u, cudaStream_t st) {
  c->sweep = 1;   // the update kernel after a prep sweeps last to first (newest prep rows in L2)
  Prep3Params p;
  p.tab = c->d_tab;
  p.u = u;
  p.sgn = c->d_sign;
  p.prep = c->d_prep;
  p.nt = c->nt;
  p.ps = prep3_stride(c->nt);
  static const bool tile = [] {
    const char* e = getenv("HDGC_PREP");
    return !(e && e[0] == '0');
  }();
  if (tile) {
    // measured at cfg5 (196608 tets, k=3): see DESIGN.md §10
    using P = Prep3Mma<K>;
    const int smem = P::SMEM * (int)sizeof(double);
    if (smem > 48 * 1024)
      CUDA_TRY(cudaFuncSetAttribute(prep_tile3d_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    prep_tile3d_kernel<K><<<grid3_for(c->nt, 32), 32 * P::WARPS, smem, st>>>(c->d_tab, c->d_afrag, u, c->d_sign,
                                                                            c->d_code, c->nt, prep3_stride(c->nt),
                                                                            c->d_prep);
  } else {
    prep3d_kernel<K><<<grid3_for(c->nt, 128), 128, 0, st>>>(p);
  }
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

template <int K>
int launch3_main(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out, const StageParams& sp,
                 cudaStream_t st) {
  Conv3Params p;
  p.tab = c->d_tab;
  p.rtab = c->d_ftab;
  p.prep = c->d_prep;
  p.w = w;
  p.inflow = inflow;
  p.code = c->d_code;
  p.minv = c->d_minv;
  p.out = out;
  p.st = sp;
  p.nt = c->nt;
  p.ps = prep3_stride(c->nt);
  p.prep_dep = c->prep_dep ? 1 : 0;
  static const bool zigzag = [] { const char* e = getenv("HDGC_ZIGZAG"); return !(e && e[0] == '0'); }();
  p.rev = zigzag ? (int)(c->sweep++ & 1u) : 0;
  const unsigned blocks = grid3_for(c->nt, Dims3<K>::EPB);
  constexpr int smem = Dims3<K>::SMEM;
  auto launch = [&](auto kern) -> int {
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CUDA_TRY(launch_maybe_pdl(kern, blocks, Dims3<K>::THREADS, smem, st, c->pdl, p));
    return HDGC_OK;
  };
  int rc = mode == MODE_SUBSTEP ? launch(conv3d_kernel<K, MODE_SUBSTEP>)
           : mode == MODE_STAGE ? launch(conv3d_kernel<K, MODE_STAGE>)
                                : launch(conv3d_kernel<K, MODE_APPLY>);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

template <int K>
int launch3_transfer(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st) {
  const long long work = (long long)c->nt * Dims3<K>::NB;
  if (dir == 0) transfer3d_kernel<K, false><<<grid3_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, in, out);
  else transfer3d_kernel<K, true><<<grid3_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, in, out);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

template <int K>
int launch3_maxspeed(hdgc_ctx* c, const double* u, double* out, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
  maxspeed3d_kernel<K><<<grid3_for(c->nt, 128), 128, 0, st>>>(c->d_tab, c->d_piola, c->nt, u,
                                                             reinterpret_cast<unsigned long long*>(out));
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

}  // namespace hdgc

#define HDGC_INSTANTIATE_ORDER3(K)                                                                  \
  namespace hdgc {                                                                                  \
  template int launch3_prep<K>(hdgc_ctx*, const double*, cudaStream_t);                             \
  template int launch3_main<K>(hdgc_ctx*, int, const double*, const double*, double*, const StageParams&, cudaStream_t); \
  template int launch3_transfer<K>(hdgc_ctx*, int, const double*, double*, cudaStream_t);           \
  template int launch3_maxspeed<K>(hdgc_ctx*, const double*, double*, cudaStream_t);                \
  template int launch3_setup<K>(hdgc_ctx*, const hdgc_tables_desc*);                               \
  }
