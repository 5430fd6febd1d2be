// order_ops.cuh — per-order kernel launchers (included by order_k<K>.cu only).
#pragma once
#include <cstdlib>
#include <cstring>

#include "context.cuh"
#include "conv2d_thread.cuh"
#include "conv2d_sf.cuh"
#include "conv2d_sfm.cuh"

namespace hdgc {

// ---------------------------------------------------------------------------
// small per-element matrix-vector products, one thread per (element, row):
// no large unrolled blocks, so every order compiles in seconds.

// I (BDM -> V_h): w[c*nbs+m] = sum_d P[c][d] (coef u)[d*nbs+m]
// I^T:            r_w[j]     = sum_{d,m} coef[d*nbs+m][j] sum_c P[c][d] r[c*nbs+m]
// one thread per (element, output row); in and out must not alias.
template <int K, bool TRANSPOSE>
__global__ void __launch_bounds__(256)
transfer2d_kernel(const double* __restrict__ tab, const double* __restrict__ piola, int nt,
                  const double* __restrict__ in, double* __restrict__ out) {
  using D = Dims<K>;
  constexpr int NB = D::NB, NBS = D::NBS;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)nt * NB) return;
  const int T = (int)(gid / NB);
  const int r = (int)(gid - (long long)T * NB);
  const double P00 = __ldg(piola + T), P01 = __ldg(piola + (size_t)nt + T);
  const double P10 = __ldg(piola + 2 * (size_t)nt + T), P11 = __ldg(piola + 3 * (size_t)nt + T);
  const double* coef = tab + D::OFF_COEF;
  const double* x = in + (size_t)T * NB;
  if (!TRANSPOSE) {
    const int c = r >= NBS ? 1 : 0, m = r - c * NBS;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double xj = __ldg(x + j);
      a0 = fma(__ldg(coef + (size_t)m * NB + j), xj, a0);
      a1 = fma(__ldg(coef + (size_t)(NBS + m) * NB + j), xj, a1);
    }
    out[gid] = c == 0 ? fma(P00, a0, P01 * a1) : fma(P10, a0, P11 * a1);
  } else {
    double a = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      const double x0 = __ldg(x + m), x1 = __ldg(x + NBS + m);
      a = fma(__ldg(coef + (size_t)m * NB + r), fma(P00, x0, P10 * x1), a);
      a = fma(__ldg(coef + (size_t)(NBS + m) * NB + r), fma(P01, x0, P11 * x1), a);
    }
    out[gid] = a;
  }
}

// max |J u_hat / detJ| over elements x volume points, one thread per
// (element, point), from the modal rows; positive doubles order as uint64
template <int K>
__global__ void __launch_bounds__(256)
maxspeed2d_kernel(const double* __restrict__ tab, const double* __restrict__ piola, int nt,
                  const double* __restrict__ modal, const double* __restrict__ minv,
                  unsigned long long* __restrict__ out) {
  using D = Dims<K>;
  constexpr int NBS = D::NBS, MR = D::NB + D::NBS1, NQV = D::NQV;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double best = 0.0;
  if (gid < (long long)nt * NQV) {
    const int T = (int)(gid / NQV);
    const int q = (int)(gid - (long long)T * NQV);
    const double* mr = modal + (size_t)T * MR;
    const double* Dq = tab + D::OFF_VD + q * NBS;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      const double d = __ldg(Dq + m);
      a = fma(__ldg(mr + m), d, a);
      b = fma(__ldg(mr + NBS + m), d, b);
    }
    const double P00 = __ldg(piola + T), P01 = __ldg(piola + (size_t)nt + T);
    const double P10 = __ldg(piola + 2 * (size_t)nt + T), P11 = __ldg(piola + 3 * (size_t)nt + T);
    const double x = fma(P00, a, P01 * b), y = fma(P10, a, P11 * b);
    best = __ldg(minv + T) > 0.0 ? sqrt(fma(x, x, y * y)) : 0.0;   // curved: curved_maxspeed_kernel
  }
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

static inline unsigned grid_for(long long work, int threads) { return (unsigned)((work + threads - 1) / threads); }

template <int K>
int launch_elem(hdgc_ctx* c, int mode, const double* u, const double* w, const double* inflow,
                       double* out, const StageParams& sp, cudaStream_t st) {
 if constexpr (K > 2) {
  (void)c; (void)mode; (void)u; (void)w; (void)inflow; (void)out; (void)sp; (void)st;
  return hdgc_set_err(HDGC_EUNSUP, "thread-per-element variant is built for k <= 2 only");
 } else {
  ElemParams p;
  p.tab = c->d_tab;
  p.u = u;
  p.w = w;
  p.inflow = inflow;
  p.code = c->d_code;
  p.piola = c->d_piola;
  p.minv = c->d_minv;
  p.out = out;
  p.st = sp;
  p.nt = c->nt;
  const int threads = THREAD_BLOCK;
  const int blocks = (c->nt + threads - 1) / threads;
  const int smem = thread_smem_bytes<K>();
  auto launch = [&](auto kern) -> int {
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CUDA_TRY(launch_maybe_pdl(kern, blocks, threads, smem, st, c->pdl, p));
    return HDGC_OK;
  };
  if (c->tprep_on && c->d_tprep) {
    p.prep = c->d_tprep;
#if HDGC_THR_SPLIT
    // one thread per (element, component): 128 threads per 64-element tile
    auto launch2 = [&](auto kern) -> int {
      constexpr int smem2 = split_smem_bytes<K>();
      if (smem2 > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      CUDA_TRY(launch_maybe_pdl(kern, blocks, 2 * threads, smem2, st, c->pdl, p));
      return HDGC_OK;
    };
    // measured (profiles/split_k2_r02.jsonl): ahead once w, out and the prep rows no
    // longer fit the L2 together (k=2, 524k triangles: 59.2 -> 53.7 us, 4.6 TB/s of
    // DRAM), behind while they do (131k: 15.5 vs 14.3-15.0 us; k=1: 7.7 vs 6.4 us)
    // HDGC_SPLIT=1 / 0 forces it on / off (tests run both kernels on small meshes)
    static const int split_force = [] { const char* se = getenv("HDGC_SPLIT"); return se ? (se[0] == '0' ? -1 : 1) : 0; }();
    const bool split = K == 2 && (split_force > 0 ||
                                  (split_force == 0 &&
                                   (size_t)c->nt * (ThreadPrep<K>::SLOTS + 2 * Dims<K>::NB) * 8 > ((size_t)96 << 20)));
    if (split && mode == MODE_SUBSTEP) return launch2(conv2d_thread_split_kernel<K, MODE_SUBSTEP>);
    if (split && mode == MODE_STAGE) return launch2(conv2d_thread_split_kernel<K, MODE_STAGE>);
#endif
    if (mode == MODE_SUBSTEP) return launch(conv2d_thread_kernel<K, MODE_SUBSTEP, true>);
    if (mode == MODE_STAGE) return launch(conv2d_thread_kernel<K, MODE_STAGE, true>);
  }
  switch (mode) {
    case MODE_APPLY: return launch(conv2d_thread_kernel<K, MODE_APPLY>);
    case MODE_SUBSTEP: return launch(conv2d_thread_kernel<K, MODE_SUBSTEP>);
    case MODE_STAGE: return launch(conv2d_thread_kernel<K, MODE_STAGE>);
    default: return launch(conv2d_thread_kernel<K, MODE_APPLY_IT>);
  }
 }
}

// frozen-velocity rows of the thread variant (k <= 2) into c->d_tprep
template <int K>
int launch_elem_prep(hdgc_ctx* c, const double* u, cudaStream_t st) {
  if constexpr (K > 2) {
    (void)c; (void)u; (void)st;
    return hdgc_set_err(HDGC_EUNSUP, "thread-per-element variant is built for k <= 2 only");
  } else {
    const int blocks = (c->nt + THREAD_BLOCK - 1) / THREAD_BLOCK;
    if (!c->d_tprep) {
      const int rc = hdgc_dev_alloc(c, (void**)&c->d_tprep,
                                    sizeof(double) * (size_t)blocks * ThreadPrep<K>::SLOTS * THREAD_BLOCK);
      if (rc) return rc;
    }
    prep_thread2d_kernel<K><<<blocks, THREAD_BLOCK, 0, st>>>(u, c->nt, c->d_tprep);
    CUDA_TRY(cudaGetLastError());
    return HDGC_OK;
  }
}

template <int K>
int launch_transfer(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st) {
  const long long work = (long long)c->nt * Dims<K>::NB;
  if (dir == 0) transfer2d_kernel<K, false><<<grid_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, in, out);
  else transfer2d_kernel<K, true><<<grid_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, in, out);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

// modal rows u_hat | div u_hat into c->d_modal
template <int K>
int launch_modal(hdgc_ctx* c, const double* u, cudaStream_t st) {
  // modal velocity rows [u_hat | div u_hat] = [coef ; divm] u (PB:357-378)
  return hdgc_modal_gemm(c, u, Dims<K>::NB, Dims<K>::NB + Dims<K>::NBS1, Dims<K>::OFF_COEF, st);
}

template <int K>
int launch_maxspeed(hdgc_ctx* c, const double* u, double* out, cudaStream_t st) {
  int rc = launch_modal<K>(c, u, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
  const long long work = (long long)c->nt * Dims<K>::NQV;
  maxspeed2d_kernel<K><<<grid_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, c->d_modal, c->d_minv,
                                                           reinterpret_cast<unsigned long long*>(out));
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

// frozen-velocity prep rows (alpha | beta | gamma | s) into c->d_prep
// orders that run the modal-prep variant (conv2d_sfm.cuh); HDGC_MODAL=0 turns
// it off, HDGC_MODAL=<digits> selects the orders (development A/B switch)
template <int K>
bool modal_enabled() {
  if constexpr (K < 3 || K > 6) {
    return false;
  } else {
    // default off: measured at cfg2 (k = 4, 131k triangles) the modal kernel
    // moves 106 MB per launch instead of 188 MB but executes 1.34 GFLOP
    // instead of 0.92 and runs 80-86 us against 59 us
    const char* e = getenv("HDGC_MODAL");
    if (!e) return false;
    for (const char* q = e; *q; ++q)
      if (*q - '0' == K) return true;
    return false;
  }
}

template <int K>
int sf_prep(hdgc_ctx* c, const double* u, cudaStream_t st) {
  // the prep writes its tiles first to last: the update kernel after it sweeps
  // last to first and finds the newest prep tiles in L2 (SFParams::rev)
  c->sweep = 1;
  if constexpr (K >= 3 && K <= 6) {
    if (c->modal) {
      const int smem = PrepMma<K>::SMEM * (int)sizeof(double);
      if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(prep_modal2d_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      prep_modal2d_kernel<K><<<(c->nt + 31) / 32, 32 * SF<K>::N, smem, st>>>(c->d_tab, c->d_afrag, u, c->d_minv,
                                                                           c->nt, c->d_mprep);
      CUDA_TRY(cudaGetLastError());
      return HDGC_OK;
    }
  }
  // Measured per launch at 131072 elements (ncu, cold): k=3 the fused
  // thread-per-element kernel (24 us; tile 39 us); k>=4 the tile kernel with
  // its DMMA modal stage (k=4 47 us vs fused 84; k=5 87 vs the round-1 cuBLAS DGEMM 41 + rows 78;
  // k=6 122 vs 81 + 125; k=7 241 vs 102 + 220; k=8 386 vs 123 + 293).
  // HDGC_PREP=0 selects the older paths (A/B; the modal rows now by modal_rows_kernel).
  if constexpr (K >= 4) {
    static const bool tile = [] {
      const char* e = getenv("HDGC_PREP");
      return !(e && e[0] == '0');
    }();
    if (tile && c->d_afrag) {
      const int smem = PrepMma<K>::SMEM * (int)sizeof(double);
      if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(prep_tile2d_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      prep_tile2d_kernel<K><<<(c->nt + 31) / 32, 32 * SF<K>::N, smem, st>>>(c->d_tab, c->d_afrag, u, c->nt,
                                                                          c->d_prep);
      CUDA_TRY(cudaGetLastError());
      return HDGC_OK;
    }
  }
  if constexpr (K >= 3 && K <= 4) {
    prep_fused2d_kernel<K><<<grid_for(c->nt, 128), 128, 0, st>>>(u, c->nt, c->d_prep);
    CUDA_TRY(cudaGetLastError());
    return HDGC_OK;
  }
  if constexpr (K >= 3) {
    int rc = launch_modal<K>(c, u, st);
    if (rc) return rc;
    prep_rows2d_kernel<K><<<(c->nt + 15) / 16, 16 * SF<K>::N, 0, st>>>(c->d_tab, u, c->d_modal, c->nt,
                                                                       c->d_prep);
    CUDA_TRY(cudaGetLastError());
    return HDGC_OK;
  } else {
    (void)c; (void)u; (void)st;
    return hdgc_set_err(HDGC_EUNSUP, "sum-factorised variant needs k >= 3");
  }
}

template <int K>
int sf_main(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out, const StageParams& sp,
                   cudaStream_t st) {
  if constexpr (K >= 3) {
    using F = SF<K>;
    SFParams p;
    p.prep = c->d_prep;
    p.w = w;
    p.inflow = inflow;
    p.code = c->d_code;
    p.minv = c->d_minv;
    p.ftab = c->d_ftab;
    p.out = out;
    p.st = sp;
    p.nt = c->nt;
    p.prep_dep = c->prep_dep ? 1 : 0;
    // HDGC_ZIGZAG=0: every launch sweeps forward (development A/B)
    static const bool zigzag = [] { const char* e = getenv("HDGC_ZIGZAG"); return !(e && e[0] == '0'); }();
    p.rev = zigzag ? (int)(c->sweep++ & 1u) : 0;
    if constexpr (K <= 6) {
      // three-warp kernel (conv2d_sfm.cuh): modal prep, or (HDGC_SFM3=1) the point prep
      static const bool sfm3 = [] { const char* e = getenv("HDGC_SFM3"); return e && e[0] == '1'; }();
      if (c->modal || sfm3) {
        using S = SFM<K>;
        const int blocks = (c->nt + S::EPB - 1) / S::EPB;
        auto launch = [&](auto kern, int smem) -> int {
          if (smem > 48 * 1024)
            CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          CUDA_TRY(launch_maybe_pdl(kern, blocks, S::THREADS, smem, st, c->pdl, p));
          return HDGC_OK;
        };
        if (c->modal) {
          p.prep = c->d_mprep;
          const int smem = S::template L<true>::SMEM_DOUBLES * (int)sizeof(double);
          if (mode == MODE_SUBSTEP) return launch(conv2d_sfm_kernel<K, MODE_SUBSTEP, true>, smem);
          if (mode == MODE_STAGE) return launch(conv2d_sfm_kernel<K, MODE_STAGE, true>, smem);
          return launch(conv2d_sfm_kernel<K, MODE_APPLY, true>, smem);
        }
        const int smem = S::template L<false>::SMEM_DOUBLES * (int)sizeof(double);
        if (mode == MODE_SUBSTEP) return launch(conv2d_sfm_kernel<K, MODE_SUBSTEP, false>, smem);
        if (mode == MODE_STAGE) return launch(conv2d_sfm_kernel<K, MODE_STAGE, false>, smem);
        return launch(conv2d_sfm_kernel<K, MODE_APPLY, false>, smem);
      }
    }
    const int smem = F::smem_doubles(mode) * (int)sizeof(double);
    const int blocks = (c->nt + F::EPB - 1) / F::EPB;
    auto launch = [&](auto kern) -> int {
      if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CUDA_TRY(launch_maybe_pdl(kern, blocks, F::THREADS, smem, st, c->pdl, p));
      return HDGC_OK;
    };
    if (mode == MODE_SUBSTEP) return launch(conv2d_sf_kernel<K, MODE_SUBSTEP>);
    if (mode == MODE_STAGE) return launch(conv2d_sf_kernel<K, MODE_STAGE>);
    return launch(conv2d_sf_kernel<K, MODE_APPLY>);
  } else {
    return hdgc_set_err(HDGC_EUNSUP, "sum-factorised variant needs k >= 3");
  }
}

// upload the sum-factorisation tables (constant bank) and facet tables
template <int K>
int sf_setup(hdgc_ctx* c, const hdgc_tables_desc* t, const std::vector<double>& packed) {
  if constexpr (K >= 3) {
    using F = SF<K>;
    using D = Dims<K>;
    if (t->col_n != F::N || !t->col_A || !t->col_Ad || !t->col_B || !t->col_Bd || !t->col_xi ||
        !t->col_wa || !t->col_wy || !t->col_inv1my)
      return hdgc_set_err(HDGC_EINVAL, "collapsed (sum-factorisation) tables missing or n=%d != %d", t->col_n, F::N);
    std::vector<double> h(F::C_TOTAL);
    memcpy(&h[F::C_A], t->col_A, sizeof(double) * F::N * F::NE);
    memcpy(&h[F::C_AD], t->col_Ad, sizeof(double) * F::N * F::NE);
    memcpy(&h[F::C_B], t->col_B, sizeof(double) * F::N * F::NBS);
    memcpy(&h[F::C_BD], t->col_Bd, sizeof(double) * F::N * F::NBS);
    // per-point factors of alpha/beta/gamma: point p = b*n + a (collapsed rule order)
    for (int b = 0; b < F::N; ++b)
      for (int a = 0; a < F::N; ++a) {
        const double wp = t->col_wa[a] * t->col_wy[b];
        h[F::C_PA + b * F::N + a] = wp * t->col_inv1my[b];
        h[F::C_PB + b * F::N + a] = wp * t->col_xi[a] * t->col_inv1my[b];
        h[F::C_PW + b * F::N + a] = wp;
      }
    if (F::SYM) {
      // mirror symmetry of the xi rule and of the facet rule, used by sf_row / facets_v2:
      // A_i(N-1-a) = (-1)^i A_i(a), A'_i(N-1-a) = (-1)^(i+1) A'_i(a), L_l(t_{NF-1-q}) = (-1)^l L_l(t_q)
      double bad = 0.0;
      for (int a = 0; a < F::N; ++a)
        for (int i = 0; i <= K; ++i) {
          const double sg = (i & 1) ? -1.0 : 1.0;
          bad = fmax(bad, fabs(t->col_A[(F::N - 1 - a) * F::NE + i] - sg * t->col_A[a * F::NE + i]));
          bad = fmax(bad, fabs(t->col_Ad[(F::N - 1 - a) * F::NE + i] + sg * t->col_Ad[a * F::NE + i]));
        }
      for (int q = 0; q < F::NF; ++q)
        for (int l = 0; l < F::NE; ++l) {
          const double sg = (l & 1) ? -1.0 : 1.0;
          bad = fmax(bad, fabs(packed[D::OFF_FL + (F::NF - 1 - q) * F::NE + l] - sg * packed[D::OFF_FL + q * F::NE + l]));
        }
      if (bad > 1e-12)
        return hdgc_set_err(HDGC_EINVAL, "collapsed / facet tables are not mirror-symmetric (defect %.3e)", bad);
    }
    CUDA_TRY(cudaMemcpyToSymbol(c_sf, h.data(), sizeof(double) * F::C_TOTAL));
    CUDA_TRY(cudaMemcpyToSymbol(c_fd, &packed[D::OFF_FD], sizeof(double) * 3 * F::NF * F::NBS));
    CUDA_TRY(cudaMemcpyToSymbol(c_fl, &packed[D::OFF_FL], sizeof(double) * F::NF * F::NE));
    // smem table for the substep kernel: edge trace maps
    //   R_e[l][m] = int_0^1 D_m(x_e(t)) L_l(t) dt = sum_q w_q fD[e][q][m] L[q][l]  (exact, degree 2k)
    std::vector<double> ft(F::TAB_PAD, 0.0);
    for (int e = 0; e < 3; ++e)
      for (int l = 0; l < F::NE; ++l)
        for (int m = 0; m < F::NBS; ++m) {
          double a = 0.0;
          for (int q = 0; q < F::NF; ++q)
            a += packed[D::OFF_FW + q] * packed[D::OFF_FD + (e * F::NF + q) * F::NBS + m] *
                 packed[D::OFF_FL + q * F::NE + l];
          ft[e * F::RSTR + l * F::NBS + m] = a;
        }
    {
      // structured trace maps for facets_v2 (conv2d_sf.cuh): R_0 diagonal in i, R_1
      // lower-triangular in the total degree, R_2 = (-1)^(i+l) R_1 -- checked here
      std::vector<double> r0(F::NBS, 0.0), r1(F::NE * F::NBS, 0.0);
      double bad = 0.0;
      for (int i = 0; i <= K; ++i)
        for (int j = 0; j <= K - i; ++j) {
          const int m = midx(i, j);
          for (int l = 0; l < F::NE; ++l) {
            const double v0 = ft[0 * F::RSTR + l * F::NBS + m], v1 = ft[1 * F::RSTR + l * F::NBS + m],
                         v2 = ft[2 * F::RSTR + l * F::NBS + m];
            if (l == i) r0[m] = v0; else bad = fmax(bad, fabs(v0));
            if (l <= i + j) r1[l * F::NBS + m] = v1; else bad = fmax(bad, fabs(v1));
            bad = fmax(bad, fabs(v2 - (((i + l) & 1) ? -v1 : v1)));
          }
        }
      if (bad > 1e-12)
        return hdgc_set_err(HDGC_EINVAL, "facet tables do not have the Dubiner edge-trace structure (defect %.3e)", bad);
      CUDA_TRY(cudaMemcpyToSymbol(c_r0, r0.data(), sizeof(double) * F::NBS));
      CUDA_TRY(cudaMemcpyToSymbol(c_r1, r1.data(), sizeof(double) * F::NE * F::NBS));
      std::vector<double> tr;   // order of use in edge_traces / edge_test
      for (int d = 0; d <= K; ++d)
        for (int j = 0; j <= d; ++j) {
          const int m = midx(d - j, j);
          tr.push_back(r0[m]);
          for (int l = 0; l <= d; ++l) tr.push_back(r1[l * F::NBS + m]);
        }
      tr.resize((tr.size() + 1) & ~size_t(1), 0.0);
      if (tr.size() * sizeof(double) != sizeof(c_tr)) return hdgc_set_err(HDGC_EINVAL, "trace table size");
      CUDA_TRY(cudaMemcpyToSymbol(c_tr, tr.data(), sizeof(double) * tr.size()));
    }
#if HDGC_CM_FUSED
    {
      // [coef ; divm] | fL | fw | flen for the fused prep kernel
      std::vector<double> cm((F::NB + F::NBS1) * F::NB + F::NF * F::NE + F::NF + 3);
      memcpy(&cm[0], &packed[D::OFF_COEF], sizeof(double) * (F::NB + F::NBS1) * F::NB);
      size_t o2 = (size_t)(F::NB + F::NBS1) * F::NB;
      memcpy(&cm[o2], &packed[D::OFF_FL], sizeof(double) * F::NF * F::NE); o2 += F::NF * F::NE;
      memcpy(&cm[o2], &packed[D::OFF_FW], sizeof(double) * F::NF); o2 += F::NF;
      memcpy(&cm[o2], &packed[D::OFF_FLEN], sizeof(double) * 3);
      CUDA_TRY(cudaMemcpyToSymbol(c_cm, cm.data(), sizeof(double) * cm.size()));
    }
#endif
    if constexpr (K >= 4) {
      // A fragments of the tile prep's DMMA stage (prep_tile2d_kernel): M = [coef ; divm]
      using P = PrepMma<K>;
      std::vector<double> af(P::AFRAG, 0.0);
      dmma_a_fragments(&packed[D::OFF_COEF], P::NR, P::NB, af.data());   // coef rows then divm rows
      int rc0 = hdgc_dev_alloc(c, (void**)&c->d_afrag, sizeof(double) * P::AFRAG);
      if (rc0) return rc0;
      CUDA_TRY(cudaMemcpy(c->d_afrag, af.data(), sizeof(double) * P::AFRAG, cudaMemcpyHostToDevice));
    }
    int rc = hdgc_dev_alloc(c, (void**)&c->d_ftab, sizeof(double) * F::TAB_PAD);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(c->d_ftab, ft.data(), sizeof(double) * F::TAB_PAD, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpyToSymbol(c_fw, &packed[D::OFF_FW], sizeof(double) * F::NF));
    if constexpr (K >= 4 && K <= 6) c->modal = modal_enabled<K>();
    if (c->modal) {
      const size_t n = (size_t)((c->nt + 31) / 32) * 2 * SFM<K>::MTILE;   // whole 32-element prep CTAs
      rc = hdgc_dev_alloc(c, (void**)&c->d_mprep, sizeof(double) * n);
      if (rc) return rc;
      CUDA_TRY(cudaMemset(c->d_mprep, 0, sizeof(double) * n));
    } else {
      rc = hdgc_dev_alloc(c, (void**)&c->d_prep, sizeof(double) * (size_t)((c->nt + 15) / 16) * F::PREP_TILE);
      if (rc) return rc;
      CUDA_TRY(cudaMemset(c->d_prep, 0, sizeof(double) * (size_t)((c->nt + 15) / 16) * F::PREP_TILE));
    }
    c->variant = 1;
    return HDGC_OK;
  } else {
    // thread-per-element variant: the packed tables into this order's constant bank
    (void)t;
    CUDA_TRY(cudaMemcpyToSymbol(c_th, packed.data(), sizeof(double) * Dims<K>::TAB));
    return HDGC_OK;
  }
}

}  // namespace hdgc

#define HDGC_INSTANTIATE_ORDER(K)                                                                 \
  namespace hdgc {                                                                                \
  template int launch_elem<K>(hdgc_ctx*, int, const double*, const double*, const double*, double*, \
                              const StageParams&, cudaStream_t);                                              \
  template int launch_elem_prep<K>(hdgc_ctx*, const double*, cudaStream_t);                      \
  template int launch_transfer<K>(hdgc_ctx*, int, const double*, double*, cudaStream_t);          \
  template int launch_maxspeed<K>(hdgc_ctx*, const double*, double*, cudaStream_t);               \
  template int sf_prep<K>(hdgc_ctx*, const double*, cudaStream_t);                                \
  template int sf_main<K>(hdgc_ctx*, int, const double*, const double*, double*, const StageParams&, cudaStream_t); \
  template int sf_setup<K>(hdgc_ctx*, const hdgc_tables_desc*, const std::vector<double>&);        \
  }
