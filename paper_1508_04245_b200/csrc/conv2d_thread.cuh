// Variant "thread" (k <= 2): one thread per element, fused volume + upwind
// facets, tables as constant-bank operands (fully unrolled point loops).
//
// Operator, geometry-free reference form
// on affine elements, evaluated in the equivalent
// "flux-difference" form
//
//   r[c,m] =  sum_p w_p ( u_hat.grad_hat w_c + w_c div_hat u_hat )(p) D_m(p)
//           + sum_e sum_{q: F<0} w_q F_e(t_q) ( w_ext - w_own )_c(t_q) D_m(x_e(t_q))
//
// which equals the textbook form  -int w (x) u : grad z + int (u.n) w_hat z
// exactly (divergence theorem; both rules integrate the polynomial integrands
// exactly: volume degree 3k-1, facet degree 3k), but does not cancel two large
// terms against each other, so its fp64 rounding error stays ~1e-15 relative
// where the textbook form loses 2-4 digits on fine meshes.
//   F_e(t) = |e_hat| sum_l u[e*(k+1)+l] L_l(t)   (= u.n ds/dt)
//   w_ext  = neighbour trace at t' = 1 - t (mesh2d.py:201), or inflow data
#pragma once
#include "common.cuh"

namespace hdgc {

#ifndef HDGC_ORDER
#error "define HDGC_ORDER before including conv2d_thread.cuh"
#endif
#if HDGC_ORDER <= 2
// the packed reference tables of this translation unit's order (Dims<K> layout)
// in the constant bank: with every loop over points and edges unrolled, each
// table entry is an immediate uniform operand of its DFMA (no LDS per FMA)
__constant__ double c_th[Dims<HDGC_ORDER>::TAB];
#else
__constant__ double c_th[1];
#endif

#ifndef HDGC_THR_BLOCK
#define HDGC_THR_BLOCK 64
#endif
constexpr int THREAD_BLOCK = HDGC_THR_BLOCK;   // small blocks: 2048 CTAs at 131k elements fill the SMs in ~2 full waves

#ifndef HDGC_THR_TMA
#define HDGC_THR_TMA 1   // stage the CTA's u and w rows with TMA bulk copies (0: per-thread global loads)
#endif
// smem (doubles): neighbour-side facet traces fD [3][NF][NBS] (padded even) |
//                 TMA: u tile [64][NB] | w tile [64][NB]
template <int K>
__host__ __device__ constexpr int thread_fd_doubles() { return (3 * Dims<K>::NF * Dims<K>::NBS + 1) & ~1; }
template <int K>
__host__ __device__ constexpr int thread_smem_bytes() {
  return (thread_fd_doubles<K>() + (HDGC_THR_TMA ? 2 * THREAD_BLOCK * Dims<K>::NB : 0)) * 8;
}

// copy a row of N doubles (16-byte aligned when N is even) with 16-byte
// accesses where possible
template <int N, bool LDG = false>
__device__ __forceinline__ void row_load(double* dst, const double* src) {
  if constexpr (N % 2 == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      const double2 t = LDG ? __ldg(s2 + j) : s2[j];
      dst[2 * j] = t.x;
      dst[2 * j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = LDG ? __ldg(src + j) : src[j];
  }
}

// Frozen-velocity prep of the thread variant (substep batches, hdgc_propagate,
// Richardson: u is frozen over the batch): per element the
// velocity at the NQV volume points, u_hat_0(q), u_hat_1(q), div u_hat(q), and
// the inflow weights s_e(q) = w_q F_e(t_q) where F < 0 (else 0), evaluated with
// the same FMA sequences as the update kernel uses without a prep (so both
// paths give bitwise identical results); the update kernels then neither redo
// the modal transform (NB^2 FMA) nor the velocity evaluation.
// Quadrature-point data, not an assembled matrix.
// Layout [cta][slot][THREAD_BLOCK]: coalesced for writer and readers.
template <int K>
struct ThreadPrep {
  static constexpr int NQV = Dims<K>::NQV, NF = Dims<K>::NF;
  static constexpr int S_FAC = 3 * NQV;
  static constexpr int SLOTS = 3 * NQV + 3 * NF;
};

template <int K>
__global__ void __launch_bounds__(THREAD_BLOCK)
prep_thread2d_kernel(const double* __restrict__ u, int nt, double* __restrict__ prep) {
  static_assert(K == HDGC_ORDER && K <= 2, "thread variant: k <= 2, tables per translation unit");
  using D = Dims<K>;
  using TP = ThreadPrep<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NBS1 = D::NBS1, NE = D::NE, NF = D::NF, NQV = D::NQV;
  const double* coef = c_th + D::OFF_COEF;
  const double* divm = c_th + D::OFF_DIVM;
  const double* vD = c_th + D::OFF_VD;
  const double* fw = c_th + D::OFF_FW;
  const double* fL = c_th + D::OFF_FL;
  const double* flen = c_th + D::OFF_FLEN;
  const int T = blockIdx.x * blockDim.x + threadIdx.x;
  if (T >= nt) return;
  double* out = prep + (size_t)blockIdx.x * TP::SLOTS * THREAD_BLOCK + threadIdx.x;
  double x[NB];
  {
    const double2* ug = reinterpret_cast<const double2*>(u + (size_t)T * NB);
#pragma unroll
    for (int j = 0; j < NB / 2; ++j) {
      const double2 t = __ldg(ug + j);
      x[2 * j] = t.x;
      x[2 * j + 1] = t.y;
    }
  }
#pragma unroll
  for (int e = 0; e < 3; ++e) {
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      double a = 0.0;
#pragma unroll
      for (int l = 0; l < NE; ++l) a = fma(x[e * NE + l], fL[q * NE + l], a);
      const double Fq = a * flen[e];
      out[(TP::S_FAC + e * NF + q) * THREAD_BLOCK] = Fq < 0.0 ? fw[q] * Fq : 0.0;
    }
  }
  double uh[NB], dv[NBS1];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) a = fma(coef[i * NB + j], x[j], a);
    uh[i] = a;
  }
#pragma unroll
  for (int i = 0; i < NBS1; ++i) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) a = fma(divm[i * NB + j], x[j], a);
    dv[i] = a;
  }
#pragma unroll
  for (int q = 0; q < NQV; ++q) {
    const double* Dq = vD + q * NBS;
    double u0 = 0.0, u1 = 0.0, dvq = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      u0 = fma(uh[m], Dq[m], u0);
      u1 = fma(uh[NBS + m], Dq[m], u1);
      if (m < NBS1) dvq = fma(dv[m], Dq[m], dvq);
    }
    out[(3 * q + 0) * THREAD_BLOCK] = u0;
    out[(3 * q + 1) * THREAD_BLOCK] = u1;
    out[(3 * q + 2) * THREAD_BLOCK] = dvq;
  }
}

template <int K, int MODE, bool PREP = false>
#ifndef HDGC_THR_MINB2
#define HDGC_THR_MINB2 8
#endif
__global__ void __launch_bounds__(THREAD_BLOCK, K == 2 ? HDGC_THR_MINB2 * 64 / THREAD_BLOCK : 14 * 64 / THREAD_BLOCK)   // 128 / 72 registers: 8 / 14 CTAs per SM
conv2d_thread_kernel(ElemParams p) {
  static_assert(K == HDGC_ORDER && K <= 2, "thread variant: k <= 2, tables per translation unit");
  using D = Dims<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NBS1 = D::NBS1, NE = D::NE, NF = D::NF, NQV = D::NQV;
  if (MODE == MODE_STAGE && stage_stopped(p.st)) return;   // converged Richardson iteration
  const double* coef = c_th + D::OFF_COEF;
  const double* divm = c_th + D::OFF_DIVM;
  const double* vw = c_th + D::OFF_VW;
  const double* vD = c_th + D::OFF_VD;
  const double* vG = c_th + D::OFF_VG;
  const double* fw = c_th + D::OFF_FW;
  const double* fL = c_th + D::OFF_FL;
  const double* fD = c_th + D::OFF_FD;
  const double* flen = c_th + D::OFF_FLEN;
  // neighbour-side facet traces are indexed by the neighbour's local edge (per
  // lane): from a shared-memory copy instead of divergent constant loads
  extern __shared__ __align__(16) double s_fD[];
  hdgc_debug_prologue(s_fD, thread_smem_bytes<K>() / 8);
  const int tb = blockIdx.x * blockDim.x;
  const int T0 = tb + threadIdx.x;
  const bool active = T0 < p.nt;
  const int T = active ? T0 : p.nt - 1;   // tail lanes recompute the last element, write nothing
  const int nel = min((int)blockDim.x, p.nt - tb);
  // TMA: the CTA's u rows and (after griddepcontrol.wait) w rows arrive as two
  // bulk copies; each thread then reads its own row from smem, and in-tile
  // neighbours' rows come from smem too
  double* s_u = s_fD + thread_fd_doubles<K>();
  double* s_w = s_u + THREAD_BLOCK * NB;
  __shared__ __align__(8) uint64_t tbar[2];
  if (HDGC_THR_TMA && threadIdx.x == 0) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    fence_mbar_init();
  }
  // (filled here, first read in the facet loop: the barrier sits there, so the
  // table's global latency overlaps the u loads and the volume term)
  for (int i = threadIdx.x; i < 3 * NF * NBS; i += blockDim.x) s_fD[i] = p.tab[D::OFF_FD + i];
  if (HDGC_THR_TMA) {
    __syncthreads();   // mbarrier init visible
    if (!PREP && threadIdx.x == 0) {
      mbar_arrive_expect_tx(&tbar[0], (uint32_t)(nel * NB * sizeof(double)));
      bulk_g2s(s_u, p.u + (size_t)tb * NB, (uint32_t)(nel * NB * sizeof(double)), &tbar[0]);
    }
  }

  // PREP: the frozen-velocity rows of this element (prep_thread2d_kernel), all loads
  // in flight before griddepcontrol.wait
  using TP = ThreadPrep<K>;
  double pa[PREP ? 3 * NQV : 1], ps[PREP ? 3 * NF : 1];
  if constexpr (PREP) {
    const double* pr = p.prep + (size_t)blockIdx.x * TP::SLOTS * THREAD_BLOCK + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 3 * NQV; ++i) pa[i] = __ldg(pr + (size_t)i * THREAD_BLOCK);
#pragma unroll
    for (int i = 0; i < 3 * NF; ++i) ps[i] = __ldg(pr + (size_t)(TP::S_FAC + i) * THREAD_BLOCK);
  }
  // modal velocity u_hat = coef u and its modal divergence dv = divm u (in P_{k-1})
  double uh[NB];
  double dv[NBS1];
  if constexpr (!PREP) {
    double u[NB];
    if (HDGC_THR_TMA) {
      mbar_wait(&tbar[0], 0);
      const double2* us = reinterpret_cast<const double2*>(s_u + (T - tb) * NB);
#pragma unroll
      for (int j = 0; j < NB / 2; ++j) {
        const double2 t = us[j];
        u[2 * j] = t.x;
        u[2 * j + 1] = t.y;
      }
    } else {
      const double2* ug = reinterpret_cast<const double2*>(p.u + (size_t)T * NB);
#pragma unroll
      for (int j = 0; j < NB / 2; ++j) {
        const double2 t = __ldg(ug + j);
        u[2 * j] = t.x;
        u[2 * j + 1] = t.y;
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) a = fma(coef[i * NB + j], u[j], a);
      uh[i] = a;
    }
#pragma unroll
    for (int i = 0; i < NBS1; ++i) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) a = fma(divm[i * NB + j], u[j], a);
      dv[i] = a;
    }
  }
  // everything above depends on u and the tables only; w (and x) are the
  // previous update kernel's output under a PDL launch (common.cuh)
  pdl_wait();
  pdl_trigger();
  double w[NB];
  if (HDGC_THR_TMA) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&tbar[1], (uint32_t)(nel * NB * sizeof(double)));
      bulk_g2s(s_w, p.w + (size_t)tb * NB, (uint32_t)(nel * NB * sizeof(double)), &tbar[1]);
    }
    mbar_wait(&tbar[1], 0);
    const double2* ws = reinterpret_cast<const double2*>(s_w + (T - tb) * NB);
#pragma unroll
    for (int j = 0; j < NB / 2; ++j) {
      const double2 t = ws[j];
      w[2 * j] = t.x;
      w[2 * j + 1] = t.y;
    }
  } else {
    const double2* wg = reinterpret_cast<const double2*>(p.w + (size_t)T * NB);
#pragma unroll
    for (int j = 0; j < NB / 2; ++j) {
      const double2 t = __ldg(wg + j);
      w[2 * j] = t.x;
      w[2 * j + 1] = t.y;
    }
  }
  double r[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) r[j] = 0.0;

  // ---- volume: f_c = u.grad w_c + w_c div u, tested against D_m
#pragma unroll
  for (int q = 0; q < NQV; ++q) {
    const double* Dq = vD + q * NBS;
    const double* Gq = vG + q * NBS * 2;
    double w0 = 0.0, w1 = 0.0, u0 = 0.0, u1 = 0.0, dvq = 0.0;
    double w0x = 0.0, w0y = 0.0, w1x = 0.0, w1y = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      const double d = Dq[m], gx = Gq[2 * m], gy = Gq[2 * m + 1];
      w0 = fma(w[m], d, w0);
      w1 = fma(w[NBS + m], d, w1);
      if constexpr (!PREP) {
        u0 = fma(uh[m], d, u0);
        u1 = fma(uh[NBS + m], d, u1);
        if (m < NBS1) dvq = fma(dv[m], d, dvq);
      }
      w0x = fma(w[m], gx, w0x);
      w0y = fma(w[m], gy, w0y);
      w1x = fma(w[NBS + m], gx, w1x);
      w1y = fma(w[NBS + m], gy, w1y);
    }
    if constexpr (PREP) {
      u0 = pa[3 * q];
      u1 = pa[3 * q + 1];
      dvq = pa[3 * q + 2];
    }
    const double wt = vw[q];
    const double f0 = wt * fma(u0, w0x, fma(u1, w0y, w0 * dvq));
    const double f1 = wt * fma(u0, w1x, fma(u1, w1y, w1 * dvq));
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      r[m] = fma(f0, Dq[m], r[m]);
      r[NBS + m] = fma(f1, Dq[m], r[NBS + m]);
    }
  }

  __syncthreads();   // s_fD complete
  // ---- facets: upwind jump on inflow points only (element-owned, no atomics)
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    double F[NF];   // PREP: the inflow weights s_q (0 where F >= 0), else F itself
    bool inflow_edge = false;
    if constexpr (PREP) {
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        F[q] = ps[e * NF + q];
        inflow_edge |= F[q] != 0.0;
      }
    } else {
      double ue[NE];
#pragma unroll
      for (int l = 0; l < NE; ++l) ue[l] = HDGC_THR_TMA ? s_u[(T - tb) * NB + e * NE + l] : __ldg(p.u + (size_t)T * NB + e * NE + l);
      const double len = flen[e];
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        double a = 0.0;
#pragma unroll
        for (int l = 0; l < NE; ++l) a = fma(ue[l], fL[q * NE + l], a);
        F[q] = a * len;
        inflow_edge |= F[q] < 0.0;
      }
    }
    if (!inflow_edge) continue;  // pure outflow edge: w_hat = own trace, jump = 0
    const int code = __ldg(p.code + (size_t)T * 3 + e);
    const double* infl = nullptr;
    double* wn = uh;  // reuse registers: u_hat is dead after the volume term
    int e2 = 0;
    if (code >= 0) {
      HDGC_ASSERT((code >> 2) < p.nt && (code & 3) < 3);
      const int nbT = code >> 2;
      e2 = code & 3;
      if (HDGC_THR_TMA && nbT >= tb && nbT < tb + nel) {
        row_load<NB>(wn, s_w + (nbT - tb) * NB);   // in-tile neighbour: its row is staged
      } else {
        row_load<NB, true>(wn, p.w + (size_t)nbT * NB);
      }
    } else if (p.inflow != nullptr) {
      infl = p.inflow + (size_t)(-1 - code) * NF * 2;
    } else {
      continue;  // boundary without inflow data: exterior value = own trace
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      const double Fq = F[q];
      if (PREP ? Fq == 0.0 : !(Fq < 0.0)) continue;
      const double* De = fD + (e * NF + q) * NBS;
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int m = 0; m < NBS; ++m) {
        o0 = fma(w[m], De[m], o0);
        o1 = fma(w[NBS + m], De[m], o1);
      }
      double x0, x1;
      if (code >= 0) {
        double Dn[NBS];   // per-lane row (the neighbour's local edge): 16-byte LDS when NBS is even
        row_load<NBS>(Dn, s_fD + (e2 * NF + (NF - 1 - q)) * NBS);
        x0 = 0.0; x1 = 0.0;
#pragma unroll
        for (int m = 0; m < NBS; ++m) {
          x0 = fma(wn[m], Dn[m], x0);
          x1 = fma(wn[NBS + m], Dn[m], x1);
        }
      } else {
        x0 = __ldg(infl + 2 * q);
        x1 = __ldg(infl + 2 * q + 1);
      }
      const double s = PREP ? Fq : fw[q] * Fq;
      const double j0 = s * (x0 - o0), j1 = s * (x1 - o1);
#pragma unroll
      for (int m = 0; m < NBS; ++m) {
        r[m] = fma(j0, De[m], r[m]);
        r[NBS + m] = fma(j1, De[m], r[NBS + m]);
      }
    }
  }

  // ---- epilogue
  // APPLY / SUBSTEP with TMA: the rows go back through the w tile and one bulk
  // store (coalesced), instead of 12 strided 8-byte stores per thread
  constexpr bool TSTORE = HDGC_THR_TMA && (MODE == MODE_APPLY || MODE == MODE_SUBSTEP);
  if constexpr (TSTORE) {
    if (MODE == MODE_SUBSTEP && p.st.cres && active) {
      const double mflag = __ldg(p.minv + T);
      if (mflag < 0.0) {
        double* cr = p.st.cres + (size_t)((int)(-mflag) - 1) * NB;   // curved: raw residual to the fix-up
#pragma unroll
        for (int j = 0; j < NB; ++j) cr[j] = r[j];
      }
    }
    double v[NB];
    if (MODE == MODE_APPLY) {
#pragma unroll
      for (int j = 0; j < NB; ++j) v[j] = r[j];
    } else {
      const double cm = p.st.c * __ldg(p.minv + T);
      double chk = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        v[j] = fma(cm, r[j], w[j]);
        chk += v[j];
      }
      guard_finite(p.st.flag, chk);
    }
    __syncthreads();   // every thread's facet loop is done reading the w tile
    if (active) {
      double2* ws = reinterpret_cast<double2*>(s_w + (T - tb) * NB);
#pragma unroll
      for (int j = 0; j < NB / 2; ++j) ws[j] = make_double2(v[2 * j], v[2 * j + 1]);
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(p.out + (size_t)tb * NB, s_w, (uint32_t)(nel * NB * sizeof(double)));
      bulk_wait_read();
    }
    return;
  }
  if (!active) return;
  double* og = p.out + (size_t)T * NB;
  if ((MODE == MODE_SUBSTEP || MODE == MODE_STAGE) && p.st.cres) {
    const double mflag = __ldg(p.minv + T);
    if (mflag < 0.0) {
      // curved element: hand the raw residual to curved_fixup_kernel
      double* cr = p.st.cres + (size_t)((int)(-mflag) - 1) * NB;
#pragma unroll
      for (int j = 0; j < NB; ++j) cr[j] = r[j];
    }
  }
  if (MODE == MODE_APPLY) {
#pragma unroll
    for (int j = 0; j < NB; ++j) og[j] = r[j];
  } else if (MODE == MODE_SUBSTEP) {
    const double cm = p.st.c * __ldg(p.minv + T);
    double chk = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double v = fma(cm, r[j], w[j]);
      og[j] = v;
      chk += v;
    }
    guard_finite(p.st.flag, chk);
  } else if (MODE == MODE_STAGE) {
    const double mi = __ldg(p.minv + T);
    const double cm = p.st.c * mi;
    {
      const double* xg = p.st.x + (size_t)T * NB;
      const double tm = -p.st.tau * mi;
      double acc0 = 0.0, acc1 = 0.0, chk = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const double xv = __ldg(xg + j);
        const double v = fma(p.st.b, xv, fma(cm, r[j], p.st.a * w[j]));
        og[j] = v;
        chk += v;
        const double res = fma(tm, r[j], xv - w[j]);
        if (j < NBS) acc0 = fma(res, res, acc0); else acc1 = fma(res, res, acc1);
      }
      guard_finite(p.st.flag, chk);
      if (p.st.rn) {
        p.st.rn[2 * (size_t)T] = acc0;
        p.st.rn[2 * (size_t)T + 1] = acc1;
      }
    }
  } else {
    // r_w = I^T r: s[d*nbs+m] = sum_c P[c][d] r[c*nbs+m]; r_w[j] = sum_i coef[i][j] s[i]
    const double P00 = __ldg(p.piola + T), P01 = __ldg(p.piola + p.nt + T);
    const double P10 = __ldg(p.piola + 2 * (size_t)p.nt + T), P11 = __ldg(p.piola + 3 * (size_t)p.nt + T);
    double s[NB];
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      s[m] = fma(P00, r[m], P10 * r[NBS + m]);
      s[NBS + m] = fma(P01, r[m], P11 * r[NBS + m]);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) a = fma(coef[i * NB + j], s[i], a);
      og[j] = a;
    }
  }
}

// ---------------------------------------------------------------------------
// Component-split update kernel (frozen-velocity batches: PREP rows present).
// The two Cartesian components of w are advected independently by the same
// velocity (C^V acts on w_c componentwise), so one thread per
// (element, component): 128 threads per 64-element tile, the component is
// warp-uniform (threads 0..63 -> c = 0, 64..127 -> c = 1).  Half the registers
// of the one-thread-per-element kernel (w, r, neighbour row of one component;
// the prep rows are read from a TMA-staged smem tile where they are used
// instead of being held in 66 registers), so twice the warps are resident and
// each carries half the dependent FMA chain.  Every output value is computed
// with the same FMA sequence as in conv2d_thread_kernel: bitwise identical.
#ifndef HDGC_THR_SPLIT
#define HDGC_THR_SPLIT 1
#endif
#ifndef HDGC_THR_SPLIT_MINB
#define HDGC_THR_SPLIT_MINB 8
#endif
template <int K>
__host__ __device__ constexpr int split_smem_bytes() {
  return (thread_fd_doubles<K>() + THREAD_BLOCK * Dims<K>::NB + ThreadPrep<K>::SLOTS * THREAD_BLOCK) * 8;
}

template <int K, int MODE>
__global__ void __launch_bounds__(2 * THREAD_BLOCK, HDGC_THR_SPLIT_MINB)
conv2d_thread_split_kernel(ElemParams p) {
  static_assert(K == HDGC_ORDER && K <= 2, "thread variant: k <= 2, tables per translation unit");
  static_assert(MODE == MODE_SUBSTEP || MODE == MODE_STAGE, "split kernel: update modes of a frozen-velocity batch");
  static_assert(THREAD_BLOCK % 32 == 0, "component must be warp-uniform");
  using D = Dims<K>;
  using TP = ThreadPrep<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NF = D::NF, NQV = D::NQV;
  if (MODE == MODE_STAGE && stage_stopped(p.st)) return;   // converged Richardson iteration
  const double* vw = c_th + D::OFF_VW;
  const double* vD = c_th + D::OFF_VD;
  const double* vG = c_th + D::OFF_VG;
  const double* fD = c_th + D::OFF_FD;
  extern __shared__ __align__(16) double s_fD[];
  hdgc_debug_prologue(s_fD, split_smem_bytes<K>() / 8);
  const int el = threadIdx.x & (THREAD_BLOCK - 1);
  const int c = threadIdx.x / THREAD_BLOCK;
  const int tb = blockIdx.x * THREAD_BLOCK;
  const bool active = tb + el < p.nt;
  const int T = active ? tb + el : p.nt - 1;   // tail lanes recompute the last element, write nothing
  const int nel = min(THREAD_BLOCK, p.nt - tb);
  double* s_w = s_fD + thread_fd_doubles<K>();
  double* s_p = s_w + THREAD_BLOCK * NB;
  __shared__ __align__(8) uint64_t tbar[2];
  if (threadIdx.x == 0) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    fence_mbar_init();
    // the tile's frozen-velocity rows [slot][64]: written by prep_thread2d_kernel
    // before this batch (never launched with a PDL edge to it), so requested
    // first thing, before the table fill and the wait
    constexpr uint32_t pbytes = TP::SLOTS * THREAD_BLOCK * sizeof(double);
    mbar_arrive_expect_tx(&tbar[0], pbytes);
    bulk_g2s(s_p, p.prep + (size_t)blockIdx.x * TP::SLOTS * THREAD_BLOCK, pbytes, &tbar[0]);
  }
  for (int i = threadIdx.x; i < 3 * NF * NBS; i += blockDim.x) s_fD[i] = p.tab[D::OFF_FD + i];
  int code[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) code[e] = __ldg(p.code + (size_t)T * 3 + e);
  const double mi = __ldg(p.minv + T);
  __syncthreads();   // mbarrier init visible, s_fD complete
  // w (and x) are the previous update kernel's output under a PDL launch
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&tbar[1], (uint32_t)(nel * NB * sizeof(double)));
    bulk_g2s(s_w, p.w + (size_t)tb * NB, (uint32_t)(nel * NB * sizeof(double)), &tbar[1]);
  }
  double xs[MODE == MODE_STAGE ? NBS : 1];
  if constexpr (MODE == MODE_STAGE) {
    const double* xg = p.st.x + (size_t)T * NB + c * NBS;
#pragma unroll
    for (int j = 0; j < NBS; ++j) xs[j] = __ldg(xg + j);
  }
  mbar_wait(&tbar[1], 0);
  double w[NBS];
  {
    row_load<NBS>(w, s_w + (T - tb) * NB + c * NBS);
  }
  mbar_wait(&tbar[0], 0);
  const double* pr = s_p + el;
  double r[NBS];
#pragma unroll
  for (int j = 0; j < NBS; ++j) r[j] = 0.0;

  // ---- volume: f_c = u.grad w_c + w_c div u, tested against D_m
#pragma unroll
  for (int q = 0; q < NQV; ++q) {
    const double* Dq = vD + q * NBS;
    const double* Gq = vG + q * NBS * 2;
    double w0 = 0.0, wx = 0.0, wy = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      w0 = fma(w[m], Dq[m], w0);
      wx = fma(w[m], Gq[2 * m], wx);
      wy = fma(w[m], Gq[2 * m + 1], wy);
    }
    const double u0 = pr[(3 * q) * THREAD_BLOCK], u1 = pr[(3 * q + 1) * THREAD_BLOCK];
    const double dvq = pr[(3 * q + 2) * THREAD_BLOCK];
    const double f = vw[q] * fma(u0, wx, fma(u1, wy, w0 * dvq));
#pragma unroll
    for (int m = 0; m < NBS; ++m) r[m] = fma(f, Dq[m], r[m]);
  }

  // ---- facets: upwind jump on inflow points only (element-owned, no atomics).
  // (Measured and not adopted: neighbour rows requested one edge ahead through a
  // generic smem-or-global pointer, 53.7 -> 63-72 us at 524k triangles.)
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    double F[NF];   // inflow weights s_q = w_q F_e(t_q) where F < 0, else 0
    bool inflow_edge = false;
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      F[q] = pr[(TP::S_FAC + e * NF + q) * THREAD_BLOCK];
      inflow_edge |= F[q] != 0.0;
    }
    if (!inflow_edge) continue;  // pure outflow edge: w_hat = own trace, jump = 0
    const int cd = code[e];
    const double* infl = nullptr;
    double wn[NBS];
    int e2 = 0;
    if (cd >= 0) {
      HDGC_ASSERT((cd >> 2) < p.nt && (cd & 3) < 3);
      const int nbT = cd >> 2;
      e2 = cd & 3;
      if (nbT >= tb && nbT < tb + nel) {
        row_load<NBS>(wn, s_w + (nbT - tb) * NB + c * NBS);   // in-tile neighbour: its row is staged
      } else {
        row_load<NBS, true>(wn, p.w + (size_t)nbT * NB + c * NBS);
      }
    } else if (p.inflow != nullptr) {
      infl = p.inflow + (size_t)(-1 - cd) * NF * 2 + c;
    } else {
      continue;  // boundary without inflow data: exterior value = own trace
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      const double Fq = F[q];
      if (Fq == 0.0) continue;
      const double* De = fD + (e * NF + q) * NBS;
      double o = 0.0;
#pragma unroll
      for (int m = 0; m < NBS; ++m) o = fma(w[m], De[m], o);
      double x;
      if (cd >= 0) {
        double Dn[NBS];   // per-lane row (the neighbour's local edge): 16-byte LDS
        row_load<NBS>(Dn, s_fD + (e2 * NF + (NF - 1 - q)) * NBS);
        x = 0.0;
#pragma unroll
        for (int m = 0; m < NBS; ++m) x = fma(wn[m], Dn[m], x);
      } else {
        x = __ldg(infl + 2 * q);
      }
      const double jmp = Fq * (x - o);
#pragma unroll
      for (int m = 0; m < NBS; ++m) r[m] = fma(jmp, De[m], r[m]);
    }
  }

  // ---- epilogue
  if (p.st.cres && active && mi < 0.0) {
    // curved element: hand the raw residual to curved_fixup_kernel
    double* cr = p.st.cres + (size_t)((int)(-mi) - 1) * NB + c * NBS;
#pragma unroll
    for (int j = 0; j < NBS; ++j) cr[j] = r[j];
  }
  const double cm = p.st.c * mi;
  if constexpr (MODE == MODE_SUBSTEP) {
    // the rows go back through the w tile and one bulk store (coalesced)
    double v[NBS];
    double chk = 0.0;
#pragma unroll
    for (int j = 0; j < NBS; ++j) {
      v[j] = fma(cm, r[j], w[j]);
      chk += v[j];
    }
    guard_finite(p.st.flag, chk);
    __syncthreads();   // every thread's facet loop is done reading the w tile
    if (active) {
      double* ws = s_w + (T - tb) * NB + c * NBS;
      if constexpr (NBS % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NBS / 2; ++j) reinterpret_cast<double2*>(ws)[j] = make_double2(v[2 * j], v[2 * j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < NBS; ++j) ws[j] = v[j];
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(p.out + (size_t)tb * NB, s_w, (uint32_t)(nel * NB * sizeof(double)));
      bulk_wait_read();
    }
  } else {
    if (!active) return;
    double* og = p.out + (size_t)T * NB + c * NBS;
    const double tm = -p.st.tau * mi;
    double acc = 0.0, chk = 0.0;
#pragma unroll
    for (int j = 0; j < NBS; ++j) {
      const double v = fma(p.st.b, xs[j], fma(cm, r[j], p.st.a * w[j]));
      og[j] = v;
      chk += v;
      const double res = fma(tm, r[j], xs[j] - w[j]);
      acc = fma(res, res, acc);
    }
    guard_finite(p.st.flag, chk);
    if (p.st.rn) p.st.rn[2 * (size_t)T + c] = acc;
  }
}

}  // namespace hdgc
