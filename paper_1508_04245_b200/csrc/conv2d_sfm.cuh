// Variant "sfm": the sum-factorised flux-difference apply of conv2d_sf.cuh
// with a MODAL frozen-velocity prep.
//
// conv2d_sf_kernel streams, every substep, the velocity data alpha / beta /
// gamma at the n x n collapsed points plus the inflow weights: 3n^2 + 3nf
// doubles per element (129 at k = 4, 1032 B — 4.3x the 240 B of w; ncu:
// 188 MB of DRAM traffic per cfg2 launch, 1.93x the algorithmic bytes).
// Here the prep keeps the velocity in modal form, per element
//   u_hat (NB) | div u_hat (NBS1) | |e_hat| u[e(k+1)+l] (3(k+1)) | (M^V)^{-1} (1)
// (56 doubles at k = 4, 448 B), and the substep kernel rebuilds alpha / beta /
// gamma row by row by sum factorisation (u is frozen over a
// substep batch, so this is the same quadrature-point data, re-derived in
// registers instead of re-read from HBM; "no matrix stored"):
//   row b: H0_i = sum_j u_hat_x,ij B_ij(b), H1_i (u_hat_y), Hd_i (div),
//          u0/u1/dq at point a = sum_i A_i(a) H_i,
//          alpha = w_p (u0 + xi u1)/(1 - y), beta = w_p u1, gamma = w_p dq.
// The inflow weights s_e(q) = w_q F_e(t_q) [F < 0], F = |e| sum_l u_el L_l(t_q)
// (SURVEY A.4), are rebuilt by the facet warp from the stored edge dofs.
//
// Work split: one CTA = EPB = 16 elements, three warps.  Warps 0 and 1 are
// volume warps, warp 2 the upwind-facet warp (the old two-warp split left
// the facet warp idle ~60% of every tile: volume ~1100 FMA per lane, facets
// ~450).  Lane l of any warp owns (element l/2, component l%2).  Volume warp v
// takes the collapsed rows [v n/2, (v+1) n/2); for each row the two lanes of
// an element each evaluate the velocity at half of the row's points into a
// per-warp smem row buffer (the modal H sums are computed by both), then both
// run the row's w contraction (sf_row, shared with conv2d_sf).  Volume warp
// 1 and the facet warp leave partial residuals in smem; warp 0 adds them,
// runs the epilogue and bulk-stores the tile.  No atomics: deterministic.
//
// DRAM bytes per element and substep: 448 (modal row) + 240 (w in) + 240
// (w out) + 12 (neighbour codes) = 940 B (cfg2: 123 MB per launch, 1.28x the
// pinned algorithmic B(k) = 736 B).
#pragma once
#include "conv2d_sf.cuh"

namespace hdgc {

template <int K>
struct SFM {
  using F = SF<K>;
  static constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NBS1 = F::NBS1, NF = F::NF;
  static constexpr int EPB = 16;
  // modal prep slots (per element), tile-blocked slot-major [tile][MP][EPB]
  static constexpr int S_UH = 0;                 // u_hat: x modes then y modes (NB)
  static constexpr int S_DV = NB;                // div u_hat in P_{k-1} (NBS1)
  static constexpr int S_FX = NB + NBS1;         // edge flux coefficients |e| u[e(k+1)+l] (3 NE)
  static constexpr int S_MI = S_FX + 3 * NE;     // (M^V)^{-1} = 2/detJ (curved: -(slot+1))
  static constexpr int MP = (S_MI + 2) & ~1;     // padded to 16-byte rows
  static constexpr int MTILE = MP * EPB;         // doubles per modal tile
  static constexpr int NVW = 2;                  // volume warps
  static constexpr int THREADS = 32 * (NVW + 1);
  static constexpr int RB = (N + 1) / 2;         // rows per volume warp (warp 1: N - RB)
  static constexpr int PA = (N + 1) / 2;         // points of a row evaluated by the c = 0 lane
  // smem (doubles): mbarrier | modal tile | w tile [EPB][NB] | halo [32][NBS] |
  //                 vpart [32][NBS] | abg rows [NVW][3][N][EPB] | R tables [3][RSTR]
  // MODAL = false: the same three-warp kernel on conv2d_sf's point prep tile
  // ([PREP][EPB]: alpha | beta | gamma | s), no row buffers
  template <bool MODAL>
  struct L {
    static constexpr int SM_BAR = 0;
    static constexpr int SM_MOD = 2;
    static constexpr int SM_W = SM_MOD + (MODAL ? MTILE : F::PREP_TILE);
    static constexpr int SM_HALO = SM_W + EPB * NB;
    static constexpr int SM_VPART = SM_HALO + 32 * NBS + ((32 * NBS) & 1);
    static constexpr int SM_ABG = SM_VPART + 32 * NBS + ((32 * NBS) & 1);
    static constexpr int ABG = 3 * N * EPB;        // one warp's row buffer
    static constexpr int SM_FD = SM_ABG + (MODAL ? NVW * ABG : 0);
    static constexpr int SMEM_DOUBLES = SM_FD + F::TAB_PAD;
  };
};

#if HDGC_ORDER >= 3
__constant__ double c_fw[SF<HDGC_ORDER>::NF];    // facet rule weights
#else
__constant__ double c_fw[1];
#endif

// ---------------------------------------------------------------------------
// modal prep: one CTA per 32 elements (two modal tiles).  [u_hat | div u_hat]
// = [coef ; divm] u is the DMMA stage of prep_tile2d_kernel (FP64 tensor
// cores, A fragments precomputed); then the 32 x MP modal rows are written
// tile-blocked and slot-major (coalesced 128-B segments).
template <int K>
__global__ void __launch_bounds__(32 * SF<K>::N)
prep_modal2d_kernel(const double* __restrict__ tab, const double* __restrict__ afrag, const double* __restrict__ u,
                    const double* __restrict__ minv, int nt, double* __restrict__ mprep) {
  using D = Dims<K>;
  using F = SF<K>;
  using S = SFM<K>;
  using P = PrepMma<K>;
  constexpr int N = F::N, NE = F::NE, NB = F::NB, LD = P::LD;
  constexpr int NTH = 32 * N;
  extern __shared__ __align__(16) double smp[];
  double* s_u = smp;                   // [KS*4][LD]: u transposed, zero rows j >= NB
  double* s_h = smp + P::KS * 4 * LD;  // [MT*8][LD]: u_hat | div u_hat
  hdgc_debug_prologue(smp, P::SMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T0 = blockIdx.x * 32;
  const int nel = min(32, nt - T0);
  {
    constexpr int LOADS = (32 * NB + NTH - 1) / NTH;
    double v[LOADS];
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = tid + r * NTH;
      v[r] = (i < 32 * NB && i / NB < nel) ? __ldg(u + (size_t)T0 * NB + i) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = tid + r * NTH;
      if (i < 32 * NB) s_u[(i % NB) * LD + i / NB] = v[r];
    }
  }
  for (int i = tid; i < (P::KS * 4 - NB) * 32; i += NTH) s_u[(NB + i / 32) * LD + (i & 31)] = 0.0;
  __syncthreads();
  for (int t = warp; t < P::MT * 4; t += N) {
    const int mt = t >> 2, n0 = (t & 3) * 8;
    const double* af = afrag + (size_t)mt * P::KS * 32 + lane;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < P::KS; ++ks)
      dmma_m8n8k4(d0, d1, __ldg(af + ks * 32), s_u[(ks * 4 + (lane & 3)) * LD + n0 + (lane >> 2)]);
    *reinterpret_cast<double2*>(s_h + (mt * 8 + (lane >> 2)) * LD + n0 + 2 * (lane & 3)) = make_double2(d0, d1);
  }
  __syncthreads();
  // slot-major write-out: thread (slot, element) pairs; lanes = consecutive elements
  double* out = mprep + (size_t)blockIdx.x * 2 * S::MTILE;
  for (int i = tid; i < S::MP * 32; i += NTH) {
    const int slot = i >> 5, e = i & 31;
    double v = 0.0;
    if (e < nel) {
      if (slot < S::S_FX) {
        v = s_h[slot * LD + e];                                   // u_hat | div u_hat
      } else if (slot < S::S_MI) {
        const int ed = (slot - S::S_FX) / NE;
        v = __ldg(tab + D::OFF_FLEN + ed) * s_u[(slot - S::S_FX) * LD + e];   // |e| u[e(k+1)+l]
      } else if (slot == S::S_MI) {
        v = __ldg(minv + T0 + e);
      }
    }
    out[(e >> 4) * S::MTILE + slot * S::EPB + (e & 15)] = v;
  }
}

// velocity on row b of the collapsed rule, points [a0, a1), into the warp's
// row buffer abg ([3][N][EPB], element column le): alpha | beta | gamma
template <int K>
__device__ __forceinline__ void sfm_velocity_row(const double* __restrict__ mod, int b, int a0, int a1,
                                                 double* abg) {
  using F = SF<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, EPB = SFM<K>::EPB;
  const double* C = sf_tab<K>();
  const double* Bb = C + F::C_B + b * NBS;
  double H0[NE], H1[NE], Hd[NE];
#pragma unroll
  for (int i = 0; i <= K; ++i) {
    double s0 = 0.0, s1 = 0.0, sd = 0.0;
#pragma unroll
    for (int j = 0; j <= K - i; ++j) {
      const int m = midx(i, j);
      const double bm = Bb[m];
      s0 = fma(mod[(SFM<K>::S_UH + m) * EPB], bm, s0);
      s1 = fma(mod[(SFM<K>::S_UH + NBS + m) * EPB], bm, s1);
      if (i + j < K) sd = fma(mod[(SFM<K>::S_DV + m) * EPB], bm, sd);
    }
    H0[i] = s0; H1[i] = s1; Hd[i] = sd;
  }
#pragma unroll
  for (int a = 0; a < N; ++a) {
    if (a < a0 || a >= a1) continue;
    double u0 = 0.0, u1 = 0.0, dq = 0.0;
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      const double Ai = C[F::C_A + a * NE + i];
      u0 = fma(Ai, H0[i], u0);
      u1 = fma(Ai, H1[i], u1);
      if (i < K) dq = fma(Ai, Hd[i], dq);
    }
    const int p = b * N + a;
    abg[a * EPB] = fma(C[F::C_PA + p], u0, C[F::C_PB + p] * u1);
    abg[(N + a) * EPB] = C[F::C_PW + p] * u1;
    abg[(2 * N + a) * EPB] = C[F::C_PW + p] * dq;
  }
}

// F_e(t_q) = sum_l fx[l] L_l(t_q) (fx = |e| u_e,l: u.n ds/dt)
template <int K>
__device__ __forceinline__ double sfm_flux(const double* fx, int q) {
  using F = SF<K>;
  const double* FL = fl_tab<K>();
  double a = 0.0;
#pragma unroll
  for (int l = 0; l < F::NE; ++l) a = fma(fx[l * SFM<K>::EPB], FL[q * F::NE + l], a);
  return a;
}

#ifdef HDGC_SFM_MINB
#define HDGC_SFM_MINB_OF(K) HDGC_SFM_MINB
#else
#define HDGC_SFM_MINB_OF(K) (K <= 4 ? 5 : 3)
#endif
#ifndef HDGC_SFM_WREG
#define HDGC_SFM_WREG 1   // volume warps keep their w_c column in registers (0: read it from smem)
#endif
template <int K, int MODE, bool MODAL>
__global__ void __launch_bounds__(SFM<K>::THREADS, HDGC_SFM_MINB_OF(K))
conv2d_sfm_kernel(SFParams p) {
  using F = SF<K>;
  using S = SFM<K>;
  using LY = typename SFM<K>::template L<MODAL>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NF = F::NF, EPB = S::EPB;
  extern __shared__ __align__(128) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + LY::SM_BAR);
  double* s_mod = sm + LY::SM_MOD;         // modal [MP][EPB] or point prep [PREP][EPB]
  double* s_w = sm + LY::SM_W;             // [EPB][NB]
  double* s_halo = sm + LY::SM_HALO;       // [32][NBS]: facet warp halo, then its partial r
  double* s_vpart = sm + LY::SM_VPART;     // [32][NBS]: volume warp 1's partial r
  double* s_fD = sm + LY::SM_FD;           // edge trace maps [3][RSTR]
  constexpr int TILE = MODAL ? S::MTILE : F::PREP_TILE;
  hdgc_debug_prologue(sm, LY::SMEM_DOUBLES);

  const int T0 = blockIdx.x * EPB;
  const int nel = min(EPB, p.nt - T0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bm = (uint32_t)(TILE * sizeof(double));
    const uint32_t bw = (uint32_t)(nel * NB * sizeof(double));
    const uint32_t bt = (uint32_t)(F::TAB_PAD * sizeof(double));
    mbar_arrive_expect_tx(bar, bm + bw + bt);
    bulk_g2s(s_mod, p.prep + (size_t)blockIdx.x * TILE, bm, bar);
    bulk_g2s(s_fD, p.ftab, bt, bar);
    pdl_wait();   // w is the previous update kernel's output (PDL launch in a substep batch)
    bulk_g2s(s_w, p.w + (size_t)T0 * NB, bw, bar);
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int le = lane >> 1;
  const int c = lane & 1;
  const bool active = le < nel;
  const int lc = active ? le : 0;          // column of this lane's element in the tiles
  const int T = T0 + lc;
  const double* mod = s_mod + lc;          // modal column (slot j at mod[j * EPB])
  double r[NBS];
#pragma unroll
  for (int m = 0; m < NBS; ++m) r[m] = 0.0;

  if (warp < S::NVW) {
    // ===================== volume warps =====================
    pdl_wait();
    const int stopped = MODE == MODE_STAGE ? stage_stop_flag(p.st) : 0;   // converged Richardson iteration
    pdl_trigger();
    mbar_wait(bar, 0);
    if (stopped) return;
    const double* wc = s_w + lc * NB + c * NBS;
    const int b0 = warp == 0 ? 0 : S::RB, b1 = warp == 0 ? S::RB : N;
    auto rows = [&](const auto& wv) {
      if constexpr (MODAL) {
        double* abg = sm + LY::SM_ABG + warp * LY::ABG;
        const int a0 = c == 0 ? 0 : S::PA, a1 = c == 0 ? S::PA : N;
#pragma unroll 1
        for (int b = b0; b < b1; ++b) {
          if (active) sfm_velocity_row<K>(mod, b, a0, a1, abg + lc);
          __syncwarp();
          const double* al = abg + lc;
          sf_row<K>(wv, al, al + N * EPB, al + 2 * N * EPB, b, r);
          __syncwarp();   // the row buffer is refilled for the next row
        }
      } else {
#pragma unroll 1
        for (int b = b0; b < b1; ++b)
          sf_row<K>(wv, mod + (F::P_AL + b * N) * EPB, mod + (F::P_BE + b * N) * EPB,
                    mod + (F::P_GA + b * N) * EPB, b, r);
      }
    };
    double wo[NBS];
    if (HDGC_SFM_WREG) {
#pragma unroll
      for (int m = 0; m < NBS; ++m) wo[m] = wc[m];
      rows(wo);
    } else {
      rows(wc);
    }
    if (warp == 1) {
#pragma unroll
      for (int m = 0; m < NBS; ++m) s_vpart[lane * NBS + m] = r[m];
      asm volatile("bar.arrive 1, %0;\n" ::"n"(S::THREADS) : "memory");   // (A) partial ready
      return;
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(S::THREADS) : "memory");   // (A) all partials ready
    if (!HDGC_SFM_WREG) {
#pragma unroll
      for (int m = 0; m < NBS; ++m) wo[m] = wc[m];
    }
    double racc = 0.0;   // STAGE: this lane's residual sum of squares
    if (active) {
      const double mi = (MODE == MODE_SUBSTEP || MODE == MODE_STAGE)
                            ? (MODAL ? mod[S::S_MI * EPB] : __ldg(p.minv + T)) : 0.0;
      const double* part = s_halo + lane * NBS;
      const double* vp = s_vpart + lane * NBS;
      double* wo_s = s_w + le * NB + c * NBS;
#pragma unroll
      for (int m = 0; m < NBS; ++m) r[m] += vp[m];
      if ((MODE == MODE_SUBSTEP || MODE == MODE_STAGE) && mi < 0.0 && p.st.cres) {
        // curved element: hand the raw residual to curved_fixup_kernel
        double* cr = p.st.cres + (size_t)((int)(-mi) - 1) * NB + c * NBS;
#pragma unroll
        for (int m = 0; m < NBS; ++m) cr[m] = r[m] + part[m];
      }
      if (MODE == MODE_SUBSTEP) {
        const double cm = p.st.c * mi;
        double chk = 0.0;
#pragma unroll
        for (int m = 0; m < NBS; ++m) {
          const double v = fma(cm, r[m] + part[m], wo[m]);
          wo_s[m] = v;
          chk += v;
        }
        guard_finite(p.st.flag, chk);
      } else if (MODE == MODE_STAGE) {
        racc = stage_x(p.st, mi, p.st.c * mi, r, part, wo, wo_s, p.st.x + (size_t)T * NB + c * NBS,
                       p.st.rn ? p.st.rn + 2 * (size_t)T + c : nullptr);
      } else {
#pragma unroll
        for (int m = 0; m < NBS; ++m) wo_s[m] = r[m] + part[m];
      }
    }
    fence_proxy_async();
    __syncwarp();
    if (threadIdx.x == 0) {
      bulk_s2g(p.out + (size_t)T0 * NB, s_w, (uint32_t)(nel * NB * sizeof(double)));
      bulk_wait_read();
    }
    if (MODE == MODE_STAGE && p.st.rpart) rich_cta_partial(p.st, racc, (int)blockIdx.x);
  } else {
    // ===================== facet warp =====================
    int codes[3];
#pragma unroll
    for (int ed = 0; ed < 3; ++ed) codes[ed] = active ? __ldg(p.code + (size_t)T * 3 + ed) : -1;
    pdl_wait();   // halo gathers below read the previous kernel's w
    const int stopped = MODE == MODE_STAGE ? stage_stop_flag(p.st) : 0;
    pdl_trigger();
    mbar_wait(bar, 0);
    if (stopped) return;
    const double* wc = s_w + lc * NB + c * NBS;
    const double* fx = mod + S::S_FX * EPB;          // edge flux coefficients, edge e at fx[e NE EPB]
    // inflow edges of this element: any point with F < 0 (modal: F from the edge dofs)
    bool inflow_edge[3];
#pragma unroll
    for (int ed = 0; ed < 3; ++ed) {
      bool any = false;
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        if constexpr (MODAL) any |= sfm_flux<K>(fx + ed * NE * EPB, q) < 0.0;
        else any |= mod[(F::P_S + ed * NF + q) * EPB] != 0.0;
      }
      inflow_edge[ed] = any && active;
    }
    double* halo = s_halo + lane * NBS;
    int halo_edge = -1;
    if (active) {
#pragma unroll
      for (int ed = 0; ed < 3; ++ed) {
        const int code = codes[ed];
        if (code < 0 || halo_edge >= 0 || !inflow_edge[ed]) continue;
        const int nbT = code >> 2;
        if (nbT >= T0 && nbT < T0 + nel) continue;
        halo_edge = ed;
        const double* g = p.w + (size_t)nbT * NB + c * NBS;
#pragma unroll
        for (int m = 0; m < NBS; ++m) cp_async8(halo + m, g + m);
      }
    }
    if (halo_edge >= 0) cp_async_wait_all();
    __shared__ double zero_row_m[NBS];
    for (int m = lane; m < NBS; m += 32) zero_row_m[m] = 0.0;
    __syncwarp();
    unsigned emask = 0;
#pragma unroll
    for (int ed = 0; ed < 3; ++ed) {
      const bool has_ext = codes[ed] >= 0 || p.inflow != nullptr;   // else exterior = own trace
      if (inflow_edge[ed] && has_ext) emask |= 1u << ed;
    }
    const int nmine = __popc(emask);
    const int nmax = __reduce_max_sync(0xffffffffu, (unsigned)nmine);
    // jumps in the edge's own P_k basis through the trace maps R_e (conv2d_sf.cuh)
    const double* FL = fl_tab<K>();
#pragma unroll 1
    for (int j = 0; j < nmax; ++j) {
      const bool on = j < nmine;
      const int ed = on ? __ffs(emask) - 1 : 0;
      if (on) emask &= emask - 1;
      const int code = ed == 0 ? codes[0] : (ed == 1 ? codes[1] : codes[2]);
      const double* src = zero_row_m;
      const double* infl = nullptr;
      int e2 = 0;
      if (on && code >= 0) {
        const int nbT = code >> 2;
        e2 = code & 3;
        src = (nbT >= T0 && nbT < T0 + nel) ? s_w + (nbT - T0) * NB + c * NBS
              : (ed == halo_edge) ? halo : p.w + (size_t)nbT * NB + c * NBS;
      } else if (on) {
        infl = p.inflow + (size_t)(-1 - code) * NF * 2 + c;
      }
      const double* Re = s_fD + ed * F::RSTR;
      const double* Rn = s_fD + e2 * F::RSTR;
      double dl[NE];
#pragma unroll
      for (int l = 0; l < NE; ++l) dl[l] = 0.0;
#pragma unroll 3
      for (int m = 0; m < NBS; ++m) {
        const double wn = src[m], wm = wc[m];
#pragma unroll
        for (int l = 0; l < NE; ++l) {
          const double tn = (l & 1) ? -wn : wn;
          dl[l] = fma(tn, Rn[l * NBS + m], fma(-wm, Re[l * NBS + m], dl[l]));
        }
      }
      const double* fxe = fx + ed * NE * EPB;
      double fxr[NE];
#pragma unroll
      for (int l = 0; l < NE; ++l) fxr[l] = MODAL ? fxe[l * EPB] : 0.0;
      double rho[NE];
#pragma unroll
      for (int l = 0; l < NE; ++l) rho[l] = 0.0;
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        double Fq = 0.0, J = 0.0;
#pragma unroll
        for (int l = 0; l < NE; ++l) {
          if (MODAL) Fq = fma(fxr[l], FL[q * NE + l], Fq);
          J = fma(dl[l], FL[q * NE + l], J);
        }
        double sq;
        if constexpr (MODAL) sq = (on && Fq < 0.0) ? c_fw[q] * Fq : 0.0;
        else sq = on ? mod[(F::P_S + ed * NF + q) * EPB] : 0.0;
        if (infl != nullptr && sq != 0.0) J += __ldg(infl + 2 * q);
        const double sj = sq * J;
#pragma unroll
        for (int l = 0; l < NE; ++l) rho[l] = fma(sj, FL[q * NE + l], rho[l]);
      }
#pragma unroll
      for (int m = 0; m < NBS; ++m) {
        double acc = r[m];
#pragma unroll
        for (int l = 0; l < NE; ++l) acc = fma(Re[l * NBS + m], rho[l], acc);
        r[m] = acc;
      }
    }
    __syncwarp();          // halo reads of all lanes done before the partials overwrite it
#pragma unroll
    for (int m = 0; m < NBS; ++m) halo[m] = r[m];
    asm volatile("bar.arrive 1, %0;\n" ::"n"(S::THREADS) : "memory");   // (A)
  }
}

}  // namespace hdgc
