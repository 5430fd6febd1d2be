// Variant "sf": sum-factorised flux-difference apply for k >= 3 on the
// collapsed (Duffy) volume rule, n = (3k+1)/2 points per direction.
//
// The convecting velocity is frozen over an apply and over a whole substep
// batch, so everything that depends on u alone is
// evaluated once per batch (prep_tile2d_kernel, prep_fused2d_kernel, or modal_rows_kernel + prep_rows2d_kernel) into a
// per-element "prep row":
//   alpha(p) = w_p (u0 + xi_p u1) / (1 - y_p),   beta(p) = w_p u1,
//   gamma(p) = w_p div u_hat                      at the n^2 volume points,
//   s_e(q)   = w_q F_e(t_q) if F_e(t_q) < 0 else 0   (inflow points, 3 nf)
// (u_hat = Piola-free reference velocity, F = u.n ds/dt from the edge dofs,
// SURVEY.md A.3/A.4).  This is quadrature-point data, not an assembled
// matrix.  The per-substep kernel then only moves w:
//
//   r_c[ij] = sum_b B_ij(b) sum_a A_i(a) g_c(a,b)
//   g_c     = alpha d_xi w_c + beta d_y|xi w_c + gamma w_c
//           ( = w_p (u.grad w_c + w_c div u) at the point, flux-difference
//             form, see conv2d_thread.cuh )
//   w_c and its derivatives at the points by sum factorisation: per row b
//   H_i = sum_j w_c,ij B_ij(b), H'_i = sum_j w_c,ij dB_ij/dy(b), then
//   w = sum_i A_i(a) H_i, d_xi w = sum_i A'_i(a) H_i, d_y|xi w = sum_i A_i(a) H'_i.
//   + sum_e sum_{q inflow} s_e(q) (w_ext - w_own)_c(q) D_m(x_e(q))
//
// FMA per element (k=4): volume 2 x 6 x (30 + 6 x 23 + 15) = 2196 plus the
// inflow facet points, against 7395 for the pinned direct form.
//
// Work split: one CTA = EPB elements, two threads per element (one per output
// component c); prep rows and w (interleaved (m, c)) staged in shared memory;
// A/A'/B/B' tables in the constant bank (uniform operands).
#pragma once
#include "common.cuh"

namespace hdgc {

__host__ __device__ constexpr int midx(int i, int j) { return (i + j) * (i + j + 1) / 2 + j; }

template <int K>
struct SF {
  static constexpr int N = (3 * K + 1) / 2;   // collapsed points per direction
  static constexpr int NQ = N * N;
  static constexpr int NE = K + 1;
  static constexpr int NBS = (K + 1) * (K + 2) / 2;
  static constexpr int NB = 2 * NBS;
  static constexpr int NBS1 = K * (K + 1) / 2;
  static constexpr int NF = (3 * K + 3) / 2;
  // constant-bank table layout (doubles)
  static constexpr int C_A = 0;                    // [N][K+1]  P_i(2 xi_a - 1)
  static constexpr int C_AD = C_A + N * NE;        // [N][K+1]  d/dxi
  static constexpr int C_B = C_AD + N * NE;        // [N][NBS]  c_ij (1-y)^i P_j^(2i+1,0)(2y-1)
  static constexpr int C_BD = C_B + N * NBS;       // [N][NBS]  d/dy at fixed xi
  static constexpr int C_PA = C_BD + N * NBS;      // [NQ] w_p / (1 - y_p)
  static constexpr int C_PB = C_PA + NQ;           // [NQ] w_p xi_p / (1 - y_p)
  static constexpr int C_PW = C_PB + NQ;           // [NQ] w_p
  static constexpr int C_TOTAL = C_PW + NQ;
  // prep data per element: alpha | beta | gamma | s (PREP slots).  Global layout is
  // tile-blocked and slot-major, prep[tile][slot][e] with e < EPB, so that the
  // prep kernels write coalesced, a tile is one contiguous bulk copy, and lanes
  // of the substep kernel read consecutive addresses (conflict-free).
  static constexpr int P_AL = 0;
  static constexpr int P_BE = NQ;
  static constexpr int P_GA = 2 * NQ;
  static constexpr int P_S = 3 * NQ;
  static constexpr int PREP = 3 * NQ + 3 * NF;
  static constexpr int EPB = 16;                    // elements per CTA
  static constexpr int THREADS = 4 * EPB;            // two warps: volume | facets
#ifdef HDGC_FACET_ROWS
  static constexpr int FACET_ROWS = HDGC_FACET_ROWS;
#else
  // volume rows taken by the facet warp to balance the two warps (measured per
  // k at 131k triangles with the mirror-pair rows and the one-round halo traces:
  // k=3 0/1/2 rows 33.4/33.6/39.6 us, k=4 0/1/2 rows 46.0/46.8/54.6, k=6 1/2/3 rows
  // 159/142/137.6)
  static constexpr int FACET_ROWS = K == 3 ? 1 : K == 4 ? 1 : K == 6 ? 3 : (K == 5 ? 1 : 0);
#endif
  static constexpr int PREP_TILE = PREP * 16;      // doubles per tile (EPB = 16)
#ifdef HDGC_SF_RING
  static constexpr bool RING = HDGC_SF_RING;
#else
  // high orders: stream the prep tile row by row through a two-slot smem ring
  // (cp.async) instead of staging it whole, and keep w in smem instead of
  // registers: the whole-tile prep (60 KB at k = 8) and the register copy of w
  // cost occupancy and spills there
  static constexpr bool RING = K >= 7;
#endif
#ifdef HDGC_SMEM_BT
  static constexpr bool SMBT = RING || HDGC_SMEM_BT;
#else
  static constexpr bool SMBT = RING;
#endif
#ifdef HDGC_W_SMEM
  static constexpr bool WSMEM = HDGC_W_SMEM;
#else
  // volume rows read w_c from the smem tile in every row instead of a register
  // copy (k=4: 121 registers without spills, 54.3 vs 55.5 us)
  static constexpr bool WSMEM = K == 4;
#endif
#ifdef HDGC_SYM
  static constexpr bool SYM = HDGC_SYM;
#else
  // mirror-pair evaluation of the xi direction (sf_row) and of the facet points:
  // k=3 34.7 vs 37.4 us, k=4 49.9 vs 55.0, k=6 146 vs 160 at 131k triangles; k=5
  // (work-list facet stage, 186 registers) 119.8 vs 105.7: off there
  static constexpr bool SYM = !RING && K != 5;
#endif
#ifdef HDGC_OWNF
  static constexpr bool OWNF = HDGC_OWNF;
#else
  // facets_v2: own edge traces computed by the facet warp (no cross-warp barrier)
  // instead of the volume warp
  static constexpr bool OWNF = false;
#endif
  static constexpr int RING_SLOT = 3 * N * 16;     // alpha | beta | gamma of one row, [3][N][16]
  // smem (doubles): mbarrier | prep tile [PREP][EPB] or ring [2][3][N][EPB] |
  //                 w tile [EPB][NB] | halo [THREADS][NBS] | fD [3][NF][NBS]
  static constexpr int SM_BAR = 0;
  static constexpr int SM_PREP = 2;
  static constexpr int SM_W = SM_PREP + (RING ? 2 * RING_SLOT : PREP_TILE);
  static constexpr int SM_HALO = SM_W + EPB * NB;
#ifdef HDGC_FV2
  static constexpr bool FV2 = HDGC_FV2;
#else
  // structured-trace facet stage (facets_v2 below).  Measured at 131k triangles
  // against the per-lane work-list stage it replaces: k=3 37.0 vs 44.0 us, k=4
  // 54.3 vs 59.4, k=6 165 vs 186; k=5 118.6 vs 105.6 (its 208 registers cost the
  // fifth CTA per SM), k=7 356 vs 323, k=8 547 vs 458 (ring mode): those keep
  // the work-list stage.
  static constexpr bool FV2 = K == 3 || K == 4 || K == 6;
#endif
  // per-lane stride of the halo / partial-residual / published-trace rows (odd:
  // the 32 lanes' rows spread over all banks)
  static constexpr int HSTR = FV2 ? (((NBS > 3 * NE) ? NBS : 3 * NE) | 1) : NBS;
  static constexpr int SM_TR = SM_HALO + 32 * HSTR + ((32 * HSTR) & 1);   // FV2: traces [32][HSTR]
  static constexpr int SM_FD = SM_TR + (FV2 ? 32 * HSTR + ((32 * HSTR) & 1) : 0);
  // smem edge trace maps R[3][NE][NBS], per-edge stride odd (bank spread across lanes)
  static constexpr int RSTR = (NE * NBS) | 1;
  static constexpr int TAB = 3 * NF * NBS;          // constant-bank facet table size (fD)
  static constexpr int TAB_PAD = (3 * RSTR + 1) & ~1; // smem R table, 16-B multiple for the bulk copy
  static constexpr int TAB_SM = FV2 ? 0 : TAB_PAD;    // FV2 reads the trace maps from the constant bank
  // ring mode: B / B' row tables interleaved [N][NBS](B, B') in smem (uniform LDS.128
  // instead of runtime-indexed constant loads, which ptxas hoists into registers)
  static constexpr int SM_BT = SM_FD + TAB_SM;
  static constexpr int SMEM_DOUBLES = SM_BT + (SMBT ? 2 * N * NBS : 0);
  // STAGE mode adds the x tile [EPB][NB] (bulk-copied with w) after SMEM_DOUBLES
  static constexpr int SM_X = SMEM_DOUBLES;
#ifndef HDGC_XTILE
#define HDGC_XTILE 1
#endif
  static constexpr bool XTILE = HDGC_XTILE;
  __host__ __device__ static constexpr int smem_doubles(int mode) { return SMEM_DOUBLES + (mode == 3 && XTILE ? EPB * NB : 0); }
};

// The constant-bank tables of the order compiled in this translation unit
// (order_k<K>.cu defines HDGC_ORDER before including the kernels).
#ifndef HDGC_ORDER
#error "define HDGC_ORDER (the order k of this translation unit) before including conv2d_sf.cuh"
#endif
#if HDGC_ORDER >= 3
__constant__ double c_sf[SF<HDGC_ORDER>::C_TOTAL];
__constant__ double c_fd[SF<HDGC_ORDER>::TAB];   // Dubiner traces fD[3][NF][NBS]
__constant__ double c_fl[SF<HDGC_ORDER>::NF * SF<HDGC_ORDER>::NE];   // Legendre at facet points
// structured edge trace maps (facets_v2): R_0[i][m(i,j)] (the only non-zeros of
// edge 0) and R_1[l][m] (zero for l > i + j); R_2[l][m] = (-1)^(i+l) R_1[l][m]
__constant__ double c_r0[SF<HDGC_ORDER>::NBS];
__constant__ double c_r1[SF<HDGC_ORDER>::NE * SF<HDGC_ORDER>::NBS];
// the same non-zeros in order of use (edge_traces / edge_test), read in pairs
__constant__ __align__(16) double c_tr[(SF<HDGC_ORDER>::NBS + (SF<HDGC_ORDER>::NE) * (SF<HDGC_ORDER>::NE + 1) * (2 * SF<HDGC_ORDER>::NE + 1) / 6 + 1) & ~1];
// fused prep (k <= 6): [coef ; divm] (NB + NBS1 rows x NB) | fL (NF x NE) | fw (NF) | flen (3)
#define HDGC_CM_FUSED (HDGC_ORDER <= 4)
#if HDGC_CM_FUSED
__constant__ double c_cm[(SF<HDGC_ORDER>::NB + SF<HDGC_ORDER>::NBS1) * SF<HDGC_ORDER>::NB +
                         SF<HDGC_ORDER>::NF * SF<HDGC_ORDER>::NE + SF<HDGC_ORDER>::NF + 3];
#else
__constant__ double c_cm[1];
#endif
#else
__constant__ double c_sf[1];
__constant__ double c_fd[1];
__constant__ double c_fl[1];
__constant__ double c_r0[1];
__constant__ double c_r1[1];
__constant__ __align__(16) double c_tr[2];
#define HDGC_CM_FUSED 0
__constant__ double c_cm[1];
#endif

template <int K> __device__ __forceinline__ const double* sf_tab() {
  static_assert(K == HDGC_ORDER, "sum-factorisation tables are per translation unit");
  return c_sf;
}
template <int K> __device__ __forceinline__ const double* fl_tab() {
  static_assert(K == HDGC_ORDER, "facet tables are per translation unit");
  return c_fl;
}
template <int K> __device__ __forceinline__ const double* fd_tab() {
  static_assert(K == HDGC_ORDER, "facet tables are per translation unit");
  return c_fd;
}

// ---------------------------------------------------------------------------
// fused prep (k <= 4), one thread per element: modal u_hat = coef u and
// div = divm u with the matrices as constant-bank operands, then alpha/beta/
// gamma at the n x n points by sum factorisation of the velocity (per row b:
// H_i = sum_j u_hat_ij B_ij(b), then sum_i A_i(a) H_i), and the inflow weights.
template <int K>
__global__ void __launch_bounds__(128)
prep_fused2d_kernel(const double* __restrict__ u, int nt, double* __restrict__ prep) {
  pdl_trigger();   // the update kernel after a prep may launch now (PDL, SFParams::prep_dep)
  using F = SF<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NBS1 = F::NBS1, NF = F::NF;
  constexpr int O_FL = (NB + NBS1) * NB, O_FW = O_FL + NF * NE, O_FLEN = O_FW + NF;
  const double* CM = c_cm;
  const double* C = sf_tab<K>();
  const int T = blockIdx.x * blockDim.x + threadIdx.x;
  if (T >= nt) return;
  double* out = prep + (size_t)(T / 16) * F::PREP_TILE + (T % 16);   // slot stride 16
  double uh[NB], dv[NBS1 > 0 ? NBS1 : 1];
  {
    double x[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) x[j] = __ldg(u + (size_t)T * NB + j);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        double a = 0.0;
#pragma unroll
        for (int l = 0; l < NE; ++l) a = fma(x[e * NE + l], CM[O_FL + q * NE + l], a);
        const double Fq = a * CM[O_FLEN + e];
        out[(F::P_S + e * NF + q) * 16] = Fq < 0.0 ? CM[O_FW + q] * Fq : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) a = fma(CM[i * NB + j], x[j], a);
      uh[i] = a;
    }
#pragma unroll
    for (int i = 0; i < NBS1; ++i) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) a = fma(CM[(NB + i) * NB + j], x[j], a);
      dv[i] = a;
    }
  }
#pragma unroll 1
  for (int b = 0; b < N; ++b) {
    const double* Bb = C + F::C_B + b * NBS;
    double H0[NE], H1[NE], Hd[NE];
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      double s0 = 0.0, s1 = 0.0, sd = 0.0;
#pragma unroll
      for (int j = 0; j <= K - i; ++j) {
        const int m = midx(i, j);
        s0 = fma(uh[m], Bb[m], s0);
        s1 = fma(uh[NBS + m], Bb[m], s1);
        if (i + j < K) sd = fma(dv[m], Bb[m], sd);
      }
      H0[i] = s0; H1[i] = s1; Hd[i] = sd;
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double u0 = 0.0, u1 = 0.0, dq = 0.0;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const double Ai = C[F::C_A + a * NE + i];
        u0 = fma(Ai, H0[i], u0);
        u1 = fma(Ai, H1[i], u1);
        if (i < K) dq = fma(Ai, Hd[i], dq);
      }
      const int p = b * N + a;
      out[(F::P_AL + p) * 16] = fma(C[F::C_PA + p], u0, C[F::C_PB + p] * u1);
      out[(F::P_BE + p) * 16] = C[F::C_PW + p] * u1;
      out[(F::P_GA + p) * 16] = C[F::C_PW + p] * dq;
    }
  }
}

// ---------------------------------------------------------------------------
// prep, stage 2 (stage 1 = modal rows u_hat | div u_hat, modal_rows_kernel): one CTA
// per tile of 16 elements, one thread per (element, collapsed row b).  The
// tile's modal rows are staged in smem; thread (e, b) evaluates the velocity on
// row b by sum factorisation (H_i = sum_j u_ij B_ij(b), values via A_i(xi_a))
// and writes alpha/beta/gamma of its N points; threads with b < 3 also write
// the inflow weights of edge b.  Writes are tile-blocked and slot-major, so
// the 16 lanes of an element group store consecutive addresses.
template <int K>
__global__ void __launch_bounds__(16 * SF<K>::N)
prep_rows2d_kernel(const double* __restrict__ tab, const double* __restrict__ u,
                   const double* __restrict__ modal, int nt, double* __restrict__ prep) {
  pdl_trigger();   // the update kernel after a prep may launch now (PDL, SFParams::prep_dep)
  using D = Dims<K>;
  using F = SF<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NBS1 = F::NBS1, NF = F::NF;
  constexpr int NR = NB + NBS1;
  __shared__ double s_mod[16 * NR];
  const int T0 = blockIdx.x * 16;
  const int nel = min(16, nt - T0);
  {
    // every load of this thread in flight before the smem stores
    constexpr int LOADS = (16 * NR + 16 * N - 1) / (16 * N);
    double v[LOADS];
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = threadIdx.x + r * 16 * N;
      v[r] = i < nel * NR ? __ldg(modal + (size_t)T0 * NR + i) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = threadIdx.x + r * 16 * N;
      if (i < nel * NR) s_mod[i] = v[r];
    }
  }
  __syncthreads();
  const int e = threadIdx.x & 15;
  const int b = threadIdx.x >> 4;
  if (e >= nel) return;
  const double* C = sf_tab<K>();
  const double* mr = s_mod + e * NR;
  double* out = prep + (size_t)blockIdx.x * F::PREP_TILE + e;
  {
    const double* Bb = C + F::C_B + b * NBS;
    double H0[NE], H1[NE], Hd[NE];
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      double s0 = 0.0, s1 = 0.0, sd = 0.0;
#pragma unroll
      for (int j = 0; j <= K - i; ++j) {
        const int m = midx(i, j);
        s0 = fma(mr[m], Bb[m], s0);
        s1 = fma(mr[NBS + m], Bb[m], s1);
        if (i + j < K) sd = fma(mr[NB + m], Bb[m], sd);
      }
      H0[i] = s0; H1[i] = s1; Hd[i] = sd;
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double u0 = 0.0, u1 = 0.0, dq = 0.0;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const double Ai = C[F::C_A + a * NE + i];
        u0 = fma(Ai, H0[i], u0);
        u1 = fma(Ai, H1[i], u1);
        if (i < K) dq = fma(Ai, Hd[i], dq);
      }
      const int p = b * N + a;
      out[(F::P_AL + p) * 16] = fma(C[F::C_PA + p], u0, C[F::C_PB + p] * u1);
      out[(F::P_BE + p) * 16] = C[F::C_PW + p] * u1;
      out[(F::P_GA + p) * 16] = C[F::C_PW + p] * dq;
    }
  }
  if (b < 3) {
    // inflow weights of edge b: F = |e| sum_l u[b(k+1)+l] L_l(t_q)
    const double* ue = u + (size_t)(T0 + e) * NB + b * NE;
    double x[NE];
#pragma unroll
    for (int l = 0; l < NE; ++l) x[l] = __ldg(ue + l);
    const double len = __ldg(tab + D::OFF_FLEN + b);
    const double* FL = fl_tab<K>();
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      double a = 0.0;
#pragma unroll
      for (int l = 0; l < NE; ++l) a = fma(x[l], FL[q * NE + l], a);
      const double Fq = a * len;
      out[(F::P_S + b * NF + q) * 16] = Fq < 0.0 ? __ldg(tab + D::OFF_FW + q) * Fq : 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// tile prep (k = 3..6): one CTA per 32 elements (two prep tiles), one warp per
// collapsed row b.
// Stage 1, the modal rows [u_hat | div u_hat] = M u with M = [coef ; divm]
// (NR x NB), is a small dense GEMM per CTA: (NR x NB) x (NB x 32 elements), on
// the FP64 tensor cores (mma.sync m8n8k4 f64, SASS DMMA).  A operands are
// precomputed host-side in fragment order (PrepMma::afrag, one coalesced
// 256-B load per fragment, L1-resident across CTAs); B operands come from u
// staged transposed in smem ([j][e], row stride 40 doubles: the 4 k-rows x 8
// columns of a fragment load hit 2 wavefronts, the minimum); D fragments go to
// s_h [i][e] (row stride 40: conflict-free double2 stores).  The LDS-fed DFMA
// version of this stage was LDS-bandwidth bound (two LDS per FMA).
// Stage 2: warp b evaluates the velocity on collapsed row b by sum
// factorisation and writes alpha/beta/gamma of its N points; warps 0..2 also
// write the inflow weights of edge 0..2.  Table operands are warp-uniform
// (constant bank); the slot-major prep writes of a warp are two full 128-B
// segments.
template <int K>
struct PrepMma {
  static constexpr int NB = SF<K>::NB, NR = SF<K>::NB + SF<K>::NBS1;
  static constexpr int MT = (NR + 7) / 8;      // 8-row tiles of M
  static constexpr int KS = (NB + 3) / 4;      // k-steps of 4
  static constexpr int LD = 40;                // smem row stride (doubles) of s_u and s_h
  static constexpr int AFRAG = MT * KS * 32;   // doubles of precomputed A fragments
  static constexpr int SMEM = KS * 4 * LD + MT * 8 * LD;   // s_u [KS*4][LD] | s_h [MT*8][LD]
};

template <int K>
#ifndef HDGC_PREP_CPASYNC
#define HDGC_PREP_CPASYNC 0
#endif
// resident CTAs per SM (register caps), measured on the cfg2-size single apply:
// k=4 4 / 5 / 6 CTAs (76 / 64 / 56 registers, no spills) 93.2 / 89.2 / 87.1 us
#ifndef HDGC_PREP_MINB4
#define HDGC_PREP_MINB4 6
#endif
// k=5 3 / 4 / 5 CTAs 185.8 / 183.3 / 184.4 us, k=6 3 / 4 / 5 CTAs 250.7 / 255.0 / 318 (spills),
// k=7, 8 2 / 3 CTAs 541 / 554 and 785 / 820
#ifndef HDGC_PREP_MINB5
#define HDGC_PREP_MINB5 4
#endif
#ifndef HDGC_PREP_MINB56
#define HDGC_PREP_MINB56 3
#endif
#ifndef HDGC_PREP_MINB78
#define HDGC_PREP_MINB78 2
#endif
__global__ void __launch_bounds__(32 * SF<K>::N, K == 4 ? HDGC_PREP_MINB4 : K == 5 ? HDGC_PREP_MINB5 : (K <= 6 ? HDGC_PREP_MINB56 : HDGC_PREP_MINB78))
prep_tile2d_kernel(const double* __restrict__ tab, const double* __restrict__ afrag, const double* __restrict__ u,
                   int nt, double* __restrict__ prep) {
  pdl_trigger();   // the update kernel after a prep may launch now (PDL, SFParams::prep_dep)
  using D = Dims<K>;
  using F = SF<K>;
  using P = PrepMma<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NF = F::NF, LD = P::LD;
  constexpr int NTH = 32 * N;
  extern __shared__ __align__(16) double smp[];
  double* s_u = smp;                   // [KS*4][LD]: u transposed, zero rows j >= NB
  double* s_h = smp + P::KS * 4 * LD;  // [MT*8][LD]: u_hat | div u_hat (rows >= NR unused)
  hdgc_debug_prologue(smp, P::SMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T0 = blockIdx.x * 32;
  const int nel = min(32, nt - T0);
  {
    // all of this thread's u loads in flight before the first smem store (a
    // rolled load->store loop serialised the global latency: 40% of the stalls)
    constexpr int LOADS = (32 * NB + NTH - 1) / NTH;
#if HDGC_PREP_CPASYNC
    // straight into the transposed position with cp.async (no register round trip)
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = tid + r * NTH;
      if (i < 32 * NB) {
        if (i / NB < nel) cp_async8(&s_u[(i % NB) * LD + i / NB], u + (size_t)T0 * NB + i);
        else s_u[(i % NB) * LD + i / NB] = 0.0;
      }
    }
    cp_async_wait_all();
#else
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
#endif
  }
  for (int i = tid; i < (P::KS * 4 - NB) * 32; i += NTH) s_u[(NB + i / 32) * LD + (i & 31)] = 0.0;
  __syncthreads();
  // stage 1: MT row tiles of 8 x 32 over the warps; the four 8 x 8 column tiles of a
  // row tile share each A fragment and run as four independent DMMA chains (a
  // single chain per 8 x 8 tile serialised KS dependent DMMAs per tile)
  for (int mt = warp; mt < P::MT; mt += N) {
    const double* af = afrag + (size_t)mt * P::KS * 32 + lane;
    double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int ks = 0; ks < P::KS; ++ks) {
      const double a = __ldg(af + ks * 32);
      const double* bs = s_u + (ks * 4 + (lane & 3)) * LD + (lane >> 2);
#pragma unroll
      for (int nq = 0; nq < 4; ++nq) dmma_m8n8k4(d[nq][0], d[nq][1], a, bs[nq * 8]);
    }
#pragma unroll
    for (int nq = 0; nq < 4; ++nq)
      *reinterpret_cast<double2*>(s_h + (mt * 8 + (lane >> 2)) * LD + nq * 8 + 2 * (lane & 3)) =
          make_double2(d[nq][0], d[nq][1]);
  }
  const bool active = lane < nel;
  double* out = prep + (size_t)(blockIdx.x * 2 + (lane >> 4)) * F::PREP_TILE + (lane & 15);
  if (warp >= N - 3 && active) {
    // inflow weights of edge N-1-warp (the last warps: they have the fewest row
    // tiles in stage 1): F = |e| sum_l u[e(k+1)+l] L_l(t_q)
    const int ed = N - 1 - warp;
    const double len = __ldg(tab + D::OFF_FLEN + ed);
    const double* FL = fl_tab<K>();
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      double a = 0.0;
#pragma unroll
      for (int l = 0; l < NE; ++l) a = fma(s_u[(ed * NE + l) * LD + lane], FL[q * NE + l], a);
      const double Fq = a * len;
      out[(F::P_S + ed * NF + q) * 16] = Fq < 0.0 ? __ldg(tab + D::OFF_FW + q) * Fq : 0.0;
    }
  }
  __syncthreads();
  // stage 2: velocity on row b = warp
  const int b = warp;
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
      s0 = fma(s_h[m * LD + lane], bm, s0);
      s1 = fma(s_h[(NBS + m) * LD + lane], bm, s1);
      if (i + j < K) sd = fma(s_h[(NB + m) * LD + lane], bm, sd);
    }
    H0[i] = s0; H1[i] = s1; Hd[i] = sd;
  }
  if (!active) return;
#pragma unroll
  for (int a = 0; a < N; ++a) {
    double u0 = 0.0, u1 = 0.0, dq = 0.0;
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      const double Ai = C[F::C_A + a * NE + i];
      u0 = fma(Ai, H0[i], u0);
      u1 = fma(Ai, H1[i], u1);
      if (i < K) dq = fma(Ai, Hd[i], dq);
    }
    const int p = b * N + a;
    out[(F::P_AL + p) * 16] = fma(C[F::C_PA + p], u0, C[F::C_PB + p] * u1);
    out[(F::P_BE + p) * 16] = C[F::C_PW + p] * u1;
    out[(F::P_GA + p) * 16] = C[F::C_PW + p] * dq;
  }
}

// ---------------------------------------------------------------------------
// per-apply / per-substep kernel
struct SFParams {
  const double* __restrict__ prep;    // tile-blocked [tile][PREP][16]
  const double* __restrict__ w;       // (NT, NB)
  const double* __restrict__ inflow;  // (NBF, NF, 2) or nullptr
  const int32_t* __restrict__ code;   // (NT, 3)
  const double* __restrict__ minv;    // (NT,)
  const double* __restrict__ ftab;    // fD[3][NF][NBS] (global copy)
  double* __restrict__ out;           // (NT, NB)
  StageParams st;
  int nt;
  // 1: launched (with PDL) right after the frozen-velocity prep, so the prep
  // tile is the previous kernel's output and w is not: stage w (and the
  // tables) before griddepcontrol.wait, the prep tile after it
  int prep_dep;
  int rev;   // 1: sweep the tiles from the last to the first (alternates from launch to launch)
};

#ifndef HDGC_PF_AHEAD
#define HDGC_PF_AHEAD 0
#endif
#ifndef HDGC_A_UNROLL
#define HDGC_A_UNROLL 2   // ring mode (k >= 7): measured k=8 474 us vs 572 us fully unrolled
#endif
// One volume row b of the collapsed rule for one (element, component):
// H_i = sum_j w_ij B_ij(b), H'_i (dB/dy), then values/derivatives at the n
// points via A_i(xi_a), g = alpha d_xi w + beta d_y|xi w + gamma w, and the
// test back into r.  wv: w_c (register array or smem pointer); al/be/ga: the
// element's alpha/beta/gamma of row b, point a at [a * EPB].
template <int K, class WS>
__device__ __forceinline__ void sf_row(const WS& wv, const double* al, const double* be, const double* ga,
                                       int b, double (&r)[SF<K>::NBS], const double2* sBT = nullptr) {
  using F = SF<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, EPB = F::EPB;
  const double* C = sf_tab<K>();
  const double* Bb = C + F::C_B + b * NBS;
  const double* Bdb = C + F::C_BD + b * NBS;
  const double2* BT = sBT + b * NBS;        // ring mode: (B, B') of row b in smem
  double Hw[NE], Hwd[NE];
#pragma unroll
  for (int i = 0; i <= K; ++i) {
    double sw = 0.0, swd = 0.0;
#pragma unroll
    for (int j = 0; j <= K - i; ++j) {
      const int m = midx(i, j);
      const double x = wv[m];
      if (F::SMBT) {
        const double2 t = BT[m];
        sw = fma(x, t.x, sw);
        swd = fma(x, t.y, swd);
      } else {
        sw = fma(x, Bb[m], sw);
        swd = fma(x, Bdb[m], swd);
      }
    }
    Hw[i] = sw;
    Hwd[i] = swd;
  }
  double Kc[NE];
#pragma unroll
  for (int i = 0; i <= K; ++i) Kc[i] = 0.0;
  if constexpr (F::SYM) {
    // The xi points are Gauss-Legendre on [0, 1], symmetric about 1/2, and
    // A_i(a) = P_i(2 xi_a - 1): A_i(N-1-a) = (-1)^i A_i(a), A'_i(N-1-a) =
    // (-1)^(i+1) A'_i(a) (checked on the uploaded tables by sf_setup).  Values at
    // a mirror pair from the even-i / odd-i partial sums, and the test through
    // g(a) +- g(a'): 34 instead of 46 FP64 instructions per pair at k = 4.
#pragma unroll
    for (int a = 0; a < N / 2; ++a) {
      const int a2 = N - 1 - a;
      double ve = 0.0, vo = 0.0, ye = 0.0, yo = 0.0, xs = 0.0, xa = 0.0;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const double Ai = C[F::C_A + a * NE + i], Adi = C[F::C_AD + a * NE + i];
        if (i & 1) {
          vo = fma(Ai, Hw[i], vo);
          yo = fma(Ai, Hwd[i], yo);
          xs = fma(Adi, Hw[i], xs);
        } else {
          ve = fma(Ai, Hw[i], ve);
          ye = fma(Ai, Hwd[i], ye);
          xa = fma(Adi, Hw[i], xa);
        }
      }
      const double g1 = fma(al[a * EPB], xs + xa, fma(be[a * EPB], ye + yo, ga[a * EPB] * (ve + vo)));
      const double g2 = fma(al[a2 * EPB], xs - xa, fma(be[a2 * EPB], ye - yo, ga[a2 * EPB] * (ve - vo)));
      const double gp = g1 + g2, gm = g1 - g2;
#pragma unroll
      for (int i = 0; i <= K; ++i) Kc[i] = fma((i & 1) ? gm : gp, C[F::C_A + a * NE + i], Kc[i]);
    }
    if constexpr (N & 1) {
      // centre point xi = 1/2: odd-i values and even-i derivatives vanish
      constexpr int a = N / 2;
      double ve = 0.0, ye = 0.0, xs = 0.0;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        if (i & 1) xs = fma(C[F::C_AD + a * NE + i], Hw[i], xs);
        else {
          ve = fma(C[F::C_A + a * NE + i], Hw[i], ve);
          ye = fma(C[F::C_A + a * NE + i], Hwd[i], ye);
        }
      }
      const double g = fma(al[a * EPB], xs, fma(be[a * EPB], ye, ga[a * EPB] * ve));
#pragma unroll
      for (int i = 0; i <= K; i += 2) Kc[i] = fma(g, C[F::C_A + a * NE + i], Kc[i]);
    }
  } else {
#ifdef HDGC_A_UNROLL_SF
  constexpr int AU = F::RING ? HDGC_A_UNROLL : HDGC_A_UNROLL_SF;
#else
  constexpr int AU = F::RING ? HDGC_A_UNROLL : 64;
#endif
#pragma unroll AU
  for (int a = 0; a < N; ++a) {
    double wv0 = 0.0, wxi = 0.0, wyy = 0.0;
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      const double Ai = C[F::C_A + a * NE + i];
      wv0 = fma(Ai, Hw[i], wv0);
      wxi = fma(C[F::C_AD + a * NE + i], Hw[i], wxi);
      wyy = fma(Ai, Hwd[i], wyy);
    }
    const double g = fma(al[a * EPB], wxi, fma(be[a * EPB], wyy, ga[a * EPB] * wv0));
#pragma unroll
    for (int i = 0; i <= K; ++i) Kc[i] = fma(g, C[F::C_A + a * NE + i], Kc[i]);
  }
  }
#pragma unroll
  for (int i = 0; i <= K; ++i) {
#pragma unroll
    for (int j = 0; j <= K - i; ++j) {
      const int m = midx(i, j);
      r[m] = fma(Kc[i], F::SMBT ? BT[m].x : Bb[m], r[m]);
    }
  }
}

// Volume rows [b0, b1) with w_c cached in registers; row: the element's prep
// column (slot j at row[j * EPB], smem tile or global).
#ifndef HDGC_ROW_UNROLL
#define HDGC_ROW_UNROLL 1
#endif
// Volume rows [b0, b1) with w_c cached in registers; row: the element's prep
// column (slot j at row[j * EPB], smem tile or global).
#ifndef HDGC_ROW_UNROLL
#define HDGC_ROW_UNROLL 1
#endif
#ifndef HDGC_ROW_SWITCH
#define HDGC_ROW_SWITCH 0
#endif
// one row with a compile-time row index (immediate constant-bank operands for B, B')
template <int K, int B, class WS>
__device__ __forceinline__ void sf_row_fixed(const WS& wv, const double* row, double (&r)[SF<K>::NBS],
                                             const double2* sBT) {
  using F = SF<K>;
  sf_row<K>(wv, row + (F::P_AL + B * F::N) * F::EPB, row + (F::P_BE + B * F::N) * F::EPB,
            row + (F::P_GA + B * F::N) * F::EPB, B, r, sBT);
}
template <int K, class WS, int... Bs>
__device__ __forceinline__ void sf_row_switch(int b, const WS& wv, const double* row, double (&r)[SF<K>::NBS],
                                              const double2* sBT, std::integer_sequence<int, Bs...>) {
  ((b == Bs ? sf_row_fixed<K, Bs>(wv, row, r, sBT) : void()), ...);
}
template <int K, int B0, int B1>
__device__ __forceinline__ void sf_rows(const double* wc, const double* row, double (&r)[SF<K>::NBS],
                                        const double2* sBT) {
  constexpr int b0 = B0, b1 = B1, RU = HDGC_ROW_UNROLL;
  using F = SF<K>;
  constexpr int N = F::N, NBS = F::NBS, EPB = F::EPB;
  if constexpr (F::RING || F::WSMEM) {
    // w_c read from the smem tile in every row (no register copy)
#pragma unroll 1
    for (int b = b0; b < b1; ++b) {
      if (F::WSMEM) asm volatile("" ::: "memory");   // keep the w loads inside the loop
      sf_row<K>(wc, row + (F::P_AL + b * N) * EPB, row + (F::P_BE + b * N) * EPB, row + (F::P_GA + b * N) * EPB,
                b, r, sBT);
    }
  } else {
    double wo[NBS];
#pragma unroll
    for (int m = 0; m < NBS; ++m) wo[m] = wc[m];
#pragma unroll RU
    for (int b = b0; b < b1; ++b)
      sf_row<K>(wo, row + (F::P_AL + b * N) * EPB, row + (F::P_BE + b * N) * EPB, row + (F::P_GA + b * N) * EPB,
                b, r, sBT);
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

// Volume rows [0, nrows) for the whole warp, prep streamed row by row from
// the global tile (gtile, slot-major [PREP][16]) through the two-slot smem
// ring with cp.async (16-B pieces, all lanes), one row ahead; w_c read from
// smem (wc).  Lane (le, c): its element's column is le.
template <int K>
__device__ __forceinline__ void sf_rows_ring(const double* wc, const double* __restrict__ gtile, double* ring,
                                             int le, int lane, int nrows, double (&r)[SF<K>::NBS],
                                             const double2* sBT) {
  using F = SF<K>;
  constexpr int N = F::N, EPB = F::EPB;
  constexpr int PIECES = N * EPB / 2;          // 16-B pieces per alpha/beta/gamma row block
  auto issue = [&](int b) {
    double* dst = ring + (b & 1) * F::RING_SLOT;
#pragma unroll
    for (int t = lane; t < 3 * PIECES; t += 32) {
      const int blk = t / PIECES, off = 2 * (t - blk * PIECES);
      const int slot = (blk == 0 ? F::P_AL : (blk == 1 ? F::P_BE : F::P_GA)) + b * N;
      cp_async16(dst + blk * N * EPB + off, gtile + slot * EPB + off);
    }
    cp_async_commit();
  };
  issue(0);
#pragma unroll 1
  for (int b = 0; b < nrows; ++b) {
    if (b + 1 < nrows) issue(b + 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const double* sl = ring + (b & 1) * F::RING_SLOT + le;
    sf_row<K>(wc, sl, sl + N * EPB, sl + 2 * N * EPB, b, r, sBT);
    __syncwarp();                                  // slot b & 1 is refilled at b + 1
  }
}

// stage epilogue with the extra vector x (SSP-RK2 second stage, Richardson):
// out = a w + b x + c minv r, optional residual sum of squares (StageParams)
template <int NBS>
__device__ __forceinline__ double stage_x(const StageParams& st, double mi, double cm, const double (&r)[NBS],
                                     const double* part, const double (&wo)[NBS], double* out,
                                     const double* __restrict__ xg, double* rn) {
  const double tm = -st.tau * mi;
  double acc = 0.0, chk = 0.0;
#pragma unroll
  for (int m = 0; m < NBS; ++m) {
    const double rv = r[m] + part[m];
    const double xv = xg[m];
    const double v = fma(st.b, xv, fma(cm, rv, st.a * wo[m]));
    out[m] = v;
    chk += v;
    const double res = fma(tm, rv, xv - wo[m]);
    acc = fma(res, res, acc);
  }
  guard_finite(st.flag, chk);
  if (rn) *rn = acc;
  return acc;
}

// ---------------------------------------------------------------------------
// Structured edge traces (facets_v2).  The trace of a Dubiner mode
// D_ij = c_ij (1-y)^i P_i(2 xi - 1) P_j^(2i+1,0)(2y - 1) on a reference edge,
// expanded in the orthonormal Legendre basis L_l of the edge parameter t:
//   edge 0 (y = 0, xi = t):      only l = i           -> R_0[i][m]   (NBS values)
//   edge 1 (xi = 1, y = t):      degree i + j in t    -> R_1[l][m], l <= i + j
//   edge 2 (xi = 0, y = 1 - t):  P_i(-1) = (-1)^i and L_l(1-t) = (-1)^l L_l(t)
//                                -> R_2[l][m] = (-1)^(i+l) R_1[l][m]
// so the traces of one coefficient vector on all three edges cost
// NBS + sum_d (d+1)^2 FMA with compile-time (immediate constant-bank) operands:
// E_l / O_l = the even-i / odd-i parts of R_1 w, t1 = E + O, t2 = (-1)^l (E - O).
// sf_setup checks the three identities on the uploaded tables.
// The table c_tr holds the non-zeros in the order the unrolled loops below use
// them: for d = i + j = 0..k, j = 0..d: R_0[i][m], R_1[0..d][m]; it is read in
// pairs with pinned (asm volatile) constant loads right before their use --
// left to itself ptxas hoists the ~70 loads of each copy of this code to its
// top and shuffles them between uniform and vector registers (spills).
__device__ __forceinline__ double2 ldc_pair(const double* q) {
  double2 v;
  asm volatile("ld.const.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(__cvta_generic_to_constant(q)));
  return v;
}

template <int K>
__device__ __forceinline__ void edge_traces(const double (&w)[SF<K>::NBS], double (&t0)[SF<K>::NE],
                                            double (&t1)[SF<K>::NE], double (&t2)[SF<K>::NE]) {
  static_assert(K == HDGC_ORDER, "trace tables are per translation unit");
  constexpr int NE = SF<K>::NE;
  double E[NE], O[NE];
#pragma unroll
  for (int l = 0; l < NE; ++l) t0[l] = E[l] = O[l] = 0.0;
  int idx = 0;
  double2 cv = make_double2(0.0, 0.0);
  auto next = [&]() -> double {
    if ((idx & 1) == 0) cv = ldc_pair(c_tr + idx);
    const double v = (idx & 1) ? cv.y : cv.x;
    ++idx;
    return v;
  };
#pragma unroll
  for (int d = 0; d <= K; ++d) {
#pragma unroll
    for (int j = 0; j <= d; ++j) {
      const int i = d - j, m = midx(i, j);
      t0[i] = fma(next(), w[m], t0[i]);
#pragma unroll
      for (int l = 0; l <= d; ++l) {
        if (i & 1) O[l] = fma(next(), w[m], O[l]);
        else E[l] = fma(next(), w[m], E[l]);
      }
    }
  }
#pragma unroll
  for (int l = 0; l < NE; ++l) {
    t1[l] = E[l] + O[l];
    t2[l] = (l & 1) ? O[l] - E[l] : E[l] - O[l];
  }
}

// r += sum_e R_e^T rho_e with the same structure (transpose of edge_traces)
template <int K>
__device__ __forceinline__ void edge_test(const double (&rho0)[SF<K>::NE], const double (&rho1)[SF<K>::NE],
                                          const double (&rho2)[SF<K>::NE], double (&r)[SF<K>::NBS]) {
  constexpr int NE = SF<K>::NE;
  double P[NE], M[NE];   // even-i / odd-i combinations of rho_1 and rho_2
#pragma unroll
  for (int l = 0; l < NE; ++l) {
    const double s2 = (l & 1) ? -rho2[l] : rho2[l];
    P[l] = rho1[l] + s2;
    M[l] = rho1[l] - s2;
  }
  int idx = 0;
  double2 cv = make_double2(0.0, 0.0);
  auto next = [&]() -> double {
    if ((idx & 1) == 0) cv = ldc_pair(c_tr + idx);
    const double v = (idx & 1) ? cv.y : cv.x;
    ++idx;
    return v;
  };
#pragma unroll
  for (int d = 0; d <= K; ++d) {
#pragma unroll
    for (int j = 0; j <= d; ++j) {
      const int i = d - j, m = midx(i, j);
      double acc = fma(next(), rho0[i], r[m]);
#pragma unroll
      for (int l = 0; l <= d; ++l) acc = fma(next(), (i & 1) ? M[l] : P[l], acc);
      r[m] = acc;
    }
  }
}

// More than 32 halo rows in one tile (not on the BASELINE meshes): the
// neighbour's coefficients straight from global memory, rolled loops, out of line.
template <int K>
__device__ __noinline__ void halo_overflow(const double* __restrict__ g, int e2, const double* own, double* dl) {
  constexpr int NE = SF<K>::NE, NBS = SF<K>::NBS;
  for (int l = 0; l < NE; ++l) {
    double t = 0.0;
    for (int i = 0; i <= K; ++i)
      for (int j = 0; j <= K - i; ++j) {
        const int m = midx(i, j);
        double R = 0.0;
        if (e2 == 0) R = l == i ? c_r0[m] : 0.0;
        else if (l <= i + j) R = (e2 == 2 && ((i + l) & 1)) ? -c_r1[l * NBS + m] : c_r1[l * NBS + m];
        t = fma(R, g[m], t);
      }
    dl[l] = ((l & 1) ? -t : t) - own[l];
  }
}

// The upwind facet term of one (element, component) lane, all three edges in
// uniform code.  Own traces on the three edges -> published in s_tr for the
// in-tile neighbours; out-of-tile neighbours with inflow points get a halo slot
// (claimed with warp ballots, filled by cp.async while the own traces are
// computed) and their trace is evaluated here; jump coefficients
// d_l = (-1)^l t_nbr,l - t_own,l (reversed neighbour parameter, MESH:201), jump at
// the nf points through L_l(t_q), weighted by the frozen inflow weights s_q,
// folded back through L and R^T.  No per-lane table reads from shared memory.
template <int K>
__device__ __forceinline__ void facets_v2(const SFParams& p, const double* row, const double* wc,
                                          const int (&codes)[3], double* s_tr, double* s_halo, int T0, int nel,
                                          int lane, int c, bool active, double (&r)[SF<K>::NBS],
                                          const double2* sBT) {
  using F = SF<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NF = F::NF, EPB = F::EPB, HSTR = F::HSTR;
  const double* FL = fl_tab<K>();
  unsigned emask = 0, hmask = 0;
  if (active) {
#pragma unroll
    for (int ed = 0; ed < 3; ++ed) {
      bool any = false;
#pragma unroll
      for (int q = 0; q < NF; ++q) any |= row[(F::P_S + ed * NF + q) * EPB] != 0.0;
      const bool has_ext = codes[ed] >= 0 || p.inflow != nullptr;   // else exterior = own trace
      if (any && has_ext) {
        emask |= 1u << ed;
        const int nbT = codes[ed] >> 2;
        if (codes[ed] >= 0 && (nbT < T0 || nbT >= T0 + nel)) hmask |= 1u << ed;
      }
    }
  }
  // halo slots: lane-ordered claims per edge; slots >= 32 (rare) read global memory directly.
  // The claiming lane starts the copy of the neighbour's coefficients into the slot;
  // the neighbour's local edge id of slot s goes to bit s of two warp-wide masks.
  int hslot[3];
  int nslots = 0;
  unsigned e2lo = 0, e2hi = 0;
  {
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int ed = 0; ed < 3; ++ed) {
      const bool need = (hmask >> ed) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, need);
      hslot[ed] = need ? nslots + __popc(bal & lt) : -1;
      nslots += __popc(bal);
      if (need && hslot[ed] < 32) {
        HDGC_ASSERT((codes[ed] >> 2) < p.nt && (codes[ed] & 3) < 3);
        const double* g = p.w + (size_t)(codes[ed] >> 2) * NB + c * NBS;
        double* dst = s_halo + hslot[ed] * HSTR;
#pragma unroll
        for (int m = 0; m < NBS; ++m) cp_async8(dst + m, g + m);
        e2lo |= (unsigned)(codes[ed] & 1) << hslot[ed];
        e2hi |= (unsigned)((codes[ed] >> 1) & 1) << hslot[ed];
      }
    }
  }
  if constexpr (F::OWNF) {
    // own traces on the three edges -> s_tr row of this lane (own side of the
    // jumps, and the in-tile neighbours), while the halo rows are in flight
    double wv[NBS];
#pragma unroll
    for (int m = 0; m < NBS; ++m) wv[m] = wc[m];
    double t0[NE], t1[NE], t2[NE];
    edge_traces<K>(wv, t0, t1, t2);
    double* mine = s_tr + lane * HSTR;
#pragma unroll
    for (int l = 0; l < NE; ++l) {
      mine[l] = t0[l];
      mine[NE + l] = t1[l];
      mine[2 * NE + l] = t2[l];
    }
  }
  // balance: the facet warp takes the last FACET_ROWS volume rows, while its halo
  // rows are in flight
#pragma unroll
  for (int m = 0; m < NBS; ++m) r[m] = 0.0;
  if (F::FACET_ROWS > 0) sf_rows<K, N - F::FACET_ROWS, N>(wc, row, r, sBT);
  // halo traces: lane s evaluates the trace of slot s on the neighbour's edge and
  // writes it back over the start of the slot -- one round whatever the number of
  // out-of-tile inflow edges per lane (the ends of a tile have two or three).
  // Every lane runs the same code; lanes without a slot discard the result.
  if (nslots > 0) {   // warp-uniform
    e2lo = __reduce_or_sync(0xffffffffu, e2lo);
    e2hi = __reduce_or_sync(0xffffffffu, e2hi);
    cp_async_wait_all();
    __syncwarp();     // the slots were filled by other lanes' copies
    const bool mine = lane < nslots;
    double* dst = s_halo + lane * HSTR;
    const double* src = mine ? dst : wc;
    double nw[NBS];
#pragma unroll
    for (int m = 0; m < NBS; ++m) nw[m] = src[m];
    const int e2 = (int)(((e2lo >> lane) & 1u) | (((e2hi >> lane) & 1u) << 1));
    double a0[NE], a1[NE], a2[NE];
    edge_traces<K>(nw, a0, a1, a2);
    if (mine) {
#pragma unroll
      for (int l = 0; l < NE; ++l) dst[l] = e2 == 1 ? a1[l] : (e2 == 2 ? a2[l] : a0[l]);
    }
  }
  if constexpr (F::OWNF) __syncwarp();   // own traces of the tile published by this warp
  else asm volatile("bar.sync 2, 64;\n" ::: "memory");   // (T) own traces of the tile published by the volume warp
  double rho[3][NE];
#pragma unroll
  for (int ed = 0; ed < 3; ++ed) {
    const bool on = (emask >> ed) & 1u;
    const int code = codes[ed];
    const double* own = s_tr + lane * HSTR + ed * NE;
    const double* nsrc = own;     // placeholder when there is no neighbour trace
    bool has_nb = false;
    const double* infl = nullptr;
    if (hslot[ed] >= 0) {
      nsrc = s_halo + (hslot[ed] & 31) * HSTR;
      has_nb = hslot[ed] < 32;
    } else if (on && code >= 0) {
      HDGC_ASSERT((code >> 2) >= T0 && (code >> 2) < T0 + nel && (code & 3) < 3);
      nsrc = s_tr + (((code >> 2) - T0) * 2 + c) * HSTR + (code & 3) * NE;
      has_nb = true;
    } else if (on) {
      infl = p.inflow + (size_t)(-1 - code) * NF * 2 + c;
    }
    double dl[NE];
#pragma unroll
    for (int l = 0; l < NE; ++l) {
      const double tn = has_nb ? nsrc[l] : 0.0;
      dl[l] = ((l & 1) ? -tn : tn) - own[l];
      rho[ed][l] = 0.0;
    }
    if (hslot[ed] >= 32) halo_overflow<K>(p.w + (size_t)(code >> 2) * NB + c * NBS, code & 3, own, dl);
    if constexpr (F::SYM) {
      // facet points are Gauss-Legendre on [0, 1]: L_l(t_{NF-1-q}) = (-1)^l L_l(t_q), so the
      // jump at a mirror pair comes from the even-l / odd-l partial sums and the
      // fold-back goes through sj(q) +- sj(q')
#pragma unroll
      for (int q = 0; q < NF / 2; ++q) {
        const int q2 = NF - 1 - q;
        const double s1 = on ? row[(F::P_S + ed * NF + q) * EPB] : 0.0;
        const double s2 = on ? row[(F::P_S + ed * NF + q2) * EPB] : 0.0;
        double Je = 0.0, Jo = 0.0;
#pragma unroll
        for (int l = 0; l < NE; ++l) {
          if (l & 1) Jo = fma(dl[l], FL[q * NE + l], Jo);
          else Je = fma(dl[l], FL[q * NE + l], Je);
        }
        double J1 = Je + Jo, J2 = Je - Jo;
        if (infl != nullptr) {
          if (s1 != 0.0) J1 += __ldg(infl + 2 * q);
          if (s2 != 0.0) J2 += __ldg(infl + 2 * q2);
        }
        const double a1 = s1 * J1, a2 = s2 * J2;
        const double sp = a1 + a2, sm = a1 - a2;
#pragma unroll
        for (int l = 0; l < NE; ++l) rho[ed][l] = fma((l & 1) ? sm : sp, FL[q * NE + l], rho[ed][l]);
      }
      if constexpr (NF & 1) {
        constexpr int q = NF / 2;   // t = 1/2: odd-l values vanish
        const double sq = on ? row[(F::P_S + ed * NF + q) * EPB] : 0.0;
        double J = 0.0;
#pragma unroll
        for (int l = 0; l < NE; l += 2) J = fma(dl[l], FL[q * NE + l], J);
        if (infl != nullptr && sq != 0.0) J += __ldg(infl + 2 * q);
        const double sj = sq * J;
#pragma unroll
        for (int l = 0; l < NE; l += 2) rho[ed][l] = fma(sj, FL[q * NE + l], rho[ed][l]);
      }
    } else {
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      const double sq = on ? row[(F::P_S + ed * NF + q) * EPB] : 0.0;
      double J = 0.0;
#pragma unroll
      for (int l = 0; l < NE; ++l) J = fma(dl[l], FL[q * NE + l], J);
      if (infl != nullptr && sq != 0.0) J += __ldg(infl + 2 * q);
      const double sj = sq * J;
#pragma unroll
      for (int l = 0; l < NE; ++l) rho[ed][l] = fma(sj, FL[q * NE + l], rho[ed][l]);
    }
    }
  }
  edge_test<K>(rho[0], rho[1], rho[2], r);
}

// Two warps per CTA on one tile of EPB = 16 elements: warp 0 computes the
// volume term, warp 1 the upwind facet term, concurrently; lane l of either
// warp owns (element l/2, component l%2).  The facet warp leaves its partial
// residual in shared memory (its halo buffer), the volume warp adds it and
// runs the epilogue.  Splitting the two halves of the work halves the tile's
// latency and keeps each warp under ~146 registers (7 CTAs = 14 warps/SM).
#ifdef HDGC_SF_MINB
#define HDGC_SF_MINB_OF(K) HDGC_SF_MINB
#else
// register caps 128 / 256 / 255: k <= 4 runs 8 CTAs/SM at 128 registers (a few
// spilled bytes; k=4 69.8 -> 66.5 us, k=3 53.2 -> 49.7 us measured); k >= 7: 4 CTAs/SM by smem + regs
#define HDGC_SF_MINB_OF(K) (K == 3 ? 9 : K <= 4 ? 8 : (K <= 6 ? 4 : 2))
#endif
template <int K, int MODE>
__global__ void __launch_bounds__(SF<K>::THREADS, HDGC_SF_MINB_OF(K))
conv2d_sf_kernel(SFParams p) {
  using F = SF<K>;
  constexpr int N = F::N, NE = F::NE, NBS = F::NBS, NB = F::NB, NF = F::NF, EPB = F::EPB;
  extern __shared__ __align__(128) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + F::SM_BAR);
  double* s_prep = sm + F::SM_PREP;        // [PREP][EPB]
  double* s_w = sm + F::SM_W;              // [EPB][NB]  (c-major, as in global)
  double* s_halo = sm + F::SM_HALO;        // [32][NBS]: facet warp halo, then its partial r
  double* s_fD = sm + F::SM_FD;            // edge trace maps [3][RSTR]
  const double* C = sf_tab<K>();

  double* s_x = sm + F::SM_X;              // STAGE: x tile [EPB][NB]
  hdgc_debug_prologue(sm, F::smem_doubles(MODE));
  // consecutive launches of a batch sweep the tiles in alternating directions
  // (SFParams::rev): the tiles the previous substep touched last -- prep rows and
  // its output w -- are the first ones read, while they are still in L2
  const int tile = p.rev ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int T0 = tile * EPB;
  const int nel = min(EPB, p.nt - T0);
  double2* s_BT = reinterpret_cast<double2*>(sm + F::SM_BT);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (F::SMBT)
    for (int t = threadIdx.x; t < N * NBS; t += F::THREADS) s_BT[t] = make_double2(C[F::C_B + t], C[F::C_BD + t]);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bp = F::RING ? 0u : (uint32_t)(F::PREP_TILE * sizeof(double));
    const uint32_t bw = (uint32_t)(nel * NB * sizeof(double));
    const uint32_t bt = (uint32_t)(F::TAB_SM * sizeof(double));   // 0 with FV2
    mbar_arrive_expect_tx(bar, bp + bw + bt + (MODE == MODE_STAGE && F::XTILE ? bw : 0u));
    if (p.prep_dep) {
      // right after the prep kernel: w is an input, the prep tile the previous grid's output
      bulk_g2s(s_w, p.w + (size_t)T0 * NB, bw, bar);
      if (!F::FV2) bulk_g2s(s_fD, p.ftab, bt, bar);
      pdl_wait();
      if (!F::RING) bulk_g2s(s_prep, p.prep + (size_t)tile * F::PREP_TILE, bp, bar);
    } else {
      // substep batch: the prep tile is frozen, w is the previous update kernel's output
      if (!F::RING) bulk_g2s(s_prep, p.prep + (size_t)tile * F::PREP_TILE, bp, bar);
      if (!F::FV2) bulk_g2s(s_fD, p.ftab, bt, bar);
      pdl_wait();
      bulk_g2s(s_w, p.w + (size_t)T0 * NB, bw, bar);
    }
    if (MODE == MODE_STAGE && F::XTILE)
      bulk_g2s(s_x, p.st.x + (size_t)T0 * NB, bw, bar);   // x is not the previous kernel's output
#if HDGC_PF_AHEAD
    // L2 prefetch of the prep tile a CTA HDGC_PF_AHEAD positions later in the sweep will stage
    if (!F::RING) {
      const int ahead = p.rev ? tile - HDGC_PF_AHEAD : tile + HDGC_PF_AHEAD;
      if (ahead >= 0 && ahead < (int)gridDim.x)
        bulk_prefetch_l2(p.prep + (size_t)ahead * F::PREP_TILE, (uint32_t)(F::PREP_TILE * sizeof(double)));
    }
#endif
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int le = lane >> 1;
  const int c = lane & 1;
  const bool active = le < nel;
  const int T = T0 + (active ? le : 0);
  double* part = s_halo + lane * F::HSTR;
  const double* gtile = p.prep + (size_t)tile * F::PREP_TILE;
  // the element's prep column (slot j at row[j * EPB]): smem tile, or (ring) the global tile
  const double* row = (F::RING ? gtile : s_prep) + (active ? le : 0);
  double r[NBS];
  if (!F::FV2) {
#pragma unroll
    for (int m = 0; m < NBS; ++m) r[m] = 0.0;
  }

  if (warp == 0) {
    // ===================== volume warp =====================
    const double mi = (MODE == MODE_SUBSTEP || MODE == MODE_STAGE) && active ? __ldg(p.minv + T) : 0.0;
    pdl_wait();
    const int stopped = MODE == MODE_STAGE ? stage_stop_flag(p.st) : 0;   // (latency hidden by the tile wait)
    pdl_trigger();
    mbar_wait(bar, 0);
    if (stopped) return;   // converged Richardson iteration: queued after the stop, writes nothing
    const double* wc = s_w + (active ? le : 0) * NB + c * NBS;
    if constexpr (F::FV2 && !F::OWNF) {
      // own traces on the three edges -> s_tr row of this lane (read by the facet
      // warp: own side of the jumps, and the in-tile neighbours)
      double wv[NBS];
#pragma unroll
      for (int m = 0; m < NBS; ++m) wv[m] = wc[m];
      double t0[NE], t1[NE], t2[NE];
      edge_traces<K>(wv, t0, t1, t2);
      double* mine = sm + F::SM_TR + lane * F::HSTR;
#pragma unroll
      for (int l = 0; l < NE; ++l) {
        mine[l] = t0[l];
        mine[NE + l] = t1[l];
        mine[2 * NE + l] = t2[l];
      }
      asm volatile("bar.arrive 2, 64;\n" ::: "memory");   // (T)
    }
    if constexpr (F::FV2) {
#pragma unroll
      for (int m = 0; m < NBS; ++m) r[m] = 0.0;   // (not live across the traces)
    }
    if (F::RING) sf_rows_ring<K>(wc, gtile, s_prep, active ? le : 0, lane, N - F::FACET_ROWS, r, s_BT);
    else sf_rows<K, 0, N - F::FACET_ROWS>(wc, row, r, s_BT);
    asm volatile("bar.sync 1, 64;\n" ::: "memory");   // (A) facet partial r ready, in-tile w reads done
    double racc = 0.0;   // STAGE: this lane's residual sum of squares
    if (active) {
      double* wo_s = s_w + le * NB + c * NBS;
      double wo[NBS];
#pragma unroll
      for (int m = 0; m < NBS; ++m) wo[m] = wo_s[m];
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
        racc = stage_x(p.st, mi, p.st.c * mi, r, part, wo, wo_s,
                       (F::XTILE ? s_x : p.st.x + (size_t)T0 * NB) + le * NB + c * NBS,
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
    if (MODE == MODE_STAGE && p.st.rpart) rich_cta_partial(p.st, racc, tile);
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
    const double* wc = s_w + (active ? le : 0) * NB + c * NBS;
    if constexpr (F::FV2) {
      facets_v2<K>(p, row, wc, codes, sm + F::SM_TR, s_halo, T0, nel, lane, c, active, r, s_BT);
    } else {
    double* halo = part;
    int halo_edge = -1;
    if (active) {
#pragma unroll
      for (int ed = 0; ed < 3; ++ed) {
        const int code = codes[ed];
        if (code < 0 || halo_edge >= 0) continue;
        const int nbT = code >> 2;
        if (nbT >= T0 && nbT < T0 + nel) continue;
        bool any = false;
#pragma unroll
        for (int q = 0; q < NF; ++q) any |= row[(F::P_S + ed * NF + q) * EPB] != 0.0;
        if (!any) continue;
        halo_edge = ed;
        const double* g = p.w + (size_t)nbT * NB + c * NBS;
#pragma unroll
        for (int m = 0; m < NBS; ++m) cp_async8(halo + m, g + m);
      }
    }
    if (halo_edge >= 0) cp_async_wait_all();
    __shared__ double zero_row[NBS];
    for (int m = lane; m < NBS; m += 32) zero_row[m] = 0.0;
    __syncwarp();
    // inflow-edge work list: every lane walks only its own inflow edges, so the
    // warp runs max_lane(#inflow edges) iterations (usually 2) instead of all
    // three with idle lanes.  Edge tables: smem, transposed [edge][m][QP].
    unsigned emask = 0;
    if (active) {
#pragma unroll
      for (int ed = 0; ed < 3; ++ed) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < NF; ++q) any |= row[(F::P_S + ed * NF + q) * EPB] != 0.0;
        const bool has_ext = codes[ed] >= 0 || p.inflow != nullptr;   // else exterior = own trace
        if (any && has_ext) emask |= 1u << ed;
      }
    }
    const int nmine = __popc(emask);
    const int nmax = __reduce_max_sync(0xffffffffu, (unsigned)nmine);
    // Jumps in the edge's own P_k basis: the trace of a Dubiner mode on edge e is
    // D_m(x_e(t)) = sum_l R_e[l][m] L_l(t) exactly (orthonormal Legendre), the
    // neighbour's trace at t' = 1 - t has coefficients (-1)^l (R_e2 w_nbr)_l,
    // so the jump coefficients are d_l = (-1)^l (R_e2 w_nbr)_l - (R_e w_own)_l,
    // the jump at point q is sum_l d_l L_l(t_q), and the test folds back
    // through R_e^T.  R from smem (per-lane edge), L from the constant bank.
    const double* FL = fl_tab<K>();
#pragma unroll 1
    for (int j = 0; j < nmax; ++j) {
      const bool on = j < nmine;
      const int ed = on ? __ffs(emask) - 1 : 0;
      if (on) emask &= emask - 1;
      const int code = ed == 0 ? codes[0] : (ed == 1 ? codes[1] : codes[2]);
      // neighbour coefficients: CTA tile or halo (smem), rarely global (generic loads)
      const double* src = zero_row;     // zeros: no neighbour term
      const double* infl = nullptr;
      int e2 = 0;
      if (on && code >= 0) {
        const int nbT = code >> 2;
        e2 = code & 3;
        HDGC_ASSERT(nbT < p.nt && e2 < 3);
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
      double rho[NE];
#pragma unroll
      for (int l = 0; l < NE; ++l) rho[l] = 0.0;
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        const double sq = on ? row[(F::P_S + ed * NF + q) * EPB] : 0.0;
        double J = 0.0;
#pragma unroll
        for (int l = 0; l < NE; ++l) J = fma(dl[l], FL[q * NE + l], J);
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
    }   // !FV2
    // balance: the facet warp also takes the last FACET_ROWS volume rows
    if (!F::FV2 && F::FACET_ROWS > 0) sf_rows<K, N - F::FACET_ROWS, N>(wc, row, r, s_BT);
    __syncwarp();          // halo reads of all lanes done before the partials overwrite it
#pragma unroll
    for (int m = 0; m < NBS; ++m) part[m] = r[m];
    asm volatile("bar.sync 1, 64;\n" ::: "memory");   // (A)
  }
}

}  // namespace hdgc
