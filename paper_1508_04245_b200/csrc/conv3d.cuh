// 3D (tetrahedra) convection apply, BASELINE cfg5.  No reference
// code exists for 3D; the operator is the 2D one carried to tets:
//
//   r = sigma [ sum_p w_p (u_hat.grad w_c + w_c div u_hat)(p) D_m(p)
//             + sum_f sum_{q: sigma F < 0} w_q F_f(q) (w_ext - w_own)_c(q) D_m(x_f(q)) ]
//
// with sigma = sign(detJ) (tet vertices are sorted by global id, so about half
// the elements are negatively oriented) and F_f(q) = 2|f| u_hat.n_hat at face
// point q, from the face dofs.  Shared faces are parametrised identically on
// both sides (sorted vertices), so point q of the owner is point q of the
// neighbour.  Direct evaluation on the collapsed (3k+1)/2-cubed rule.
//
// Frozen-velocity prep (per element, point-major SoA for coalesced reads):
//   slot p        : alpha_x = sigma w_p u_hat_x(p)      (p < NQ)
//   slot NQ+p     : alpha_y,  2NQ+p: alpha_z,  3NQ+p: gamma = sigma w_p div u_hat
//   slot 4NQ+f*NF+q: s = sigma w_q F if sigma F < 0 else 0
#pragma once
#include "common.cuh"

namespace hdgc {

#ifndef HDGC_3D_SYM
#define HDGC_3D_SYM 1   // mirror-pair evaluation of the a direction in the volume term
#endif
template <int K>
struct Dims3 {
  static constexpr int NBS = (K + 1) * (K + 2) * (K + 3) / 6;
  static constexpr int NB = 3 * NBS;
  static constexpr int NBS1 = K * (K + 1) * (K + 2) / 6;
  static constexpr int NFD = (K + 1) * (K + 2) / 2;                 // face dofs per face
  static constexpr int N1 = (3 * K + 1) / 2;
  static constexpr int NQ = N1 * N1 * N1;                            // volume points
  static constexpr int NF = K == 1 ? 6 : ((3 * K + 3) / 2) * ((3 * K + 3) / 2);   // face points, quad_triangle(3k+1)
  // packed table layout (doubles)
  static constexpr int OFF_COEF = 0;
  static constexpr int OFF_DIVM = OFF_COEF + NB * NB;
  static constexpr int OFF_VW = OFF_DIVM + NBS1 * NB;
  static constexpr int OFF_VD = OFF_VW + NQ;
  static constexpr int OFF_VG = OFF_VD + NQ * NBS;                  // [NQ][NBS][3]
  static constexpr int OFF_FW = OFF_VG + NQ * NBS * 3;
  static constexpr int OFF_FL = OFF_FW + NF;                         // [NF][NFD] normal-trace basis
  static constexpr int OFF_FD = OFF_FL + NF * NFD;                   // [4][NF][NBS]
  static constexpr int OFF_FLEN = OFF_FD + 4 * NF * NBS;             // [4]
  static constexpr int TAB = OFF_FLEN + 4;
  static constexpr int NSYM = NFD * (NFD + 1) / 2;                   // upper triangle of a face matrix
  static constexpr int P_MASK = 4 * NQ + 4 * NF;                     // inflow-face bitmask slot
  static constexpr int P_S = P_MASK + 1;                             // face inflow matrices S_f [4][NSYM]
  static constexpr int PREP = P_S + 4 * NSYM;
  static constexpr int NFP = NF + (NF & 1);                          // face points padded (smem table)
  // face trace maps R[f][n][m] in smem with an odd per-face stride: lanes on
  // different faces hit disjoint bank pairs (the k=3 stride 200 would alias f, f+2)
  static constexpr int RSTR = (NFD * NBS) | 1;
  static constexpr int RTAB = 4 * RSTR;
  static constexpr int EPB = 32;                                     // elements per CTA
  static constexpr int THREADS = 3 * EPB;                            // one warp per component
  // Volume coefficients alpha | beta | gamma | delta are stored tile-blocked and
  // grouped by collapsed row (ic, ib): [tile of 32][row][field][ia][32], so one
  // row of one CTA is a single contiguous VROW * 32 doubles (one bulk copy);
  // the face slots (>= 4 NQ) keep the point-major SoA layout with row stride
  // ps = nt rounded up to 32 (they start exactly where the volume region ends).
  static constexpr int VROW = 4 * N1;                                // doubles per element and row
  static constexpr int NROW = N1 * N1;
  static constexpr int RBUF = VROW * EPB;                            // one staged row of a CTA
  // staged row buffers: k = 1, 3 a ring of 3 with producer / consumer
  // mbarriers, k = 2, 4 a double buffer refilled after a CTA barrier (the ring's
  // bookkeeping costs registers there: cfg5-size k=4 1993 vs 2419 us, k=2 193 vs 214)
  static constexpr bool RINGMB = K == 1 || K == 3;
  static constexpr int NRB = RINGMB ? 3 : 2;
  static constexpr int SMEM = (RTAB + 2 * NBS * 96 + NRB * RBUF) * 8;  // + own / neighbour w columns + row ring
  __host__ __device__ static constexpr size_t vofs(int T, int q, int field) {
    return ((((size_t)(T >> 5) * NROW + q / N1) * 4 + field) * N1 + q % N1) * 32 + (T & 31);
  }
};
inline int prep3_stride(int nt) { return (nt + 31) & ~31; }

// sum-factorisation tables (constant bank of the order compiled in this TU):
// D_ijl(a,b,c) = A_i(a) B_ij(b) C_ijl(c) on the collapsed n^3 rule
template <int K>
struct SF3 {
  static constexpr int N = (3 * K + 1) / 2;
  static constexpr int NE = K + 1;
  static constexpr int NPAIR = (K + 1) * (K + 2) / 2;
  static constexpr int NBS = (K + 1) * (K + 2) * (K + 3) / 6;
  static constexpr int NQ = N * N * N;
  static constexpr int C_A = 0, C_AD = C_A + N * NE, C_B = C_AD + N * NE, C_BD = C_B + N * NPAIR;
  static constexpr int C_C = C_BD + N * NPAIR, C_CD = C_C + N * NBS, C_PF = C_CD + N * NBS;
  static constexpr int NF = K == 1 ? 6 : ((3 * K + 3) / 2) * ((3 * K + 3) / 2);
  static constexpr int NFD = (K + 1) * (K + 2) / 2;
  static constexpr int C_D2 = C_PF + NQ * 5;                         // [NF][NFD] face modes at face points
  static constexpr int C_TOTAL = C_D2 + NF * NFD;
};

__host__ __device__ constexpr int midx3(int i, int j, int l) {
  return (i + j + l) * (i + j + l + 1) * (i + j + l + 2) / 6 + l * (i + j + l + 1) - l * (l - 1) / 2 + j;
}
__host__ __device__ constexpr int pidx(int i, int j) { return (i + j) * (i + j + 1) / 2 + j; }

#ifdef HDGC_ORDER3
__constant__ double c_sf3d[SF3<HDGC_ORDER3>::C_TOTAL];
#endif

inline int dims3_nq(int k) { const int n = (3 * k + 1) / 2; return n * n * n; }
inline int dims3_nf(int k) {
  return k == 1 ? 6 : ((3 * k + 3) / 2) * ((3 * k + 3) / 2);
}
inline int dims3_nbs(int k) { return (k + 1) * (k + 2) * (k + 3) / 6; }
inline int dims3_tab(int k) {
  const int nbs = dims3_nbs(k), nb = 3 * nbs, nbs1 = k * (k + 1) * (k + 2) / 6, nfd = (k + 1) * (k + 2) / 2;
  const int nq = dims3_nq(k), nf = dims3_nf(k);
  return nb * nb + nbs1 * nb + nq + nq * nbs + nq * nbs * 3 + nf + nf * nfd + 4 * nf * nbs + 4;
}

// geometry: J (columns = edges), det, Piola J/detJ (9, NT), 6/|detJ|, sign
__global__ void geometry3d_kernel(const double* __restrict__ V, const int64_t* __restrict__ tet, int nt, int nv,
                                  double* __restrict__ piola, double* __restrict__ minv,
                                  double* __restrict__ sgn, int* __restrict__ bad);

#ifdef HDGC_ORDER3   // kernels: only in the per-order translation units
#ifndef HDGC_3D_SMEM_R
#define HDGC_3D_SMEM_R 1   // w_c and the volume accumulators r in smem, registers for the sum-factorisation state
#endif
#ifndef HDGC_3D_MINB
#define HDGC_3D_MINB (HDGC_3D_SMEM_R ? 4 : 2)   // 168 / 255 registers: 4 / 2 CTAs (12 / 6 warps) per SM (k=3: 1221 us vs 2014 us)
#endif
struct Prep3Params {
  const double* __restrict__ tab;
  const double* __restrict__ u;
  const double* __restrict__ sgn;
  double* __restrict__ prep;
  int nt;
  int ps;    // SoA stride of the face slots (prep3_stride)
};

template <int K>
__global__ void __launch_bounds__(128)
prep3d_kernel(Prep3Params p) {
  pdl_trigger();   // the update kernel after a prep may launch now (PDL, Conv3Params::prep_dep)
  using D = Dims3<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NBS1 = D::NBS1, NFD = D::NFD, NQ = D::NQ, NF = D::NF;
  const int T = blockIdx.x * blockDim.x + threadIdx.x;
  if (T >= p.nt) return;
  const double* tab = p.tab;
  const double sg = __ldg(p.sgn + T);
  const size_t nt = (size_t)p.ps;   // face-slot stride
  double x[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) x[j] = __ldg(p.u + (size_t)T * NB + j);
  // inflow weights from the face dofs (first 4*NFD dofs, face-major) and the
  // bitmask of faces with at least one inflow point
  unsigned fmask = 0;
  const double* D2 = c_sf3d + SF3<K>::C_D2;
#pragma unroll 1
  for (int f = 0; f < 4; ++f) {
    const double len = __ldg(tab + D::OFF_FLEN + f);
    double sv[NF];
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < NFD; ++m) a = fma(x[f * NFD + m], __ldg(tab + D::OFF_FL + q * NFD + m), a);
      const double F = sg * a * len;
      sv[q] = F < 0.0 ? __ldg(tab + D::OFF_FW + q) * F : 0.0;
      p.prep[(size_t)(4 * NQ + f * NF + q) * nt + T] = sv[q];
      if (F < 0.0) fmask |= 1u << f;
    }
    // face inflow matrix S_f[n][n2] = sum_q s_q D2_n(q) D2_n2(q), upper triangle row-major
#pragma unroll 1
    for (int n = 0; n < NFD; ++n)
#pragma unroll 1
      for (int n2 = n; n2 < NFD; ++n2) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < NF; ++q) a = fma(sv[q] * D2[q * NFD + n], D2[q * NFD + n2], a);
        p.prep[(size_t)(D::P_S + f * D::NSYM + n * NFD - n * (n - 1) / 2 + (n2 - n)) * nt + T] = a;
      }
  }
  p.prep[(size_t)D::P_MASK * nt + T] = (double)fmask;
  double uh[NB];
#pragma unroll 1
  for (int i = 0; i < NB; ++i) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) a = fma(__ldg(tab + D::OFF_COEF + i * NB + j), x[j], a);
    uh[i] = a;     // dynamic index: local memory for large K is acceptable (once per batch)
  }
  double dv[NBS1];
#pragma unroll 1
  for (int i = 0; i < NBS1; ++i) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) a = fma(__ldg(tab + D::OFF_DIVM + i * NB + j), x[j], a);
    dv[i] = a;
  }
#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    const double* Dq = tab + D::OFF_VD + q * NBS;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, dq = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      const double d = __ldg(Dq + m);
      a0 = fma(uh[m], d, a0);
      a1 = fma(uh[NBS + m], d, a1);
      a2 = fma(uh[2 * NBS + m], d, a2);
      if (m < NBS1) dq = fma(dv[m], d, dq);
    }
    // flux-form coefficients in collapsed coordinates (chain rule of the Duffy map):
    // g = alpha w_a + beta w_b + gamma w_c + delta w
    const double* pf = c_sf3d + SF3<K>::C_PF + q * 5;
    p.prep[D::vofs(T, q, 0)] = sg * fma(pf[0], a0, pf[1] * (a1 + a2));
    p.prep[D::vofs(T, q, 1)] = sg * fma(pf[2], a1, pf[3] * a2);
    p.prep[D::vofs(T, q, 2)] = sg * pf[4] * a2;
    p.prep[D::vofs(T, q, 3)] = sg * pf[4] * dq;
  }
}

// Tile prep (replaces the thread-per-element prep3d_kernel): one CTA per 32
// tets, lane = element.
// Stage 1: modal rows [u_hat | div u_hat] = [coef ; divm] u, (NB + NBS1) x NB
//   times NB x 32, on the FP64 tensor cores (dmma_m8n8k4, A fragments
//   precomputed host-side in c->d_afrag; u staged transposed in smem).
// Faces (warps 0..3 = face f, concurrently with nothing else needing them):
//   inflow weights s_q at the NF face points, the inflow-face bitmask, and the
//   face inflow matrix S_f = D2^T diag(s) D2 (upper triangle).
// Stage 2 (warp = collapsed c-slice ic): the velocity and its divergence at
//   the n x n points of slice ic by sum factorisation (G_ij(c) -> H_i(b, c) ->
//   values at (a, b, c)), then the flux-form coefficients alpha..delta with
//   the Duffy chain rule (C_PF), all tables warp-uniform in the constant bank.
template <int K>
struct Prep3Mma {
  static constexpr int NB = Dims3<K>::NB, NR = Dims3<K>::NB + Dims3<K>::NBS1;
  static constexpr int MT = (NR + 7) / 8, KS = (NB + 3) / 4;
  static constexpr int LD = 40;
  static constexpr int AFRAG = MT * KS * 32;
  static constexpr int WARPS = SF3<K>::N > 4 ? SF3<K>::N : 4;
  static constexpr int SMEM = KS * 4 * LD + MT * 8 * LD;   // doubles: s_u | s_h
};

// k <= 3: three CTAs per SM (128 registers; k = 3 spills 312 B and still gains:
// prep 547 -> 535 us at cfg5; four CTAs / 96 registers 675 us)
#ifndef HDGC_PREP3_MINB
#define HDGC_PREP3_MINB 3
#endif
template <int K>
__global__ void __launch_bounds__(32 * Prep3Mma<K>::WARPS, K <= 2 ? 4 : K == 3 ? HDGC_PREP3_MINB : 1)
prep_tile3d_kernel(const double* __restrict__ tab, const double* __restrict__ afrag, const double* __restrict__ u,
                   const double* __restrict__ sgn, const int32_t* __restrict__ code, int nt, int ps,
                   double* __restrict__ prep) {
  pdl_trigger();   // the update kernel after a prep may launch now (PDL, Conv3Params::prep_dep)
  using D = Dims3<K>;
  using S = SF3<K>;
  using P = Prep3Mma<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NFD = D::NFD, NQ = D::NQ, NF = D::NF, LD = P::LD;
  constexpr int N = S::N, NE = S::NE, NPAIR = S::NPAIR, NTH = 32 * P::WARPS;
  extern __shared__ __align__(16) double smq[];
  double* s_u = smq;                    // [KS*4][LD]
  double* s_h = smq + P::KS * 4 * LD;   // [MT*8][LD]
  hdgc_debug_prologue(smq, P::SMEM);
  __shared__ unsigned s_mask[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T0 = blockIdx.x * 32;
  const int nel = min(32, nt - T0);
  {
    // all of this thread's u loads in flight before the first smem store (a
    // rolled load->store loop serialised the global latency: 40% of the stalls)
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
  if (tid < 32) s_mask[tid] = 0u;
  __syncthreads();
  // row tiles of 8 x 32 over the warps: the four 8 x 8 column tiles share each A
  // fragment and run as four independent DMMA chains
  for (int mt = warp; mt < P::MT; mt += P::WARPS) {
    const double* af = afrag + (size_t)mt * P::KS * 32 + lane;
    double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 5
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
  const int T = T0 + (active ? lane : 0);
  const double sg = __ldg(sgn + T);
  const size_t nts = (size_t)ps;   // face-slot stride
  if (warp < 4) {
    // ---- face f = warp: inflow weights, bitmask, inflow matrix
    const int f = warp;
    const double len = __ldg(tab + D::OFF_FLEN + f);
    const double* D2 = c_sf3d + S::C_D2;
    double sv[NF];
    bool any = false;
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < NFD; ++m) a = fma(s_u[(f * NFD + m) * LD + lane], __ldg(tab + D::OFF_FL + q * NFD + m), a);
      const double F = sg * a * len;
      sv[q] = F < 0.0 ? __ldg(tab + D::OFF_FW + q) * F : 0.0;
      any |= F < 0.0;
    }
    // the substep kernel reads s and S_f of a face only when its inflow bit is
    // set; a warp with no inflow element on this face writes nothing, a warp
    // with some writes every active lane (zeros where there is no inflow): full
    // 32-B sectors, no read-modify-write of partially written sectors in L2
    // (which cost 440 MB of DRAM reads per cfg5 prep)
    if (any && active) atomicOr(&s_mask[lane], 1u << f);
    if (__any_sync(0xffffffffu, any && active) && active) {
      // the point weights s_q are only read for boundary faces with exterior
      // data (interior faces use S_f alone)
      const bool bnd = __ldg(code + (size_t)T * 4 + f) < 0;
      if (__any_sync(__activemask(), bnd)) {
#pragma unroll
        for (int q = 0; q < NF; ++q) prep[(size_t)(4 * NQ + f * NF + q) * nts + T] = sv[q];
      }
      // fully unrolled: every D2 entry is an immediate constant-bank operand (a
      // runtime-indexed version spent 58% of the kernel in LDC/MIO stalls); k=4
      // (120 x 49 terms) would spill, so it keeps runtime n, n2
      auto sf_entry = [&](int n, int n2) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < NF; ++q) a = fma(sv[q] * D2[q * NFD + n], D2[q * NFD + n2], a);
        prep[(size_t)(D::P_S + f * D::NSYM + n * NFD - n * (n - 1) / 2 + (n2 - n)) * nts + T] = a;
      };
      if constexpr (K <= 3) {
#pragma unroll
        for (int n = 0; n < NFD; ++n)
#pragma unroll
          for (int n2 = n; n2 < NFD; ++n2) sf_entry(n, n2);
      } else {
#pragma unroll 1
        for (int n = 0; n < NFD; ++n)
#pragma unroll 1
          for (int n2 = n; n2 < NFD; ++n2) sf_entry(n, n2);
      }
    }
  }
  __syncthreads();
  if (warp == 0 && active) prep[(size_t)D::P_MASK * nts + T] = (double)s_mask[lane];
  if (warp >= N) return;
  // ---- stage 2: collapsed slice ic = warp
  const int ic = warp;
  const double* Cs = c_sf3d;
  const double* Cc = Cs + S::C_C + ic * NBS;
  double G0[NPAIR], G1[NPAIR], G2[NPAIR], Gd[NPAIR];
#pragma unroll
  for (int i = 0; i <= K; ++i)
#pragma unroll
    for (int j = 0; j <= K - i; ++j) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, sd = 0.0;
#pragma unroll
      for (int l = 0; l <= K - i - j; ++l) {
        const int m = midx3(i, j, l);
        const double cm = Cc[m];
        s0 = fma(s_h[m * LD + lane], cm, s0);
        s1 = fma(s_h[(NBS + m) * LD + lane], cm, s1);
        s2 = fma(s_h[(2 * NBS + m) * LD + lane], cm, s2);
        if (i + j + l < K) sd = fma(s_h[(NB + m) * LD + lane], cm, sd);
      }
      G0[pidx(i, j)] = s0; G1[pidx(i, j)] = s1; G2[pidx(i, j)] = s2; Gd[pidx(i, j)] = sd;
    }
  if (!active) return;
#pragma unroll 1
  for (int ib = 0; ib < N; ++ib) {
    const double* Bb = Cs + S::C_B + ib * NPAIR;
    double H0[NE], H1[NE], H2[NE], Hd[NE];
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      double h0 = 0.0, h1 = 0.0, h2 = 0.0, hd = 0.0;
#pragma unroll
      for (int j = 0; j <= K - i; ++j) {
        const double bb = Bb[pidx(i, j)];
        h0 = fma(G0[pidx(i, j)], bb, h0);
        h1 = fma(G1[pidx(i, j)], bb, h1);
        h2 = fma(G2[pidx(i, j)], bb, h2);
        if (i + j < K) hd = fma(Gd[pidx(i, j)], bb, hd);
      }
      H0[i] = h0; H1[i] = h1; H2[i] = h2; Hd[i] = hd;
    }
#pragma unroll
    for (int ia = 0; ia < N; ++ia) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, dq = 0.0;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const double Ai = Cs[S::C_A + ia * NE + i];
        a0 = fma(Ai, H0[i], a0);
        a1 = fma(Ai, H1[i], a1);
        a2 = fma(Ai, H2[i], a2);
        if (i < K) dq = fma(Ai, Hd[i], dq);
      }
      const int q = (ic * N + ib) * N + ia;
      const double* pf = Cs + S::C_PF + q * 5;
      prep[D::vofs(T, q, 0)] = sg * fma(pf[0], a0, pf[1] * (a1 + a2));
      prep[D::vofs(T, q, 1)] = sg * fma(pf[2], a1, pf[3] * a2);
      prep[D::vofs(T, q, 2)] = sg * pf[4] * a2;
      prep[D::vofs(T, q, 3)] = sg * pf[4] * dq;
    }
  }
}

struct Conv3Params {
  const double* __restrict__ tab;
  const double* __restrict__ rtab;    // face trace maps R[4][NFD][NBS]
  const double* __restrict__ prep;    // point-major SoA (PREP, NT)
  const double* __restrict__ w;       // (NT, NB)
  const double* __restrict__ inflow;  // (NBF, NF, 3) or nullptr
  const int32_t* __restrict__ code;   // (NT, 4)
  const double* __restrict__ minv;    // (NT,) 6/|detJ|
  double* __restrict__ out;
  StageParams st;
  int nt;
  int ps;    // SoA stride of the face slots (prep3_stride)
  int prep_dep;   // 1: launched (PDL) right after the prep: stage its rows after griddepcontrol.wait
  int rev;        // 1: sweep the element blocks last to first (alternates from launch to launch)
};

// one thread per (element, component); warp w of the CTA = component w of 32
// consecutive elements, so prep reads are coalesced and tables are uniform
template <int K, int MODE>
__global__ void __launch_bounds__(96, HDGC_3D_MINB)
conv3d_kernel(Conv3Params p) {
  using D = Dims3<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NQ = D::NQ, NF = D::NF;
  if (MODE == MODE_STAGE && stage_stopped(p.st)) return;   // converged Richardson iteration
  const int c = threadIdx.x / D::EPB;
  // alternating sweeps (Conv3Params::rev, as in conv2d_sf_kernel): the rows the
  // previous kernel touched last are read first, while they are still in L2
  const int tile = p.rev ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int T0 = tile * D::EPB + (threadIdx.x % D::EPB);
  const bool active = T0 < p.nt;
  const int T = active ? T0 : p.nt - 1;
  const double* tab = p.tab;
  const size_t nt = (size_t)p.ps;   // SoA stride of the face slots
  // smem: face trace maps R[4][NFD][NBS] and per-thread w_c / neighbour columns
  extern __shared__ __align__(16) double sm3[];
  double* s_R = sm3;                     // [4][NFD][NBS]
  double* s_wo = sm3 + D::RTAB;          // [NBS][96]
  double* s_wn = s_wo + NBS * 96;        // [NBS][96]
  double* s_rb = s_wn + NBS * 96;        // [NRB][VROW][32]: staged volume rows (ring)
  __shared__ __align__(8) uint64_t rbar[D::NRB];   // full: the row has landed (TMA tx count)
  __shared__ __align__(8) uint64_t ebar[D::NRB];   // empty: all three warps have consumed it
  hdgc_debug_prologue(sm3, D::SMEM / (int)sizeof(double));
  // The volume coefficients of the CTA's 32 elements arrive row by row by TMA
  // bulk copy (one contiguous VROW x 32 block per collapsed row) into a ring of
  // NRB buffers: the three component warps share one copy instead of each
  // issuing 4 n loads per row.  Producer / consumer mbarriers: each warp
  // arrives on the buffer's "empty" barrier once its FMAs have consumed the
  // row; thread 0 waits for the three arrivals, fences the async proxy (WAR
  // against the generic-proxy reads) and refills the buffer NRB rows ahead.
  // Nothing here depends on the previous kernel, so the first NRB rows go
  // before griddepcontrol.wait.
  const double* vtile = p.prep + (size_t)tile * D::NROW * D::RBUF;
  auto issue_first_rows = [&]() {
#pragma unroll
    for (int r = 0; r < D::NRB && r < D::NROW; ++r) {
      mbar_arrive_expect_tx(&rbar[r], (uint32_t)(D::RBUF * sizeof(double)));
      bulk_g2s(s_rb + r * D::RBUF, vtile + (size_t)r * D::RBUF, (uint32_t)(D::RBUF * sizeof(double)), &rbar[r]);
    }
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < D::NRB; ++b) {
      mbar_init(&rbar[b], 1);
      if (D::RINGMB) mbar_init(&ebar[b], 3);
    }
    fence_mbar_init();
    if (!p.prep_dep) issue_first_rows();
  }
  {
    // trace maps: every load of this thread in flight before the smem stores
    constexpr int TOT = 4 * D::NFD * NBS, LOADS = (TOT + D::THREADS - 1) / D::THREADS;
    double v[LOADS];
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = threadIdx.x + r * D::THREADS;
      v[r] = i < TOT ? __ldg(p.rtab + i) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int i = threadIdx.x + r * D::THREADS;
      const int f = i / (D::NFD * NBS);
      if (i < TOT) s_R[f * D::RSTR + (i - f * D::NFD * NBS)] = v[r];
    }
  }
  // neighbour codes and the inflow-face mask of the face stage, loaded now so
  // their latency hides behind the volume term (not dependent loads after it)
  const int4 codes4 = __ldg(reinterpret_cast<const int4*>(p.code) + T);
  pdl_wait();   // w (and x) come from the previous update kernel under PDL (common.cuh)
  if (p.prep_dep && threadIdx.x == 0) issue_first_rows();   // the rows are the previous (prep) grid's output
  pdl_trigger();
  const double fmask_d = __ldg(p.prep + (size_t)D::P_MASK * nt + T);
  constexpr bool SR = HDGC_3D_SMEM_R;
  // SR: w_c from smem (s_wo) and the volume accumulators in smem (s_wn doubles as
  // s_r until the face loop), so the sum-factorisation state fits in 136 registers
  double* s_r = s_wn;
  double wo[SR ? 1 : NBS], r[NBS];
#pragma unroll
  for (int m = 0; m < NBS; ++m) {
    const double x = __ldg(p.w + (size_t)T * NB + c * NBS + m);
    if constexpr (!SR) wo[m] = x;
    s_wo[m * 96 + threadIdx.x] = x;
    if constexpr (SR) s_r[m * 96 + threadIdx.x] = 0.0;
    else r[m] = 0.0;
  }
  __syncthreads();
  auto W = [&](int m) -> double { if constexpr (SR) return s_wo[m * 96 + threadIdx.x]; else return wo[m]; };
  // ---- volume, sum-factorised over the collapsed rule (c outer, b, a inner):
  //   G_ij(c) = sum_l w_ijl C_ijl(c),  H_i(b,c) = sum_j G_ij(c) B_ij(b),
  //   w(a,b,c) = sum_i A_i(a) H_i(b,c)  (and the a-, b-, c-derivatives),
  //   g = alpha w_a + beta w_b + gamma w_c + delta w, then the transpose chain.
  {
    using S = SF3<K>;
    constexpr int N = S::N, NE = S::NE, NPAIR = S::NPAIR;
    const double* Cs = c_sf3d;
#pragma unroll 1
    for (int ic = 0; ic < N; ++ic) {
      const double* Cc = Cs + S::C_C + ic * NBS;
      const double* Ccd = Cs + S::C_CD + ic * NBS;
      double G[NPAIR], Gc[NPAIR], K2[NPAIR];
#pragma unroll
      for (int i = 0; i <= K; ++i)
#pragma unroll
        for (int j = 0; j <= K - i; ++j) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int l = 0; l <= K - i - j; ++l) {
            const int m = midx3(i, j, l);
            const double x = W(m);
            s0 = fma(x, Cc[m], s0);
            s1 = fma(x, Ccd[m], s1);
          }
          G[pidx(i, j)] = s0;
          Gc[pidx(i, j)] = s1;
          K2[pidx(i, j)] = 0.0;
        }
#pragma unroll 1
      for (int ib = 0; ib < N; ++ib) {
        const double* Bb = Cs + S::C_B + ib * NPAIR;
        const double* Bbd = Cs + S::C_BD + ib * NPAIR;
        // the row's flux-form coefficients from the staged row buffer
        const int row = ic * N + ib;
        const int rbuf = row % D::NRB;
        const uint32_t rpar = (uint32_t)(row / D::NRB) & 1u;
        mbar_wait(&rbar[rbuf], rpar);
        const double* rb = s_rb + rbuf * D::RBUF + (threadIdx.x & 31);
        double pal[N], pbe[N], pga[N], pde[N];
#pragma unroll
        for (int ia = 0; ia < N; ++ia) {
          pal[ia] = rb[(0 * N + ia) * 32];
          pbe[ia] = rb[(1 * N + ia) * 32];
          pga[ia] = rb[(2 * N + ia) * 32];
          pde[ia] = rb[(3 * N + ia) * 32];
        }

        double H[NE], Hb[NE], Hc[NE], K1[NE];
#pragma unroll
        for (int i = 0; i <= K; ++i) {
          double h = 0.0, hb = 0.0, hc = 0.0;
#pragma unroll
          for (int j = 0; j <= K - i; ++j) {
            const int pp = pidx(i, j);
            h = fma(G[pp], Bb[pp], h);
            hb = fma(G[pp], Bbd[pp], hb);
            hc = fma(Gc[pp], Bb[pp], hc);
          }
          H[i] = h; Hb[i] = hb; Hc[i] = hc; K1[i] = 0.0;
        }
#if HDGC_3D_SYM
        // The a points are Gauss-Legendre on [0, 1] and A_i(a) = P_i(2a - 1):
        // A_i(N-1-ia) = (-1)^i A_i(ia), A'_i(N-1-ia) = (-1)^(i+1) A'_i(ia) (checked
        // on the uploaded tables in create3d): values at a mirror pair from the
        // even-i / odd-i partial sums, the test through g(ia) +- g(N-1-ia).
#pragma unroll
        for (int ia = 0; ia < N / 2; ++ia) {
          const int i2 = N - 1 - ia;
          double ve = 0.0, vo = 0.0, be = 0.0, bo = 0.0, ce = 0.0, co = 0.0, as = 0.0, aa = 0.0;
#pragma unroll
          for (int i = 0; i <= K; ++i) {
            const double Ai = Cs[S::C_A + ia * NE + i], Adi = Cs[S::C_AD + ia * NE + i];
            if (i & 1) {
              vo = fma(Ai, H[i], vo);
              bo = fma(Ai, Hb[i], bo);
              co = fma(Ai, Hc[i], co);
              as = fma(Adi, H[i], as);
            } else {
              ve = fma(Ai, H[i], ve);
              be = fma(Ai, Hb[i], be);
              ce = fma(Ai, Hc[i], ce);
              aa = fma(Adi, H[i], aa);
            }
          }
          const double g1 = fma(pal[ia], as + aa, fma(pbe[ia], be + bo, fma(pga[ia], ce + co, pde[ia] * (ve + vo))));
          const double g2 = fma(pal[i2], as - aa, fma(pbe[i2], be - bo, fma(pga[i2], ce - co, pde[i2] * (ve - vo))));
          const double gp = g1 + g2, gm = g1 - g2;
#pragma unroll
          for (int i = 0; i <= K; ++i) K1[i] = fma((i & 1) ? gm : gp, Cs[S::C_A + ia * NE + i], K1[i]);
        }
        if constexpr (N & 1) {
          constexpr int ia = N / 2;   // a = 1/2: odd-i values and even-i derivatives vanish
          double v = 0.0, va = 0.0, vb = 0.0, vc = 0.0;
#pragma unroll
          for (int i = 0; i <= K; ++i) {
            if (i & 1) va = fma(Cs[S::C_AD + ia * NE + i], H[i], va);
            else {
              const double Ai = Cs[S::C_A + ia * NE + i];
              v = fma(Ai, H[i], v);
              vb = fma(Ai, Hb[i], vb);
              vc = fma(Ai, Hc[i], vc);
            }
          }
          const double g = fma(pal[ia], va, fma(pbe[ia], vb, fma(pga[ia], vc, pde[ia] * v)));
#pragma unroll
          for (int i = 0; i <= K; i += 2) K1[i] = fma(g, Cs[S::C_A + ia * NE + i], K1[i]);
        }
#else
#pragma unroll
        for (int ia = 0; ia < N; ++ia) {
          double v = 0.0, va = 0.0, vb = 0.0, vc = 0.0;
#pragma unroll
          for (int i = 0; i <= K; ++i) {
            const double Ai = Cs[S::C_A + ia * NE + i];
            v = fma(Ai, H[i], v);
            va = fma(Cs[S::C_AD + ia * NE + i], H[i], va);
            vb = fma(Ai, Hb[i], vb);
            vc = fma(Ai, Hc[i], vc);
          }
          const double g = fma(pal[ia], va, fma(pbe[ia], vb, fma(pga[ia], vc, pde[ia] * v)));
#pragma unroll
          for (int i = 0; i <= K; ++i) K1[i] = fma(g, Cs[S::C_A + ia * NE + i], K1[i]);
        }
#endif
#pragma unroll
        for (int i = 0; i <= K; ++i)
#pragma unroll
          for (int j = 0; j <= K - i; ++j) K2[pidx(i, j)] = fma(K1[i], Bb[pidx(i, j)], K2[pidx(i, j)]);
        // this warp has consumed the row's coefficients (they fed the FMAs above)
        if constexpr (D::RINGMB) {
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(&ebar[rbuf]);
          if (threadIdx.x == 0 && row + D::NRB < D::NROW) {
            mbar_wait(&ebar[rbuf], rpar);   // all three warps done with the buffer
            fence_proxy_async();
            mbar_arrive_expect_tx(&rbar[rbuf], (uint32_t)(D::RBUF * sizeof(double)));
            bulk_g2s(s_rb + rbuf * D::RBUF, vtile + (size_t)(row + D::NRB) * D::RBUF,
                     (uint32_t)(D::RBUF * sizeof(double)), &rbar[rbuf]);
          }
          __syncwarp();
        } else {
          __syncthreads();   // generic-proxy reads of all warps before the async-proxy refill
          if (threadIdx.x == 0 && row + D::NRB < D::NROW) {
            fence_proxy_async();
            mbar_arrive_expect_tx(&rbar[rbuf], (uint32_t)(D::RBUF * sizeof(double)));
            bulk_g2s(s_rb + rbuf * D::RBUF, vtile + (size_t)(row + D::NRB) * D::RBUF,
                     (uint32_t)(D::RBUF * sizeof(double)), &rbar[rbuf]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i <= K; ++i)
#pragma unroll
        for (int j = 0; j <= K - i; ++j)
#pragma unroll
          for (int l = 0; l <= K - i - j; ++l) {
            const int m = midx3(i, j, l);
            if constexpr (SR) {
              double* rp = s_r + m * 96 + threadIdx.x;
              *rp = fma(K2[pidx(i, j)], Cc[m], *rp);
            } else {
              r[m] = fma(K2[pidx(i, j)], Cc[m], r[m]);
            }
          }
    }
  }
  if constexpr (SR) {
#pragma unroll
    for (int m = 0; m < NBS; ++m) r[m] = s_r[m * 96 + threadIdx.x];   // own column only: no barrier needed
  }
  // ---- faces: per-lane work list of inflow faces (the warp runs max_lane(count)
  //      iterations).  Traces are handled in the face's own P_k basis: the
  //      trace of a tet mode on face f is D_m(x_f(s,t)) = sum_n R_f[n][m] D2_n(s,t)
  //      exactly, so the jump coefficients are d = R_f2 w_nbr - R_f w_own (NFD
  //      numbers instead of NF point values), the jump at point q is
  //      sum_n d_n D2_n(q), and the test folds back through R_f^T.  Point q of
  //      the owner is point q of the neighbour (sorted tet vertices).
  {
    using S = SF3<K>;
    constexpr int NFD = D::NFD;
    const double* D2 = c_sf3d + S::C_D2;
    const int codes[4] = {codes4.x, codes4.y, codes4.z, codes4.w};
    unsigned fm = active ? (unsigned)fmask_d : 0u;
    if (p.inflow == nullptr) {
#pragma unroll
      for (int f = 0; f < 4; ++f)
        if (codes[f] < 0) fm &= ~(1u << f);   // exterior = own trace
    }
    const int nmine = __popc(fm);
    const int nmax = __reduce_max_sync(0xffffffffu, (unsigned)nmine);
#pragma unroll 1
    for (int j = 0; j < nmax; ++j) {
      const bool on = j < nmine;
      const int f = on ? __ffs(fm) - 1 : 0;
      if (on) fm &= fm - 1;
      const int code = on ? (f == 0 ? codes[0] : f == 1 ? codes[1] : f == 2 ? codes[2] : codes[3]) : -1;
      int f2 = 0;
      const double* infl = nullptr;
      if (code >= 0) {
        const double* g = p.w + (size_t)(code >> 2) * NB + c * NBS;
        f2 = code & 3;
        if constexpr (NBS % 2 == 0) {   // component rows are 16-byte aligned: half as many loads
          const double2* g2 = reinterpret_cast<const double2*>(g);
#pragma unroll
          for (int m = 0; m < NBS / 2; ++m) {
            const double2 t = __ldg(g2 + m);
            s_wn[(2 * m) * 96 + threadIdx.x] = t.x;
            s_wn[(2 * m + 1) * 96 + threadIdx.x] = t.y;
          }
        } else {
#pragma unroll
          for (int m = 0; m < NBS; ++m) s_wn[m * 96 + threadIdx.x] = __ldg(g + m);
        }
      } else {
#pragma unroll
        for (int m = 0; m < NBS; ++m) s_wn[m * 96 + threadIdx.x] = 0.0;
        if (on) infl = p.inflow + (size_t)(-1 - code) * NF * 3 + c;
      }
      const double* Rf = s_R + f * D::RSTR;
      const double* Rn = s_R + f2 * D::RSTR;
      double dl[NFD];
#pragma unroll
      for (int n = 0; n < NFD; ++n) dl[n] = 0.0;
#pragma unroll 4
      for (int m = 0; m < NBS; ++m) {
        const double wm = s_wo[m * 96 + threadIdx.x], wnm = s_wn[m * 96 + threadIdx.x];
#pragma unroll
        for (int n = 0; n < NFD; ++n) dl[n] = fma(wnm, Rn[n * NBS + m], fma(-wm, Rf[n * NBS + m], dl[n]));
      }
      // rho_n = sum_q s_q J(q) D2_n(q) with J = sum_n' dl_n' D2_n' (+ inflow data):
      // the velocity-only part is the frozen face matrix S_f[n][n'] = sum_q s_q D2_n D2_n'
      // (prep), so rho = S_f dl — NSYM independent loads instead of a dependent
      // loop over the NF face points
      double rho[NFD];
      {
        const double* Sf = p.prep + (size_t)(D::P_S + f * D::NSYM) * nt + T;
#pragma unroll
        for (int n = 0; n < NFD; ++n) rho[n] = 0.0;
#pragma unroll
        for (int n = 0; n < NFD; ++n)
#pragma unroll
          for (int n2 = n; n2 < NFD; ++n2) {
            const double sv = on ? __ldg(Sf + (size_t)(n * NFD - n * (n - 1) / 2 + (n2 - n)) * nt) : 0.0;
            rho[n] = fma(sv, dl[n2], rho[n]);
            if (n2 != n) rho[n2] = fma(sv, dl[n], rho[n2]);
          }
      }
      if (infl != nullptr) {
        // boundary face with exterior data: + sum_q s_q g(q) D2_n(q)
        const double* sf = p.prep + (size_t)(4 * NQ + f * NF) * nt + T;
#pragma unroll 1
        for (int q = 0; q < NF; ++q) {
          const double sg = __ldg(sf + (size_t)q * nt) * __ldg(infl + 3 * q);
#pragma unroll
          for (int n = 0; n < NFD; ++n) rho[n] = fma(sg, D2[q * NFD + n], rho[n]);
        }
      }
#pragma unroll
      for (int m = 0; m < NBS; ++m) {
        double acc = r[m];
#pragma unroll
        for (int n = 0; n < NFD; ++n) acc = fma(Rf[n * NBS + m], rho[n], acc);
        r[m] = acc;
      }
    }
  }
  // APPLY / SUBSTEP: the CTA's 32 output rows go through smem (the w columns
  // are dead after the face stage) and one bulk store, instead of 20 strided
  // 8-byte stores per thread
  if constexpr (MODE == MODE_APPLY || MODE == MODE_SUBSTEP) {
    double v[NBS];
    if (MODE == MODE_APPLY) {
#pragma unroll
      for (int m = 0; m < NBS; ++m) v[m] = r[m];
    } else {
      const double cm = p.st.c * __ldg(p.minv + T);
      double chk = 0.0;
#pragma unroll
      for (int m = 0; m < NBS; ++m) {
        v[m] = fma(cm, r[m], W(m));
        chk += v[m];
      }
      guard_finite(p.st.flag, chk);
    }
    __syncthreads();   // every warp is done with s_wo / s_wn
    const int tb = tile * D::EPB, nel = min(D::EPB, p.nt - tb), e = threadIdx.x % D::EPB;
    double* s_out = s_wo;   // [EPB][NB] row-major (fits in s_wo | s_wn)
    if (active) {
#pragma unroll
      for (int m = 0; m < NBS; ++m) s_out[e * NB + c * NBS + m] = v[m];
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(p.out + (size_t)tb * NB, s_out, (uint32_t)(nel * NB * sizeof(double)));
      bulk_wait_read();
    }
    return;
  }
  if (!active) return;
  double* og = p.out + (size_t)T * NB + c * NBS;
  if (MODE == MODE_SUBSTEP) {
    const double cm = p.st.c * __ldg(p.minv + T);
    double chk = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      const double v = fma(cm, r[m], W(m));
      og[m] = v;
      chk += v;
    }
    guard_finite(p.st.flag, chk);
  } else if (MODE == MODE_STAGE) {
    const double mi = __ldg(p.minv + T);
    const double cm = p.st.c * mi;
    {
      const double* xg = p.st.x + (size_t)T * NB + c * NBS;
      const double tm = -p.st.tau * mi;
      double acc = 0.0, chk = 0.0;
#pragma unroll
      for (int m = 0; m < NBS; ++m) {
        const double xv = __ldg(xg + m);
        const double wm = W(m);
        const double v = fma(p.st.b, xv, fma(cm, r[m], p.st.a * wm));
        og[m] = v;
        chk += v;
        const double res = fma(tm, r[m], xv - wm);
        acc = fma(res, res, acc);
      }
      guard_finite(p.st.flag, chk);
      if (p.st.rn) p.st.rn[3 * (size_t)T + c] = acc;
    }
  } else {
#pragma unroll
    for (int m = 0; m < NBS; ++m) og[m] = r[m];
  }
}

// I (BDM -> V_h) and I^T, one thread per (element, row); P = J/detJ (3x3, SoA)
template <int K, bool TRANSPOSE>
__global__ void __launch_bounds__(256)
transfer3d_kernel(const double* __restrict__ tab, const double* __restrict__ piola, int nt,
                  const double* __restrict__ in, double* __restrict__ out) {
  using D = Dims3<K>;
  constexpr int NB = D::NB, NBS = D::NBS;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)nt * NB) return;
  const int T = (int)(gid / NB);
  const int r = (int)(gid - (long long)T * NB);
  double P[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) P[i] = __ldg(piola + (size_t)i * nt + T);
  const double* coef = tab + D::OFF_COEF;
  const double* x = in + (size_t)T * NB;
  if (!TRANSPOSE) {
    const int c = r / NBS, m = r - c * NBS;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      const double xj = __ldg(x + j);
      a0 = fma(__ldg(coef + (size_t)m * NB + j), xj, a0);
      a1 = fma(__ldg(coef + (size_t)(NBS + m) * NB + j), xj, a1);
      a2 = fma(__ldg(coef + (size_t)(2 * NBS + m) * NB + j), xj, a2);
    }
    out[gid] = fma(P[3 * c], a0, fma(P[3 * c + 1], a1, P[3 * c + 2] * a2));
  } else {
    double a = 0.0;
#pragma unroll 4
    for (int m = 0; m < NBS; ++m) {
      const double x0 = __ldg(x + m), x1 = __ldg(x + NBS + m), x2 = __ldg(x + 2 * NBS + m);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double s = fma(P[d], x0, fma(P[3 + d], x1, P[6 + d] * x2));   // sum_c P[c][d] x_c
        a = fma(__ldg(coef + (size_t)(d * NBS + m) * NB + r), s, a);
      }
    }
    out[gid] = a;
  }
}

// max |J u_hat / detJ| over elements x volume points, one thread per element
template <int K>
__global__ void __launch_bounds__(128)
maxspeed3d_kernel(const double* __restrict__ tab, const double* __restrict__ piola, int nt,
                  const double* __restrict__ u, unsigned long long* __restrict__ out) {
  using D = Dims3<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NQ = D::NQ;
  const int T = blockIdx.x * blockDim.x + threadIdx.x;
  double best = 0.0;
  if (T < nt) {
    double x[NB], uh[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) x[j] = __ldg(u + (size_t)T * NB + j);
#pragma unroll 1
    for (int i = 0; i < NB; ++i) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) a = fma(__ldg(tab + D::OFF_COEF + i * NB + j), x[j], a);
      uh[i] = a;
    }
    double P[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) P[i] = __ldg(piola + (size_t)i * nt + T);
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll 4
      for (int m = 0; m < NBS; ++m) {
        const double d = __ldg(tab + D::OFF_VD + q * NBS + m);
        a0 = fma(uh[m], d, a0);
        a1 = fma(uh[NBS + m], d, a1);
        a2 = fma(uh[2 * NBS + m], d, a2);
      }
      double s2 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double v = fma(P[3 * c], a0, fma(P[3 * c + 1], a1, P[3 * c + 2] * a2));
        s2 = fma(v, v, s2);
      }
      best = fmax(best, sqrt(s2));
    }
  }
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

#endif  // HDGC_ORDER3

}  // namespace hdgc
