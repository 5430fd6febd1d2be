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
  static constexpr int PREP = 4 * NQ + 4 * NF;
  static constexpr int EPB = 32;                                     // elements per CTA
  static constexpr int THREADS = 3 * EPB;                            // one warp per component
};

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
__global__ void geometry3d_kernel(const double* __restrict__ V, const int64_t* __restrict__ tet, int nt,
                                  double* __restrict__ piola, double* __restrict__ minv,
                                  double* __restrict__ sgn, int* __restrict__ bad);

struct Prep3Params {
  const double* __restrict__ tab;
  const double* __restrict__ u;
  const double* __restrict__ sgn;
  double* __restrict__ prep;
  int nt;
};

template <int K>
__global__ void __launch_bounds__(128)
prep3d_kernel(Prep3Params p) {
  using D = Dims3<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NBS1 = D::NBS1, NFD = D::NFD, NQ = D::NQ, NF = D::NF;
  const int T = blockIdx.x * blockDim.x + threadIdx.x;
  if (T >= p.nt) return;
  const double* tab = p.tab;
  const double sg = __ldg(p.sgn + T);
  const size_t nt = (size_t)p.nt;
  double x[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) x[j] = __ldg(p.u + (size_t)T * NB + j);
  // inflow weights from the face dofs (first 4*NFD dofs, face-major)
#pragma unroll 1
  for (int f = 0; f < 4; ++f) {
    const double len = __ldg(tab + D::OFF_FLEN + f);
#pragma unroll 1
    for (int q = 0; q < NF; ++q) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < NFD; ++m) a = fma(x[f * NFD + m], __ldg(tab + D::OFF_FL + q * NFD + m), a);
      const double F = sg * a * len;
      p.prep[(size_t)(4 * NQ + f * NF + q) * nt + T] = F < 0.0 ? __ldg(tab + D::OFF_FW + q) * F : 0.0;
    }
  }
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
    const double wq = sg * __ldg(tab + D::OFF_VW + q);
    p.prep[(size_t)q * nt + T] = wq * a0;
    p.prep[(size_t)(NQ + q) * nt + T] = wq * a1;
    p.prep[(size_t)(2 * NQ + q) * nt + T] = wq * a2;
    p.prep[(size_t)(3 * NQ + q) * nt + T] = wq * dq;
  }
}

struct Conv3Params {
  const double* __restrict__ tab;
  const double* __restrict__ prep;    // point-major SoA (PREP, NT)
  const double* __restrict__ w;       // (NT, NB)
  const double* __restrict__ inflow;  // (NBF, NF, 3) or nullptr
  const int32_t* __restrict__ code;   // (NT, 4)
  const double* __restrict__ minv;    // (NT,) 6/|detJ|
  double* __restrict__ out;
  double dt;
  int nt;
};

// one thread per (element, component); warp w of the CTA = component w of 32
// consecutive elements, so prep reads are coalesced and tables are uniform
template <int K, int MODE>
__global__ void __launch_bounds__(96)
conv3d_kernel(Conv3Params p) {
  using D = Dims3<K>;
  constexpr int NB = D::NB, NBS = D::NBS, NQ = D::NQ, NF = D::NF;
  const int c = threadIdx.x / D::EPB;
  const int T = blockIdx.x * D::EPB + (threadIdx.x % D::EPB);
  if (T >= p.nt) return;
  const double* tab = p.tab;
  const size_t nt = (size_t)p.nt;
  double wo[NBS], r[NBS];
#pragma unroll
  for (int m = 0; m < NBS; ++m) {
    wo[m] = __ldg(p.w + (size_t)T * NB + c * NBS + m);
    r[m] = 0.0;
  }
  // ---- volume
#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    const double* Dq = tab + D::OFF_VD + q * NBS;
    const double* Gq = tab + D::OFF_VG + q * NBS * 3;
    double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
    for (int m = 0; m < NBS; ++m) {
      const double wm = wo[m];
      v = fma(wm, __ldg(Dq + m), v);
      gx = fma(wm, __ldg(Gq + 3 * m), gx);
      gy = fma(wm, __ldg(Gq + 3 * m + 1), gy);
      gz = fma(wm, __ldg(Gq + 3 * m + 2), gz);
    }
    const double ax = __ldg(p.prep + (size_t)q * nt + T);
    const double ay = __ldg(p.prep + (size_t)(NQ + q) * nt + T);
    const double az = __ldg(p.prep + (size_t)(2 * NQ + q) * nt + T);
    const double ga = __ldg(p.prep + (size_t)(3 * NQ + q) * nt + T);
    const double g = fma(ax, gx, fma(ay, gy, fma(az, gz, ga * v)));
#pragma unroll
    for (int m = 0; m < NBS; ++m) r[m] = fma(g, __ldg(Dq + m), r[m]);
  }
  // ---- faces: upwind jump at inflow points
#pragma unroll 1
  for (int f = 0; f < 4; ++f) {
    const double* sf = p.prep + (size_t)(4 * NQ + f * NF) * nt + T;
    bool any = false;
#pragma unroll 1
    for (int q = 0; q < NF; ++q) any |= __ldg(sf + (size_t)q * nt) != 0.0;
    if (!any) continue;
    const int code = __ldg(p.code + (size_t)T * 4 + f);
    double wn[NBS];
    int f2 = 0;
    const double* infl = nullptr;
    if (code >= 0) {
      const double* g = p.w + (size_t)(code >> 2) * NB + c * NBS;
      f2 = code & 3;
#pragma unroll
      for (int m = 0; m < NBS; ++m) wn[m] = __ldg(g + m);
    } else if (p.inflow != nullptr) {
      infl = p.inflow + (size_t)(-1 - code) * NF * 3 + c;
    } else {
      continue;
    }
    const double* Df = tab + D::OFF_FD + f * NF * NBS;
    const double* Dn = tab + D::OFF_FD + f2 * NF * NBS;
#pragma unroll 1
    for (int q = 0; q < NF; ++q) {
      const double sq = __ldg(sf + (size_t)q * nt);
      if (sq == 0.0) continue;
      double own = 0.0, ext = 0.0;
#pragma unroll
      for (int m = 0; m < NBS; ++m) own = fma(wo[m], __ldg(Df + q * NBS + m), own);
      if (code >= 0) {
#pragma unroll
        for (int m = 0; m < NBS; ++m) ext = fma(wn[m], __ldg(Dn + q * NBS + m), ext);
      } else {
        ext = __ldg(infl + 3 * q);
      }
      const double s = sq * (ext - own);
#pragma unroll
      for (int m = 0; m < NBS; ++m) r[m] = fma(s, __ldg(Df + q * NBS + m), r[m]);
    }
  }
  double* og = p.out + (size_t)T * NB + c * NBS;
  if (MODE == MODE_SUBSTEP) {
    const double sc = p.dt * __ldg(p.minv + T);
#pragma unroll
    for (int m = 0; m < NBS; ++m) og[m] = fma(-sc, r[m], wo[m]);
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

}  // namespace hdgc
