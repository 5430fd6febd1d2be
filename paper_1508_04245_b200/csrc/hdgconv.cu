// hdgconv.cu — C ABI, device context and setup/transfer kernels for the
// B200 fp64 upwind-DG convection apply.  See include/hdgconv.h.
#include "../../include/hdgconv.h"

#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <cstdint>
#include <cmath>
#include <initializer_list>
#include <string>
#include <vector>


#include "common.cuh"
#include "context.cuh"
#include "conv3d.cuh"

using namespace hdgc;

// ---------------------------------------------------------------------------
// error plumbing

static thread_local std::string g_err;

int hdgc_set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}


// ---------------------------------------------------------------------------
// context

int hdgc_dev_alloc(hdgc_ctx* c, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return hdgc_set_err(HDGC_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  c->bytes += (int64_t)bytes;
  return HDGC_OK;
}

// Modal velocity rows d_modal[T][r] = sum_j M[r][j] u[T][j], r < nr, with M
// = [coef ; divm] (PB:357-378): one thread per (element, row), M read through
// L1 (threads of a warp share rows), u row broadcast.  Used by max_speed and
// the HDGC_PREP=0 development prep; the hot paths stage this product on the
// FP64 tensor cores inside the tile preps.
__global__ void __launch_bounds__(256) modal_rows_kernel(const double* __restrict__ M, int nr, int nb,
                                                         const double* __restrict__ u, int nt,
                                                         double* __restrict__ out) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)nt * nr) return;
  const int T = (int)(gid / nr), r = (int)(gid - (long long)T * nr);
  const double* mr = M + (size_t)r * nb;
  const double* x = u + (size_t)T * nb;
  double a = 0.0;
#pragma unroll 6
  for (int j = 0; j < nb; ++j) a = fma(__ldg(mr + j), __ldg(x + j), a);
  out[gid] = a;
}

int hdgc_modal_gemm(hdgc_ctx* c, const double* u, int nb, int nr, size_t off, cudaStream_t st) {
  const long long work = (long long)c->nt * nr;
  modal_rows_kernel<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(c->d_tab + off, nr, nb, u, c->nt, c->d_modal);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

// out = a x + b y (extrapolated velocity)
__global__ void axpby_kernel(const double* __restrict__ x, const double* __restrict__ y, double a, double b,
                             double* __restrict__ out, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fma(a, x[i], b * y[i]);
}

// Richardson control on the device (hdgc_richardson).  ctl (ints): [0] stop
// (converged or blown up), [1] iteration it stopped at, [2] blow-up, [3]
// arrival counter of the reduction.  Each iteration's reduction sums the
// per-(element, component) residual sums rn in a fixed order — RED_CTAS
// contiguous chunks, each a fixed block tree, then the chunk partials in
// index order by whichever CTA arrives last — so norms, stop decisions and
// iteration counts are bitwise reproducible; it stores ||res_it|| into
// norms[it] and raises the stop flag at the first it with
// ||res_it|| <= rho ||res_0|| (or a non-finite norm).  Update kernels queued
// after the flag is raised return at entry (StageParams::stop).
constexpr int RED_CTAS = 256, RED_THREADS = 256;

__device__ __forceinline__ double block_sum_fixed(double a, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  }
  return a;   // valid in thread 0
}

__global__ void __launch_bounds__(RED_THREADS) richardson_reduce_kernel(const double* __restrict__ rn, size_t n, int it,
                                                                        double rho, double* part, double* norms,
                                                                        int* ctl) {
  __shared__ double red[RED_THREADS / 32];
  __shared__ int last;
  if (*(volatile int*)ctl != 0) return;   // stopped at an earlier iteration: no-op
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t b0 = min(n, (size_t)blockIdx.x * per), b1 = min(n, b0 + per);
  double a = 0.0;
  for (size_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) a += rn[i];
  a = block_sum_fixed(a, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = a;
    __threadfence();
    last = atomicAdd(&ctl[3], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __syncthreads();
  a = threadIdx.x < gridDim.x ? ((volatile double*)part)[threadIdx.x] : 0.0;
  a = block_sum_fixed(a, red);
  if (threadIdx.x == 0) {
    const double r = sqrt(a);
    norms[it] = r;
    ctl[3] = 0;
    const double r0 = it == 0 ? r : norms[0];
    if (!isfinite(r)) {
      ctl[2] = 1; ctl[1] = it; __threadfence(); ctl[0] = 1;
    } else if (r <= rho * r0) {
      ctl[1] = it; __threadfence(); ctl[0] = 1;
    }
  }
}

// Richardson residual norm, part 2 (fused path): one CTA adds the CTA
// partials of the STAGE kernel before it in index order and takes the stop
// decision.  Launched with PDL: it lets the next STAGE kernel launch at once
// (that one stages its prep / x tiles, then waits in griddepcontrol.wait for
// this kernel), and itself waits for the STAGE kernel to complete.
__global__ void __launch_bounds__(1024) richardson_final_kernel(const double* __restrict__ part, int n, int it,
                                                                double rho, double* norms, int* ctl) {
  __shared__ double red[32];
  pdl_trigger();
  pdl_wait();
  if (*(volatile int*)ctl != 0) return;   // stopped at an earlier iteration: no-op
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) a += part[i];
  a = block_sum_fixed(a, red);
  if (threadIdx.x == 0) {
    const double r = sqrt(a);
    norms[it] = r;
    const double r0 = it == 0 ? r : norms[0];
    if (!isfinite(r)) {
      ctl[2] = 1; ctl[1] = it; ctl[0] = 1;
    } else if (r <= rho * r0) {
      ctl[1] = it; ctl[0] = 1;
    }
  }
}

// global H(div) gather / scatter (fespace dof map)
__global__ void gather_kernel(const int32_t* __restrict__ dof, const double* __restrict__ fac,
                              const double* __restrict__ g, double* __restrict__ out, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fac[i] * __ldg(g + dof[i]);
}
__global__ void scatter_kernel(const int32_t* __restrict__ inv, const double* __restrict__ invf,
                               const double* __restrict__ r, double* __restrict__ out, size_t ndof) {
  const size_t d = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= ndof) return;
  const int i0 = inv[2 * d], i1 = inv[2 * d + 1];
  double a = invf[2 * d] * __ldg(r + i0);
  if (i1 >= 0) a += invf[2 * d + 1] * __ldg(r + i1);
  out[d] = a;
}

// ---------------------------------------------------------------------------
// setup kernels (on-device geometry / adjacency precompute)

// mesh validation flag: the first error found wins (kernels run in order
// geometry -> codes -> check_codes, so the most basic error is reported)
__device__ __forceinline__ void set_bad(int* bad, int code) { atomicCAS(bad, 0, code); }

// Per-element affine geometry: J = [v1-v0, v2-v0] (columns = edges, mesh2d.py:135-150),
// Piola factor J/detJ and the V_h mass inverse 2/detJ.
__global__ void geometry2d_kernel(const double* __restrict__ V, const int64_t* __restrict__ tri,
                                  int nt, int nv, double* __restrict__ piola, double* __restrict__ minv,
                                  int* __restrict__ bad) {
  int T = blockIdx.x * blockDim.x + threadIdx.x;
  if (T >= nt) return;
  const int64_t a = tri[3 * (size_t)T], b = tri[3 * (size_t)T + 1], c = tri[3 * (size_t)T + 2];
  if (a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv) { set_bad(bad, 5); return; }
  const double x0 = V[2 * a], y0 = V[2 * a + 1];
  const double j00 = V[2 * b] - x0, j10 = V[2 * b + 1] - y0;
  const double j01 = V[2 * c] - x0, j11 = V[2 * c + 1] - y0;
  const double det = j00 * j11 - j01 * j10;
  if (!(det > 0.0)) set_bad(bad, 1);
  const double id = 1.0 / det;
  piola[T] = j00 * id;
  piola[(size_t)nt + T] = j01 * id;
  piola[2 * (size_t)nt + T] = j10 * id;
  piola[3 * (size_t)nt + T] = j11 * id;
  minv[T] = 2.0 * id;
}

// 3D: J = [v1-v0, v2-v0, v3-v0], Piola J/detJ (9, NT) row-major, 6/|detJ|, sign(detJ)
__global__ void hdgc::geometry3d_kernel(const double* __restrict__ V, const int64_t* __restrict__ tet, int nt, int nv,
                                        double* __restrict__ piola, double* __restrict__ minv,
                                        double* __restrict__ sgn, int* __restrict__ bad) {
  int T = blockIdx.x * blockDim.x + threadIdx.x;
  if (T >= nt) return;
  int64_t v[4];
  for (int i = 0; i < 4; ++i) v[i] = tet[4 * (size_t)T + i];
  for (int i = 0; i < 4; ++i)
    if (v[i] < 0 || v[i] >= nv) { set_bad(bad, 5); return; }
  // conv3d.cuh pairs face point q of both neighbours, which needs every tet's
  // vertex ids in ascending order (shared faces then have the same vertex order)
  if (!(v[0] < v[1] && v[1] < v[2] && v[2] < v[3])) { set_bad(bad, 6); return; }
  double J[9];
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d) J[3 * c + d] = V[3 * v[d + 1] + c] - V[3 * v[0] + c];
  const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                     J[2] * (J[3] * J[7] - J[4] * J[6]);
  if (!(fabs(det) > 0.0)) set_bad(bad, 1);
  const double id = 1.0 / det;
  for (int i = 0; i < 9; ++i) piola[(size_t)i * nt + T] = J[i] * id;
  minv[T] = 6.0 / fabs(det);
  sgn[T] = det > 0.0 ? 1.0 : -1.0;
}

// boundary flag per facet
__global__ void bflag_kernel(const int64_t* __restrict__ fe, int nfac, int* __restrict__ flag) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nfac) flag[f] = fe[2 * (size_t)f + 1] < 0 ? 1 : 0;
}

// in-place exclusive scan of n ints, single CTA of 1024 threads (setup only):
// each thread owns a contiguous run, the 1024 run sums are scanned with warp
// shuffles, then each run is rewritten with its offset (two passes over a;
// 178 us at 197k facets, the earlier chunked Hillis-Steele version 320 us)
__global__ void scan_kernel(int* __restrict__ a, int n, int* __restrict__ total) {
  __shared__ int wsum[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (n + 1023) / 1024;
  const int b0 = min(n, t * per), b1 = min(n, b0 + per);
  int s = 0;
  for (int i = b0; i < b1; ++i) s += a[i];
  int x = s;   // inclusive warp scan of the run sums
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int v = wsum[lane];
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += y;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  int excl = x - s + (warp > 0 ? wsum[warp - 1] : 0);
  for (int i = b0; i < b1; ++i) {
    const int v = a[i];
    a[i] = excl;
    excl += v;
  }
  if (t == 1023) *total = wsum[31];
}

// element-owned neighbour codes from the facet arrays (mesh2d.py:178-207)
// The code array is pre-filled with CODE_UNSET; every (element, local facet)
// must be claimed exactly once (atomicExch returns the previous value), and
// check_codes_kernel flags any slot left unset.
constexpr int32_t CODE_UNSET = (int32_t)0x80808080;
__global__ void codes_kernel(const int64_t* __restrict__ fe, const int64_t* __restrict__ fl,
                             const int* __restrict__ slot, int nfac, int nt, int faces_per_elem,
                             int32_t* __restrict__ code, int* __restrict__ bad) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfac) return;
  const int64_t e0 = fe[2 * (size_t)f], e1 = fe[2 * (size_t)f + 1];
  const int64_t l0 = fl[2 * (size_t)f], l1 = fl[2 * (size_t)f + 1];
  if (e0 < 0 || e0 >= nt || l0 < 0 || l0 >= faces_per_elem) { set_bad(bad, 2); return; }
  if (e1 >= 0) {
    if (e1 >= nt || e1 == e0 || l1 < 0 || l1 >= faces_per_elem) { set_bad(bad, 2); return; }
    if (atomicExch(&code[e0 * faces_per_elem + l0], (int32_t)((e1 << 2) | l1)) != CODE_UNSET) set_bad(bad, 3);
    if (atomicExch(&code[e1 * faces_per_elem + l1], (int32_t)((e0 << 2) | l0)) != CODE_UNSET) set_bad(bad, 3);
  } else {
    if (atomicExch(&code[e0 * faces_per_elem + l0], -1 - slot[f]) != CODE_UNSET) set_bad(bad, 3);
  }
}
__global__ void check_codes_kernel(const int32_t* __restrict__ code, size_t n, int* __restrict__ bad) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && code[i] == CODE_UNSET) set_bad(bad, 4);
}

namespace hdgc {
HDGC_DECLARE_ORDER(1)
HDGC_DECLARE_ORDER(2)
HDGC_DECLARE_ORDER(3)
HDGC_DECLARE_ORDER(4)
HDGC_DECLARE_ORDER(5)
HDGC_DECLARE_ORDER(6)
HDGC_DECLARE_ORDER(7)
HDGC_DECLARE_ORDER(8)
}  // namespace hdgc

#define HDGC_K_SWITCH(k, CALL)                        \
  switch (k) {                                        \
    case 1: { constexpr int KK = 1; return CALL; }    \
    case 2: { constexpr int KK = 2; return CALL; }    \
    case 3: { constexpr int KK = 3; return CALL; }    \
    case 4: { constexpr int KK = 4; return CALL; }    \
    case 5: { constexpr int KK = 5; return CALL; }    \
    case 6: { constexpr int KK = 6; return CALL; }    \
    case 7: { constexpr int KK = 7; return CALL; }    \
    case 8: { constexpr int KK = 8; return CALL; }    \
    default: return hdgc_set_err(HDGC_EUNSUP, "order k=%d not supported (1..8)", k); \
  }

// ---------------------------------------------------------------------------
// Curved elements (hdgc_set_curved).  A few
// elements along a curved boundary: small generic kernels, one thread per
// (curved element, component) or (curved element, row).

// minv[T] = -(slot + 1) flags a curved element for the update kernels
__global__ void mark_curved_kernel(const int32_t* __restrict__ el, int n, double* __restrict__ minv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) minv[el[i]] = -(double)(i + 1);
}

// update epilogues of the curved rows with the full block inverse:
//   SUBSTEP: out = w + c M^-1 r;   STAGE: out = a w + b x + c M^-1 r,
//   rn[T, comp] = sum_m (x - w - tau M^-1 r)^2
__global__ void curved_fixup_kernel(int mode, const int32_t* __restrict__ el, int n, int nbs,
                                    const double* __restrict__ minv, const double* __restrict__ cres,
                                    const double* __restrict__ w, double* __restrict__ out, StageParams sp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * n) return;
  if (mode == MODE_STAGE && stage_stopped(sp)) return;   // converged Richardson iteration
  const int slot = i >> 1, comp = i & 1, nb = 2 * nbs;
  const size_t T = (size_t)el[slot];
  const double* Mi = minv + (size_t)slot * nbs * nbs;
  const double* r = cres + (size_t)slot * nb + comp * nbs;
  double acc = 0.0, chk = 0.0;
  for (int m = 0; m < nbs; ++m) {
    double s = 0.0;
    for (int l = 0; l < nbs; ++l) s = fma(Mi[m * nbs + l], r[l], s);
    const size_t g = T * nb + comp * nbs + m;
    double v;
    if (mode == MODE_SUBSTEP) {
      v = fma(sp.c, s, w[g]);
    } else {
      const double xv = sp.x[g];
      v = fma(sp.b, xv, fma(sp.c, s, sp.a * w[g]));
      const double res = fma(-sp.tau, s, xv - w[g]);
      acc = fma(res, res, acc);
    }
    out[g] = v;
    chk += v;
  }
  guard_finite(sp.flag, chk);
  if (mode == MODE_STAGE && sp.rn) sp.rn[2 * T + comp] = acc;
}

// transfer rows of curved elements: I (dir 0) out = I_T in, I^T (dir 1) out = I_T^T in
__global__ void curved_transfer_kernel(int dir, const int32_t* __restrict__ el, int n, int nb,
                                       const double* __restrict__ itrans, const double* __restrict__ in,
                                       double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * nb) return;
  const int slot = i / nb, row = i - slot * nb;
  const size_t T = (size_t)el[slot];
  const double* It = itrans + (size_t)slot * nb * nb;
  const double* x = in + T * nb;
  double a = 0.0;
  if (dir == 0)
    for (int j = 0; j < nb; ++j) a = fma(It[row * nb + j], x[j], a);
  else
    for (int j = 0; j < nb; ++j) a = fma(It[j * nb + row], x[j], a);
  out[T * nb + row] = a;
}

// max |J u_hat / detJ| over the curved elements' volume points (per-point J),
// from the modal rows (u_hat | div) of launch_maxspeed (modal_rows_kernel)
__global__ void curved_maxspeed_kernel(const int32_t* __restrict__ el, int n, int nbs, int mr, int nqv,
                                       const double* __restrict__ vD, const double* __restrict__ modal,
                                       const double* __restrict__ cpiola, unsigned long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double best = 0.0;
  if (i < n * nqv) {
    const int slot = i / nqv, q = i - slot * nqv;
    const double* mrow = modal + (size_t)el[slot] * mr;
    double a = 0.0, b = 0.0;
    for (int m = 0; m < nbs; ++m) {
      a = fma(mrow[m], vD[q * nbs + m], a);
      b = fma(mrow[nbs + m], vD[q * nbs + m], b);
    }
    const double* P = cpiola + ((size_t)slot * nqv + q) * 4;
    const double x = fma(P[0], a, P[1] * b), y = fma(P[2], a, P[3] * b);
    best = sqrt(fma(x, x, y * y));
  }
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

static int curved_fixup(hdgc_ctx* c, int mode, const double* w, double* out, const StageParams& sp, cudaStream_t st) {
  const int th = 128;
  curved_fixup_kernel<<<(2 * c->n_curved + th - 1) / th, th, 0, st>>>(mode, c->d_celems, c->n_curved, c->nbs,
                                                                    c->d_cminv, c->d_cres, w, out, sp);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

static int elem(hdgc_ctx* c, int mode, const double* u, const double* w, const double* inflow, double* out,
                const StageParams& sp, cudaStream_t st) {
  HDGC_K_SWITCH(c->k, launch_elem<KK>(c, mode, u, w, inflow, out, sp, st));
}
// k <= 2: frozen-velocity rows for a batch of update kernels on the same u
static int elem_prep(hdgc_ctx* c, const double* u, cudaStream_t st) {
  HDGC_K_SWITCH(c->k, launch_elem_prep<KK>(c, u, st));
}

static int transfer3(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st);

static int transfer_affine(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st) {
  HDGC_K_SWITCH(c->k, launch_transfer<KK>(c, dir, in, out, st));
}

static int transfer(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st) {
  if (c->dim == 3) return transfer3(c, dir, in, out, st);
  int rc = transfer_affine(c, dir, in, out, st);
  if (rc || c->n_curved == 0) return rc;
  // curved rows: the L2 projection I_T replaces the affine embedding
  const int th = 128, work = c->n_curved * c->nb;
  curved_transfer_kernel<<<(work + th - 1) / th, th, 0, st>>>(dir, c->d_celems, c->n_curved, c->nb, c->d_citrans,
                                                             in, out);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

static int prep(hdgc_ctx* c, const double* u, cudaStream_t st) {
  HDGC_K_SWITCH(c->k, sf_prep<KK>(c, u, st));
}

static int sfmain(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out, const StageParams& sp,
                  cudaStream_t st) {
  HDGC_K_SWITCH(c->k, sf_main<KK>(c, mode, w, inflow, out, sp, st));
}

static int setup_variant(hdgc_ctx* c, const hdgc_tables_desc* t, const std::vector<double>& packed) {
  HDGC_K_SWITCH(c->k, sf_setup<KK>(c, t, packed));
}

// one operator application, dispatched on the variant chosen at create
static int main3(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out, const StageParams& sp,
                 cudaStream_t st);
static int prep3(hdgc_ctx* c, const double* u, cudaStream_t st);

static int apply_any_(hdgc_ctx* c, int mode, const double* u, const double* w, const double* inflow, double* out,
                      const StageParams& sp, bool prep_done, cudaStream_t st);
static int apply_any(hdgc_ctx* c, int mode, const double* u, const double* w, const double* inflow, double* out,
                     const StageParams& sp0, bool prep_done, cudaStream_t st) {
  if (mode != MODE_SUBSTEP && mode != MODE_STAGE) return apply_any_(c, mode, u, w, inflow, out, sp0, prep_done, st);
  StageParams sp = sp0;
  sp.flag = c->d_flag;   // norm-blowup guard of the update epilogues
  if (c->n_curved == 0) return apply_any_(c, mode, u, w, inflow, out, sp, prep_done, st);
  sp.cres = c->d_cres;
  int rc = apply_any_(c, mode, u, w, inflow, out, sp, prep_done, st);
  return rc ? rc : curved_fixup(c, mode, w, out, sp, st);
}
// The update kernel right after a frozen-velocity prep launches with PDL: it
// stages w and its tables while the prep drains and reads the prep only after
// griddepcontrol.wait (SFParams / Conv3Params::prep_dep).  The modal variant
// (conv2d_sfm.cuh) and curved batches (fix-up kernel) launch normally.
static bool prep_pdl_ok(const hdgc_ctx* c) { return !c->modal && c->n_curved == 0; }
static int after_prep(hdgc_ctx* c, int (*launch)(hdgc_ctx*, int, const double*, const double*, double*,
                                                 const StageParams&, cudaStream_t),
                      int mode, const double* w, const double* inflow, double* out, const StageParams& sp,
                      cudaStream_t st) {
  const bool pdl = prep_pdl_ok(c);
  c->pdl = pdl;
  c->prep_dep = pdl;
  const int rc = launch(c, mode, w, inflow, out, sp, st);
  c->pdl = false;
  c->prep_dep = false;
  return rc;
}
static int apply_any_(hdgc_ctx* c, int mode, const double* u, const double* w, const double* inflow, double* out,
                      const StageParams& sp, bool prep_done, cudaStream_t st) {
  if (c->variant == 2) {
    if (prep_done) return main3(c, mode, w, inflow, out, sp, st);
    int rc = prep3(c, u, st);
    if (rc) return rc;
    return after_prep(c, main3, mode, w, inflow, out, sp, st);
  }
  if (c->variant == 1) {
    if (prep_done) return sfmain(c, mode, w, inflow, out, sp, st);
    int rc = prep(c, u, st);
    if (rc) return rc;
    return after_prep(c, sfmain, mode, w, inflow, out, sp, st);
  }
  // thread variant (k <= 2): the update kernels read the frozen-velocity rows when
  // the caller prepared them for this u (prep_any), else they evaluate u themselves
  c->tprep_on = prep_done && c->tprep_valid && (mode == MODE_SUBSTEP || mode == MODE_STAGE);
  const int rc = elem(c, mode, u, w, inflow, out, sp, st);
  c->tprep_on = false;
  return rc;
}
static int apply_any(hdgc_ctx* c, int mode, const double* u, const double* w, const double* inflow, double* out,
                     double dt, bool prep_done, cudaStream_t st) {
  StageParams sp;
  sp.c = -dt;
  return apply_any(c, mode, u, w, inflow, out, sp, prep_done, st);
}
// uses: how many update kernels will run on this frozen u (the thread variant's
// prep costs about 0.6 of an update kernel and saves about a third of each)
static int prep_any(hdgc_ctx* c, const double* u, cudaStream_t st, int uses = 1 << 20) {
  if (c->variant == 2) return prep3(c, u, st);
  if (c->variant == 1) return prep(c, u, st);
  static const bool tprep = [] { const char* e = getenv("HDGC_TPREP"); return !(e && e[0] == '0'); }();
  c->tprep_valid = false;
  if (!tprep || uses < 3 || c->dim != 2) return HDGC_OK;
  const int rc = elem_prep(c, u, st);
  c->tprep_valid = rc == HDGC_OK;
  return rc;
}

// ---------------------------------------------------------------------------
// C ABI

namespace hdgc {
HDGC_DECLARE_ORDER3(1)
HDGC_DECLARE_ORDER3(2)
HDGC_DECLARE_ORDER3(3)
HDGC_DECLARE_ORDER3(4)
}  // namespace hdgc

#define HDGC_K3_SWITCH(k, CALL)                       \
  switch (k) {                                        \
    case 1: { constexpr int KK = 1; return CALL; }    \
    case 2: { constexpr int KK = 2; return CALL; }    \
    case 3: { constexpr int KK = 3; return CALL; }    \
    case 4: { constexpr int KK = 4; return CALL; }    \
    default: return hdgc_set_err(HDGC_EUNSUP, "3D order k=%d not supported (1..4)", k); \
  }

static int prep3(hdgc_ctx* c, const double* u, cudaStream_t st) { HDGC_K3_SWITCH(c->k, launch3_prep<KK>(c, u, st)); }
static int main3(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out, const StageParams& sp,
                 cudaStream_t st) {
  HDGC_K3_SWITCH(c->k, launch3_main<KK>(c, mode, w, inflow, out, sp, st));
}
static int transfer3(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st) {
  HDGC_K3_SWITCH(c->k, launch3_transfer<KK>(c, dir, in, out, st));
}
static int setup3(hdgc_ctx* c, const hdgc_tables_desc* t) { HDGC_K3_SWITCH(c->k, launch3_setup<KK>(c, t)); }
static int maxspeed3(hdgc_ctx* c, const double* u, double* out, cudaStream_t st) {
  HDGC_K3_SWITCH(c->k, launch3_maxspeed<KK>(c, u, out, st));
}

extern "C" int hdgc_destroy(hdgc_ctx* c);

// setup validation flags (bad) -> error text
static int mesh_error(int bad) {
  switch (bad) {
    case 1: return hdgc_set_err(HDGC_EINVAL, "inverted or degenerate element (detJ <= 0 in 2D, detJ = 0 in 3D)");
    case 2: return hdgc_set_err(HDGC_EINVAL, "invalid facet_elems/facet_local entry (element id or local facet out of range)");
    case 3: return hdgc_set_err(HDGC_EINVAL, "an (element, local facet) pair appears in more than one facet");
    case 4: return hdgc_set_err(HDGC_EINVAL, "an (element, local facet) pair is missing from the facet arrays");
    case 5: return hdgc_set_err(HDGC_EINVAL, "element vertex id out of range [0, n_vertices)");
    case 6: return hdgc_set_err(HDGC_EINVAL, "3D: every tet's vertex ids must be sorted ascending (shared faces are then "
                                             "parametrised alike on both sides; facet_perm is not supported)");
    default: return hdgc_set_err(HDGC_EINVAL, "invalid mesh (code %d)", bad);
  }
}

// flag buffers of the norm-blowup guard
static int alloc_flag(hdgc_ctx* c) {
  int rc = hdgc_dev_alloc(c, (void**)&c->d_flag, sizeof(int));
  if (rc) return rc;
  if (cudaMemset(c->d_flag, 0, sizeof(int)) != cudaSuccess || cudaMallocHost((void**)&c->h_flag, sizeof(int)) != cudaSuccess)
    return hdgc_set_err(HDGC_ECUDA, "blow-up flag allocation failed");
  *c->h_flag = 0;
  return HDGC_OK;
}

// 3D context: tet mesh (vertices sorted per tet), Dims3<K> tables
static int create3d(const hdgc_mesh_desc* mesh, const hdgc_tables_desc* tab, hdgc_ctx** out) {
  const int k = tab->k;
  if (k < 1 || k > 4) return hdgc_set_err(HDGC_EUNSUP, "3D order k=%d not supported (1..4)", k);
  if (tab->nqv != dims3_nq(k) || tab->nf != dims3_nf(k))
    return hdgc_set_err(HDGC_EINVAL, "3D table sizes nqv=%d nf=%d do not match the k=%d rules (%d, %d)",
                        tab->nqv, tab->nf, k, dims3_nq(k), dims3_nf(k));
  if (mesh->n_elements <= 0 || mesh->n_vertices <= 0 || mesh->n_facets <= 0)
    return hdgc_set_err(HDGC_EINVAL, "empty mesh");
  if ((int64_t)mesh->n_elements * 4 > INT32_MAX) return hdgc_set_err(HDGC_EINVAL, "too many elements");
  if (!mesh->vertices || !mesh->elements || !mesh->facet_elems || !mesh->facet_local || !tab->coef ||
      !tab->div_modal || !tab->vol_w || !tab->vol_D || !tab->vol_G || !tab->fac_w || !tab->fac_L ||
      !tab->fac_D || !tab->fac_len)
    return hdgc_set_err(HDGC_EINVAL, "null array in descriptor");
  if (mesh->facet_perm)
    return hdgc_set_err(HDGC_EINVAL, "facet_perm must be NULL: pass tets with ascending vertex ids instead");
  hdgc_ctx* c = new hdgc_ctx();
  c->dim = 3;
  c->k = k;
  c->nbs = dims3_nbs(k);
  c->nb = 3 * c->nbs;
  c->nqv = tab->nqv;
  c->nf = tab->nf;
  c->nt = mesh->n_elements;
  c->nv = mesh->n_vertices;
  c->nf_facets = mesh->n_facets;
  c->variant = 2;
  const int nb = c->nb, nbs = c->nbs, nqv = c->nqv, nf = c->nf;
  const int nbs1 = k * (k + 1) * (k + 2) / 6, nfd = (k + 1) * (k + 2) / 2;
  std::vector<double> h(dims3_tab(k), 0.0);
  size_t o = 0;
  auto put = [&](const double* src, size_t n) { memcpy(&h[o], src, sizeof(double) * n); o += n; };
  put(tab->coef, (size_t)nb * nb);
  put(tab->div_modal, (size_t)nbs1 * nb);
  put(tab->vol_w, nqv);
  put(tab->vol_D, (size_t)nqv * nbs);
  put(tab->vol_G, (size_t)nqv * nbs * 3);
  put(tab->fac_w, nf);
  put(tab->fac_L, (size_t)nf * nfd);
  put(tab->fac_D, (size_t)4 * nf * nbs);
  put(tab->fac_len, 4);
  const size_t NT = c->nt, NF = c->nf_facets;
  double* d_V = nullptr;
  int64_t *d_tet = nullptr, *d_fe = nullptr, *d_fl = nullptr;
  int* d_slot = nullptr;
  auto fail = [&](int code) {
    cudaFree(d_V); cudaFree(d_tet); cudaFree(d_fe); cudaFree(d_fl); cudaFree(d_slot);
    hdgc_destroy(c);
    return code;
  };
  int rc;
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_tab, h.size() * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_code, NT * 4 * sizeof(int32_t)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_piola, NT * 9 * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_minv, NT * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_sign, NT * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_scratch, NT * nb * sizeof(double)))) return fail(rc);
  {
    // per element: alpha/beta/gamma/delta at the volume points, s at the face points,
    // the inflow-face mask and the face inflow matrices S_f (Dims3::PREP)
    const size_t nfd = (size_t)(k + 1) * (k + 2) / 2;
    const size_t prep = 4 * (size_t)nqv + 4 * (size_t)nf + 1 + 4 * (nfd * (nfd + 1) / 2);
    // (the volume region is tile-blocked by 32 elements: stride prep3_stride(NT))
    const size_t ps = (size_t)prep3_stride((int)NT);
    if ((rc = hdgc_dev_alloc(c, (void**)&c->d_prep, ps * prep * sizeof(double)))) return fail(rc);
    if (cudaMemset(c->d_prep, 0, ps * prep * sizeof(double)) != cudaSuccess) return fail(hdgc_set_err(HDGC_ECUDA, "prep memset"));
  }
#define SETUP3_TRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) \
    return fail(hdgc_set_err(HDGC_ECUDA, "%s: %s", #x, cudaGetErrorString(e_))); } while (0)
  SETUP3_TRY(cudaMemcpy(c->d_tab, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  SETUP3_TRY(cudaMalloc(&d_V, sizeof(double) * 3 * c->nv));
  SETUP3_TRY(cudaMalloc(&d_tet, sizeof(int64_t) * 4 * NT));
  SETUP3_TRY(cudaMalloc(&d_fe, sizeof(int64_t) * 2 * NF));
  SETUP3_TRY(cudaMalloc(&d_fl, sizeof(int64_t) * 2 * NF));
  SETUP3_TRY(cudaMalloc(&d_slot, sizeof(int) * (NF + 2)));
  SETUP3_TRY(cudaMemcpy(d_V, mesh->vertices, sizeof(double) * 3 * c->nv, cudaMemcpyHostToDevice));
  SETUP3_TRY(cudaMemcpy(d_tet, mesh->elements, sizeof(int64_t) * 4 * NT, cudaMemcpyHostToDevice));
  SETUP3_TRY(cudaMemcpy(d_fe, mesh->facet_elems, sizeof(int64_t) * 2 * NF, cudaMemcpyHostToDevice));
  SETUP3_TRY(cudaMemcpy(d_fl, mesh->facet_local, sizeof(int64_t) * 2 * NF, cudaMemcpyHostToDevice));
  int* d_misc = d_slot + NF;
  SETUP3_TRY(cudaMemset(d_misc, 0, 2 * sizeof(int)));
  SETUP3_TRY(cudaMemset(c->d_code, 0x80, NT * 4 * sizeof(int32_t)));   // CODE_UNSET
  {
    const int th = 256;
    geometry3d_kernel<<<(int)((NT + th - 1) / th), th>>>(d_V, d_tet, (int)NT, c->nv, c->d_piola, c->d_minv,
                                                         c->d_sign, d_misc + 1);
    bflag_kernel<<<(int)((NF + th - 1) / th), th>>>(d_fe, (int)NF, d_slot);
    scan_kernel<<<1, 1024>>>(d_slot, (int)NF, d_misc);
    codes_kernel<<<(int)((NF + th - 1) / th), th>>>(d_fe, d_fl, d_slot, (int)NF, (int)NT, 4, c->d_code, d_misc + 1);
    check_codes_kernel<<<(int)((4 * NT + th - 1) / th), th>>>(c->d_code, 4 * NT, d_misc + 1);
    SETUP3_TRY(cudaGetLastError());
  }
  int misc[2];
  SETUP3_TRY(cudaMemcpy(misc, d_misc, sizeof(misc), cudaMemcpyDeviceToHost));
  if (misc[1]) return fail(mesh_error(misc[1]));
  c->nbf = misc[0];
  if ((rc = alloc_flag(c))) return fail(rc);
  if ((rc = setup3(c, tab))) return fail(rc);
  cudaFree(d_V); cudaFree(d_tet); cudaFree(d_fe); cudaFree(d_fl); cudaFree(d_slot);
  *out = c;
  return HDGC_OK;
#undef SETUP3_TRY
}

// Device vectors are moved with 16-byte vector loads and TMA bulk copies
// (cp.async.bulk needs 16-byte aligned global addresses): reject anything
// else up front instead of faulting (a misaligned-address fault is sticky and
// destroys the process's CUDA context).
static bool misaligned(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (p && (reinterpret_cast<uintptr_t>(p) & 15u)) return true;
  return false;
}
#define HDGC_ALIGNED(...)                                                                              \
  do {                                                                                                \
    if (misaligned({__VA_ARGS__}))                                                                    \
      return hdgc_set_err(HDGC_EINVAL, "device pointers must be 16-byte aligned (%s)", #__VA_ARGS__); \
  } while (0)

extern "C" {

const char* hdgc_last_error(void) { return g_err.c_str(); }

int hdgc_check_finite(hdgc_ctx* c, void* stream) {
  if (!c) return hdgc_set_err(HDGC_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (*c->h_flag == 0) return HDGC_OK;
  *c->h_flag = 0;
  CUDA_TRY(cudaMemsetAsync(c->d_flag, 0, sizeof(int), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return hdgc_set_err(HDGC_EBLOWUP, "norm blow-up: an explicit update produced non-finite values "
                                    "(substep too large for the CFL limit?)");
}
const char* hdgc_version(void) { return "hdgconv 0.2 sm_100a fp64"; }

int hdgc_create(const hdgc_mesh_desc* mesh, const hdgc_tables_desc* tab, hdgc_ctx** out) {
  if (!mesh || !tab || !out) return hdgc_set_err(HDGC_EINVAL, "null argument");
  *out = nullptr;
  if (mesh->dim == 3) return create3d(mesh, tab, out);
  if (mesh->dim != 2) return hdgc_set_err(HDGC_EUNSUP, "dim=%d not supported (2 or 3)", mesh->dim);
  const int k = tab->k;
  if (k < 1 || k > 8) return hdgc_set_err(HDGC_EUNSUP, "order k=%d not supported (1..8)", k);
  if (tab->nqv != dims_nqv(k) || tab->nf != dims_nf(k))
    return hdgc_set_err(HDGC_EINVAL, "table sizes nqv=%d nf=%d do not match the k=%d rules (%d, %d)",
                   tab->nqv, tab->nf, k, dims_nqv(k), dims_nf(k));
  if (mesh->n_elements <= 0 || mesh->n_vertices <= 0 || mesh->n_facets <= 0)
    return hdgc_set_err(HDGC_EINVAL, "empty mesh");
  if ((int64_t)mesh->n_elements * 4 > INT32_MAX) return hdgc_set_err(HDGC_EINVAL, "too many elements");
  if (!mesh->vertices || !mesh->elements || !mesh->facet_elems || !mesh->facet_local || !tab->coef || !tab->div_modal ||
      !tab->vol_w || !tab->vol_D || !tab->vol_G || !tab->fac_w || !tab->fac_L || !tab->fac_D || !tab->fac_len)
    return hdgc_set_err(HDGC_EINVAL, "null array in descriptor");

  hdgc_ctx* c = new hdgc_ctx();
  c->dim = 2;
  c->k = k;
  c->nbs = dims_nbs(k);
  c->nb = 2 * c->nbs;
  c->nqv = tab->nqv;
  c->nf = tab->nf;
  c->nt = mesh->n_elements;
  c->nv = mesh->n_vertices;
  c->nf_facets = mesh->n_facets;
  c->variant = 0;

  // pack tables (host), Dims<K> layout
  const int nb = c->nb, nbs = c->nbs, nqv = c->nqv, nf = c->nf, ne = k + 1;
  std::vector<double> h(dims_tab(k), 0.0);
  size_t o = 0;
  memcpy(&h[o], tab->coef, sizeof(double) * nb * nb); o += (size_t)nb * nb;
  memcpy(&h[o], tab->div_modal, sizeof(double) * (k * (k + 1) / 2) * nb); o += (size_t)(k * (k + 1) / 2) * nb;
  memcpy(&h[o], tab->vol_w, sizeof(double) * nqv); o += nqv;
  memcpy(&h[o], tab->vol_D, sizeof(double) * nqv * nbs); o += (size_t)nqv * nbs;
  memcpy(&h[o], tab->vol_G, sizeof(double) * nqv * nbs * 2); o += (size_t)nqv * nbs * 2;
  memcpy(&h[o], tab->fac_w, sizeof(double) * nf); o += nf;
  memcpy(&h[o], tab->fac_L, sizeof(double) * nf * ne); o += (size_t)nf * ne;
  memcpy(&h[o], tab->fac_D, sizeof(double) * 3 * nf * nbs); o += (size_t)3 * nf * nbs;
  memcpy(&h[o], tab->fac_len, sizeof(double) * 3);

  int rc = HDGC_OK;
  double* d_V = nullptr;
  int64_t *d_tri = nullptr, *d_fe = nullptr, *d_fl = nullptr;
  int *d_slot = nullptr, *d_flag = nullptr;
  const size_t NT = c->nt, NF = c->nf_facets;
  auto fail = [&](int code) {
    cudaFree(d_V); cudaFree(d_tri); cudaFree(d_fe); cudaFree(d_fl); cudaFree(d_slot); cudaFree(d_flag);
    hdgc_destroy(c);
    return code;
  };
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_tab, h.size() * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_code, NT * 3 * sizeof(int32_t)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_piola, NT * 4 * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_minv, NT * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_scratch, NT * nb * sizeof(double)))) return fail(rc);
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_modal, NT * (nb + k * (k + 1) / 2) * sizeof(double)))) return fail(rc);
#define SETUP_TRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) \
    return fail(hdgc_set_err(HDGC_ECUDA, "%s: %s", #x, cudaGetErrorString(e_))); } while (0)
  SETUP_TRY(cudaMemcpy(c->d_tab, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  SETUP_TRY(cudaMalloc(&d_V, sizeof(double) * 2 * c->nv));
  SETUP_TRY(cudaMalloc(&d_tri, sizeof(int64_t) * 3 * NT));
  SETUP_TRY(cudaMalloc(&d_fe, sizeof(int64_t) * 2 * NF));
  SETUP_TRY(cudaMalloc(&d_fl, sizeof(int64_t) * 2 * NF));
  SETUP_TRY(cudaMalloc(&d_slot, sizeof(int) * (NF + 2)));
  SETUP_TRY(cudaMemcpy(d_V, mesh->vertices, sizeof(double) * 2 * c->nv, cudaMemcpyHostToDevice));
  SETUP_TRY(cudaMemcpy(d_tri, mesh->elements, sizeof(int64_t) * 3 * NT, cudaMemcpyHostToDevice));
  SETUP_TRY(cudaMemcpy(d_fe, mesh->facet_elems, sizeof(int64_t) * 2 * NF, cudaMemcpyHostToDevice));
  SETUP_TRY(cudaMemcpy(d_fl, mesh->facet_local, sizeof(int64_t) * 2 * NF, cudaMemcpyHostToDevice));
  int* d_misc = d_slot + NF;  // [0] = total boundary facets, [1] = bad flag
  SETUP_TRY(cudaMemset(d_misc, 0, 2 * sizeof(int)));
  SETUP_TRY(cudaMemset(c->d_code, 0x80, NT * 3 * sizeof(int32_t)));  // CODE_UNSET
  {
    const int th = 256;
    geometry2d_kernel<<<(int)((NT + th - 1) / th), th>>>(d_V, d_tri, (int)NT, c->nv, c->d_piola, c->d_minv,
                                                         d_misc + 1);
    bflag_kernel<<<(int)((NF + th - 1) / th), th>>>(d_fe, (int)NF, d_slot);
    scan_kernel<<<1, 1024>>>(d_slot, (int)NF, d_misc);
    codes_kernel<<<(int)((NF + th - 1) / th), th>>>(d_fe, d_fl, d_slot, (int)NF, (int)NT, 3, c->d_code, d_misc + 1);
    check_codes_kernel<<<(int)((3 * NT + th - 1) / th), th>>>(c->d_code, 3 * NT, d_misc + 1);
    SETUP_TRY(cudaGetLastError());
  }
  int misc[2];
  SETUP_TRY(cudaMemcpy(misc, d_misc, sizeof(misc), cudaMemcpyDeviceToHost));
  if (misc[1]) return fail(mesh_error(misc[1]));
  c->nbf = misc[0];
  if ((rc = alloc_flag(c))) return fail(rc);
  if ((rc = setup_variant(c, tab, h))) return fail(rc);
  cudaFree(d_V); cudaFree(d_tri); cudaFree(d_fe); cudaFree(d_fl); cudaFree(d_slot);
  *out = c;
  return HDGC_OK;
#undef SETUP_TRY
}

// Built-in reference tables (tables_blob.py, assembled into .rodata by build.py)
extern "C" const unsigned char hdgc_tables_blob[];
extern "C" const unsigned char hdgc_tables_blob_end[];

int hdgc_create_k(const hdgc_mesh_desc* mesh, int32_t k, hdgc_ctx** out) {
  if (!mesh || !out) return hdgc_set_err(HDGC_EINVAL, "null argument");
  *out = nullptr;
  constexpr int64_t kMagic = 0x314C425443474448LL;   // "HDGCTBL1"
  constexpr int kFields = 20;                         // tables_blob.FIELDS
  const int64_t* hdr = reinterpret_cast<const int64_t*>(hdgc_tables_blob);
  const size_t blob_bytes = (size_t)(hdgc_tables_blob_end - hdgc_tables_blob);
  if (blob_bytes < 16 || hdr[0] != kMagic) return hdgc_set_err(HDGC_EINVAL, "built-in table blob is missing or corrupt");
  const int64_t n = hdr[1];
  const int64_t per = 5 + 2 * kFields;
  const double* data = reinterpret_cast<const double*>(hdr + 2 + n * per);
  for (int64_t e = 0; e < n; ++e) {
    const int64_t* en = hdr + 2 + e * per;
    if (en[0] != mesh->dim || en[1] != k) continue;
    hdgc_tables_desc t;
    memset(&t, 0, sizeof(t));
    t.k = k;
    t.nqv = (int32_t)en[2];
    t.nf = (int32_t)en[3];
    t.col_n = (int32_t)en[4];
    const double* f[kFields];
    for (int i = 0; i < kFields; ++i) f[i] = en[6 + 2 * i] ? data + en[5 + 2 * i] : nullptr;
    t.coef = f[0]; t.div_modal = f[1]; t.vol_w = f[2]; t.vol_D = f[3]; t.vol_G = f[4];
    t.fac_w = f[5]; t.fac_L = f[6]; t.fac_D = f[7]; t.fac_len = f[8];
    t.col_A = f[9]; t.col_Ad = f[10]; t.col_B = f[11]; t.col_Bd = f[12]; t.col_xi = f[13];
    t.col_wa = f[14]; t.col_wy = f[15]; t.col_inv1my = f[16]; t.col_C = f[17]; t.col_Cd = f[18];
    t.col_pf = f[19];
    return hdgc_create(mesh, &t, out);
  }
  return hdgc_set_err(HDGC_EUNSUP, "no built-in tables for dim=%d k=%d (2D: k = 1..8, 3D: k = 1..4)", mesh->dim, k);
}

int hdgc_destroy(hdgc_ctx* c) {
  if (!c) return HDGC_OK;
  cudaFree(c->d_tab); cudaFree(c->d_code); cudaFree(c->d_piola); cudaFree(c->d_minv);
  cudaFree(c->d_sign); cudaFree(c->d_scratch); cudaFree(c->d_scratch2); cudaFree(c->d_modal); cudaFree(c->d_prep); cudaFree(c->d_ftab); cudaFree(c->d_afrag); cudaFree(c->d_mprep); cudaFree(c->d_hu); cudaFree(c->d_hw); cudaFree(c->d_hr); cudaFree(c->d_hin);
  cudaFree(c->d_uext); cudaFree(c->d_rn); cudaFree(c->d_rpart); cudaFree(c->d_fpart); cudaFree(c->d_ctl); cudaFree(c->d_norms);
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  for (int i = 0; i < 2; ++i) if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  for (auto& g : c->graphs) if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  cudaFree(c->d_dof); cudaFree(c->d_dfac); cudaFree(c->d_inv); cudaFree(c->d_invf); cudaFree(c->d_gl); cudaFree(c->d_rw);
  cudaFree(c->d_celems); cudaFree(c->d_cminv); cudaFree(c->d_citrans); cudaFree(c->d_cpiola); cudaFree(c->d_cres);
  cudaFree(c->d_flag);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  delete c;
  return HDGC_OK;
}

int hdgc_get_info(const hdgc_ctx* c, hdgc_info* info) {
  if (!c || !info) return hdgc_set_err(HDGC_EINVAL, "null argument");
  info->dim = c->dim; info->k = c->k; info->nb = c->nb; info->nbs = c->nbs;
  info->nqv = c->nqv; info->nf = c->nf;
  info->n_elements = c->nt; info->n_facets = c->nf_facets; info->n_boundary_facets = c->nbf;
  info->volume_variant = c->variant;
  info->device_bytes = c->bytes;
  return HDGC_OK;
}

int hdgc_apply_v(hdgc_ctx* c, const double* u, const double* w, const double* inflow, double* r, void* stream) {
  if (!c || !u || !w || !r) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (r == u || r == w || r == inflow) return hdgc_set_err(HDGC_EINVAL, "output aliases an input");
  HDGC_ALIGNED(u, w, inflow, r);
  return apply_any(c, MODE_APPLY, u, w, inflow, r, 0.0, false, (cudaStream_t)stream);
}

int hdgc_apply_w(hdgc_ctx* c, const double* u, const double* inflow, double* r_w, void* stream) {
  if (!c || !u || !r_w) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (r_w == u || r_w == inflow) return hdgc_set_err(HDGC_EINVAL, "output aliases an input");
  HDGC_ALIGNED(u, inflow, r_w);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = transfer(c, 0, u, c->d_scratch, st);
  if (rc) return rc;
  if (c->variant == 0 && c->n_curved == 0)
    return elem(c, MODE_APPLY_IT, u, c->d_scratch, inflow, r_w, StageParams(), st);
  // sum-factorised: r_V into scratch2, then I^T
  if (!c->d_scratch2 &&
      (rc = hdgc_dev_alloc(c, (void**)&c->d_scratch2, sizeof(double) * (size_t)c->nt * c->nb)))
    return rc;
  if ((rc = apply_any(c, MODE_APPLY, u, c->d_scratch, inflow, c->d_scratch2, 0.0, false, st))) return rc;
  return transfer(c, 1, c->d_scratch2, r_w, st);
}

// the substep batch as a launch sequence on stream st (prep + nsteps update kernels)
static int substeps_enqueue(hdgc_ctx* c, const double* u, double* w, const double* inflow, double dt, int nsteps,
                            cudaStream_t st) {
  double* a = w;
  double* b = c->d_scratch;
  if (nsteps > 0) {
    // u is frozen over the substep batch: one prep per batch
    int rc = prep_any(c, u, st, nsteps);
    if (rc) return rc;
  }
  for (int s = 0; s < nsteps; ++s) {
    // substeps after the first overlap their prologue with the previous
    // substep's drain (PDL, common.cuh), the first one with the prep's drain;
    // curved batches interpose the fix-up kernel
    c->pdl = c->n_curved == 0 && (s > 0 || (c->variant >= 1 && prep_pdl_ok(c)));
    c->prep_dep = s == 0 && c->pdl;
    int rc = apply_any(c, MODE_SUBSTEP, u, a, inflow, b, dt, true, st);
    c->pdl = false;
    c->prep_dep = false;
    if (rc) return rc;
    double* t = a; a = b; b = t;
  }
  if (a != w) CUDA_TRY(cudaMemcpyAsync(w, a, sizeof(double) * (size_t)c->nt * c->nb, cudaMemcpyDeviceToDevice, st));
  return HDGC_OK;
}

// Substep batches run as CUDA graphs: the launch sequence is captured once
// per (u, w, inflow, dt, nsteps) on a context-owned stream (the PDL launches
// become programmatic edges) and replayed with one cudaGraphLaunch on the
// caller's stream, so the host pays one launch per batch instead of nsteps+1.
// Small LRU cache; HDGC_GRAPHS=0 enqueues the kernels one by one instead.
static bool graphs_enabled() {
  // default off: measured with the captured programmatic edges (port 1 or 2) the
  // batch runs without the PDL overlap (cfg2 k=4: 67 vs 59.5 us per substep; k=1:
  // 11-12 vs 7.6 us), so stream launches win; HDGC_GRAPHS=1 opts in
  static const bool on = [] { const char* e = getenv("HDGC_GRAPHS"); return e && e[0] == '1'; }();
  return on;
}

static int substeps_graph(hdgc_ctx* c, const double* u, double* w, const double* inflow, double dt, int nsteps,
                          cudaStream_t st) {
  uint64_t dtb;
  memcpy(&dtb, &dt, sizeof(dtb));
  hdgc_graph* hit = nullptr;
  for (auto& g : c->graphs)
    if (g.exec && g.u == u && g.w == w && g.inflow == inflow && g.dt_bits == dtb && g.nsteps == nsteps) hit = &g;
  if (!hit) {
    if (!c->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    const int rc = substeps_enqueue(c, u, w, inflow, dt, nsteps, c->cap_stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->cap_stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ec != cudaSuccess) return hdgc_set_err(HDGC_ECUDA, "substep graph capture: %s", cudaGetErrorString(ec));
    if (const char* pe = getenv("HDGC_GRAPH_PORT")) {
      // development: rewrite the programmatic edges' port (1 = programmatic trigger, 2 = launch completion)
      size_t ne = 0;
      cudaGraphGetEdges_v2(graph, nullptr, nullptr, nullptr, &ne);
      std::vector<cudaGraphNode_t> from(ne), to(ne);
      std::vector<cudaGraphEdgeData> ed(ne);
      cudaGraphGetEdges_v2(graph, from.data(), to.data(), ed.data(), &ne);
      for (size_t i = 0; i < ne; ++i) {
        if (ed[i].type != cudaGraphDependencyTypeProgrammatic) continue;
        cudaGraphRemoveDependencies_v2(graph, &from[i], &to[i], &ed[i], 1);
        cudaGraphEdgeData e2 = ed[i];
        e2.from_port = (unsigned char)atoi(pe);
        cudaGraphAddDependencies_v2(graph, &from[i], &to[i], &e2, 1);
      }
    }
    if (getenv("HDGC_GRAPH_DEBUG")) {
      size_t ne = 0;
      cudaGraphGetEdges_v2(graph, nullptr, nullptr, nullptr, &ne);
      std::vector<cudaGraphNode_t> from(ne), to(ne);
      std::vector<cudaGraphEdgeData> ed(ne);
      cudaGraphGetEdges_v2(graph, from.data(), to.data(), ed.data(), &ne);
      int prog = 0;
      for (auto& e : ed) prog += e.type == cudaGraphDependencyTypeProgrammatic;
      fprintf(stderr, "[hdgc] substep graph: %zu edges, %d programmatic (from_port %d)\n", ne, prog,
              ne ? (int)ed[ne - 1].from_port : -1);
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return hdgc_set_err(HDGC_ECUDA, "substep graph instantiate: %s", cudaGetErrorString(ei));
    hit = &c->graphs[c->graph_next];
    c->graph_next = (c->graph_next + 1) % HDGC_GRAPH_CACHE;
    if (hit->exec) cudaGraphExecDestroy(hit->exec);
    *hit = hdgc_graph{u, w, inflow, dtb, nsteps, exec};
  }
  CUDA_TRY(cudaGraphLaunch(hit->exec, st));
  return HDGC_OK;
}

int hdgc_substeps(hdgc_ctx* c, const double* u, double* w, const double* inflow, double dt, int32_t nsteps,
                  void* stream) {
  if (!c || !u || !w) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (nsteps < 0) return hdgc_set_err(HDGC_EINVAL, "nsteps < 0");
  if (w == u || w == inflow) return hdgc_set_err(HDGC_EINVAL, "w aliases an input");
  HDGC_ALIGNED(u, w, inflow);
  cudaStream_t st = (cudaStream_t)stream;
  if (nsteps == 0) return HDGC_OK;
  if (graphs_enabled()) return substeps_graph(c, u, w, inflow, dt, nsteps, st);
  return substeps_enqueue(c, u, w, inflow, dt, nsteps, st);
}

int hdgc_propagate(hdgc_ctx* c, const double* u_prev, const double* u_cur, double t_prev, double t_cur,
                   double t1, double ds, int32_t nsteps, int32_t scheme, const double* inflow, double* w,
                   void* stream) {
  if (!c || !u_cur || !w) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (nsteps < 0) return hdgc_set_err(HDGC_EINVAL, "nsteps < 0");
  if (scheme != 0 && scheme != 1) return hdgc_set_err(HDGC_EINVAL, "scheme must be 0 (Euler) or 1 (SSP-RK2)");
  if (w == u_cur || w == u_prev || w == inflow) return hdgc_set_err(HDGC_EINVAL, "w aliases an input");
  if (u_prev && !(t_cur != t_prev)) return hdgc_set_err(HDGC_EINVAL, "extrapolation needs t_cur != t_prev");
  HDGC_ALIGNED(u_prev, u_cur, inflow, w);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)c->nt * c->nb;
  int rc;
  if (u_prev && !c->d_uext && (rc = hdgc_dev_alloc(c, (void**)&c->d_uext, sizeof(double) * n))) return rc;
  if (scheme == 1 && !c->d_scratch2 && (rc = hdgc_dev_alloc(c, (void**)&c->d_scratch2, sizeof(double) * n)))
    return rc;
  // velocity at pseudo time s; the prep (variants 1/2) is redone only when s changes
  bool have = false;
  bool after_update = false;   // last launch on st was an update kernel: the next may use PDL
  double at = 0.0;
  auto velocity = [&](double s, const double** uu) -> int {
    if (!u_prev) {
      *uu = u_cur;
      if (!have) { have = true; after_update = false; return prep_any(c, u_cur, st, nsteps * (scheme + 1)); }
      return HDGC_OK;
    }
    *uu = c->d_uext;
    if (have && s == at) return HDGC_OK;
    after_update = false;
    const double th = (s - t_cur) / (t_cur - t_prev);
    axpby_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(u_cur, u_prev, 1.0 + th, -th, c->d_uext, n);
    CUDA_TRY(cudaGetLastError());
    have = true;
    at = s;
    return prep_any(c, c->d_uext, st, scheme + 1);   // one prep per pseudo-time level
  };
  double* bufs[3] = {w, c->d_scratch, c->d_scratch2};
  const int nbuf = scheme == 1 ? 3 : 2;   // Euler ping-pongs, Heun rotates v, v1, v'
  int cur = 0;
  for (int i = 0; i < nsteps; ++i) {
    const double s0 = t1 + i * ds, s1 = t1 + (i + 1) * ds;
    const double* uu = nullptr;
    if ((rc = velocity(s0, &uu))) return rc;
    double* v = bufs[cur];
    double* v1 = bufs[(cur + 1) % nbuf];
    StageParams sp;
    sp.c = -ds;
    // PDL between back-to-back update kernels (common.cuh); not after a prep / axpby
    c->pdl = after_update && c->n_curved == 0;
    rc = apply_any(c, MODE_SUBSTEP, uu, v, inflow, v1, sp, true, st);
    c->pdl = false;
    if (rc) return rc;
    after_update = true;
    if (scheme == 0) { cur = (cur + 1) % nbuf; continue; }
    if ((rc = velocity(s1, &uu))) return rc;
    double* v2 = bufs[(cur + 2) % 3];
    StageParams s2;
    s2.a = 0.5; s2.b = 0.5; s2.c = -0.5 * ds; s2.x = v;
    c->pdl = after_update && c->n_curved == 0;
    rc = apply_any(c, MODE_STAGE, uu, v1, inflow, v2, s2, true, st);
    c->pdl = false;
    if (rc) return rc;
    after_update = true;
    cur = (cur + 2) % 3;
  }
  if (bufs[cur] != w) CUDA_TRY(cudaMemcpyAsync(w, bufs[cur], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  return HDGC_OK;
}

int hdgc_richardson(hdgc_ctx* c, const double* u, const double* g, const double* inflow, double tau, double ds,
                    double rho, int32_t max_iter, double* v, int32_t* iters, double* res0, double* res_final,
                    void* stream) {
  if (!c || !u || !g || !v) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (max_iter < 0) return hdgc_set_err(HDGC_EINVAL, "max_iter < 0");
  if (v == u || v == g || v == inflow) return hdgc_set_err(HDGC_EINVAL, "v aliases an input");
  HDGC_ALIGNED(u, g, inflow, v);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)c->nt * c->nb, nr = (size_t)c->nt * c->dim;
  int rc;
  if (!c->d_rn && (rc = hdgc_dev_alloc(c, (void**)&c->d_rn, sizeof(double) * nr))) return rc;
  if (!c->d_rpart && (rc = hdgc_dev_alloc(c, (void**)&c->d_rpart, sizeof(double) * RED_CTAS))) return rc;
  if (!c->d_ctl && (rc = hdgc_dev_alloc(c, (void**)&c->d_ctl, sizeof(int) * 4))) return rc;
  if (c->n_norms < max_iter + 1) {
    cudaFree(c->d_norms);
    c->d_norms = nullptr;
    if ((rc = hdgc_dev_alloc(c, (void**)&c->d_norms, sizeof(double) * (max_iter + 1)))) return rc;
    c->n_norms = max_iter + 1;
  }
  if (!c->h_ctl) CUDA_TRY(cudaMallocHost((void**)&c->h_ctl, sizeof(int) * 12));
  for (int i = 0; i < 2; ++i)
    if (!c->ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  // sum-factorised kernels (no curved elements) reduce the residual norm inside
  // the STAGE kernel (StageParams::rpart, rich_fused_reduce) and launch back to
  // back with PDL; the others write per-(element, component) sums that
  // richardson_reduce_kernel reduces
  const bool fused = c->variant == 1 && c->n_curved == 0;
  const int nblk = (c->nt + 15) / 16;        // CTAs of the sum-factorised kernels (16 elements each)
  if (fused && !c->d_fpart && (rc = hdgc_dev_alloc(c, (void**)&c->d_fpart, sizeof(double) * nblk))) return rc;
  if ((rc = prep_any(c, u, st))) return rc;   // convection frozen over the solve
  CUDA_TRY(cudaMemsetAsync(c->d_ctl, 0, sizeof(int) * 4, st));
  double* bufs[2] = {v, c->d_scratch};        // iteration it reads bufs[it & 1], writes bufs[(it + 1) & 1]
  StageParams sp;
  sp.a = 1.0 - ds; sp.b = ds; sp.c = -ds * tau; sp.tau = tau; sp.x = g; sp.stop = c->d_ctl;
  if (fused) sp.rpart = c->d_fpart;
  else sp.rn = c->d_rn;
  // No host round trip per iteration: iterations are queued in chunks of CH,
  // each chunk followed by an async copy of the control block; the host waits
  // only for the chunk BEFORE the one just queued, so the GPU always has a
  // chunk of work ahead while the host decides whether to queue more.
  constexpr int CH = 8;
  int chunk = 0;
  for (int it = 0; it <= max_iter; ++it) {
    // fused: STAGE -> final -> STAGE ... all with PDL (the stop flag is read after griddepcontrol.wait)
    c->pdl = fused && it > 0;
    rc = apply_any(c, MODE_STAGE, u, bufs[it & 1], inflow, bufs[(it + 1) & 1], sp, true, st);
    c->pdl = false;
    if (rc) return rc;
    if (fused) {
      CUDA_TRY(launch_maybe_pdl(richardson_final_kernel, 1, 1024, 0, st, true, (const double*)c->d_fpart, nblk, it,
                                rho, c->d_norms, c->d_ctl));
    } else {
      richardson_reduce_kernel<<<RED_CTAS, RED_THREADS, 0, st>>>(c->d_rn, nr, it, rho, c->d_rpart, c->d_norms,
                                                                 c->d_ctl);
      CUDA_TRY(cudaGetLastError());
    }
    if ((it + 1) % CH == 0 && it < max_iter) {
      const int slot = chunk & 1;
      CUDA_TRY(cudaMemcpyAsync(c->h_ctl + 4 * slot, c->d_ctl, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaEventRecord(c->ev[slot], st));
      if (chunk > 0) {
        CUDA_TRY(cudaEventSynchronize(c->ev[slot ^ 1]));
        if (c->h_ctl[4 * (slot ^ 1)] != 0) break;   // stopped: what is queued after it are no-ops
      }
      ++chunk;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(c->h_ctl + 8, c->d_ctl, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int* ctl = c->h_ctl + 8;
  const int it = ctl[0] ? ctl[1] : max_iter;
  double nrm[2] = {0.0, 0.0};
  CUDA_TRY(cudaMemcpy(&nrm[0], c->d_norms, sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&nrm[1], c->d_norms + it, sizeof(double), cudaMemcpyDeviceToHost));
  if (iters) *iters = it;
  if (res0) *res0 = nrm[0];
  if (res_final) *res_final = nrm[1];
  if (ctl[2]) {
    hdgc_check_finite(c, stream);
    return hdgc_set_err(HDGC_EBLOWUP, "richardson: non-finite residual norm at iteration %d (norm blow-up)", it);
  }
  if (bufs[it & 1] != v) {
    CUDA_TRY(cudaMemcpyAsync(v, bufs[it & 1], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (!ctl[0])
    return hdgc_set_err(HDGC_ENOCONV, "richardson: ||res|| %.3e > rho ||res_0|| after %d iterations", nrm[1], it);
  return HDGC_OK;
}

int hdgc_set_dofmap(hdgc_ctx* c, int64_t ndof, const int64_t* element_dofs, const double* factors) {
  if (!c || !element_dofs || !factors) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (c->dim != 2) return hdgc_set_err(HDGC_EUNSUP, "global H(div) dof map: 2D contexts only");
  const size_t n = (size_t)c->nt * c->nb;
  if (ndof <= 0 || ndof >= (int64_t)1 << 31 || n >= (size_t)1 << 31)
    return hdgc_set_err(HDGC_EINVAL, "ndof %lld out of range", (long long)ndof);
  std::vector<int32_t> dof(n), inv(2 * (size_t)ndof, -1);
  std::vector<double> invf(2 * (size_t)ndof, 0.0);
  for (size_t i = 0; i < n; ++i) {
    const int64_t d = element_dofs[i];
    if (d < 0 || d >= ndof) return hdgc_set_err(HDGC_EINVAL, "element_dofs[%zu] = %lld out of range", i, (long long)d);
    dof[i] = (int32_t)d;
    int32_t* slot = &inv[2 * (size_t)d];
    const int s = slot[0] < 0 ? 0 : (slot[1] < 0 ? 1 : 2);
    if (s == 2) return hdgc_set_err(HDGC_EINVAL, "global dof %lld used by more than two local dofs", (long long)d);
    slot[s] = (int32_t)i;
    invf[2 * (size_t)d + s] = factors[i];
  }
  for (int64_t d = 0; d < ndof; ++d)
    if (inv[2 * (size_t)d] < 0) return hdgc_set_err(HDGC_EINVAL, "global dof %lld is not used", (long long)d);
  cudaFree(c->d_dof); cudaFree(c->d_dfac); cudaFree(c->d_inv); cudaFree(c->d_invf);
  c->d_dof = nullptr; c->d_dfac = nullptr; c->d_inv = nullptr; c->d_invf = nullptr;
  int rc;
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_dof, sizeof(int32_t) * n))) return rc;
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_dfac, sizeof(double) * n))) return rc;
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_inv, sizeof(int32_t) * 2 * (size_t)ndof))) return rc;
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_invf, sizeof(double) * 2 * (size_t)ndof))) return rc;
  CUDA_TRY(cudaMemcpy(c->d_dof, dof.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_dfac, factors, sizeof(double) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_inv, inv.data(), sizeof(int32_t) * inv.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_invf, invf.data(), sizeof(double) * invf.size(), cudaMemcpyHostToDevice));
  c->ndof = ndof;
  return HDGC_OK;
}

int hdgc_gather(hdgc_ctx* c, const double* u_glob, double* u_loc, void* stream) {
  if (!c || !u_glob || !u_loc) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (!c->d_dof) return hdgc_set_err(HDGC_EINVAL, "no dof map installed (hdgc_set_dofmap)");
  const size_t n = (size_t)c->nt * c->nb;
  gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(c->d_dof, c->d_dfac, u_glob, u_loc, n);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

int hdgc_scatter(hdgc_ctx* c, const double* r_loc, double* r_glob, void* stream) {
  if (!c || !r_loc || !r_glob) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (!c->d_inv) return hdgc_set_err(HDGC_EINVAL, "no dof map installed (hdgc_set_dofmap)");
  const size_t nd = (size_t)c->ndof;
  scatter_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, (cudaStream_t)stream>>>(c->d_inv, c->d_invf, r_loc, r_glob, nd);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

int hdgc_apply_u(hdgc_ctx* c, const double* u_glob, const double* inflow, double* r_glob, void* stream) {
  if (!c || !u_glob || !r_glob) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (r_glob == u_glob) return hdgc_set_err(HDGC_EINVAL, "output aliases an input");
  const size_t n = (size_t)c->nt * c->nb;
  int rc;
  if (!c->d_gl && (rc = hdgc_dev_alloc(c, (void**)&c->d_gl, sizeof(double) * n))) return rc;
  if (!c->d_rw && (rc = hdgc_dev_alloc(c, (void**)&c->d_rw, sizeof(double) * n))) return rc;
  if ((rc = hdgc_gather(c, u_glob, c->d_gl, stream))) return rc;
  if ((rc = hdgc_apply_w(c, c->d_gl, inflow, c->d_rw, stream))) return rc;
  return hdgc_scatter(c, c->d_rw, r_glob, stream);
}

int hdgc_transfer(hdgc_ctx* c, int32_t direction, const double* in, double* out, void* stream) {
  if (!c || !in || !out) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (in == out) return hdgc_set_err(HDGC_EINVAL, "output aliases input");
  if (direction != 0 && direction != 1) return hdgc_set_err(HDGC_EINVAL, "direction must be 0 (I) or 1 (I^T)");
  HDGC_ALIGNED(in, out);
  return transfer(c, direction, in, out, (cudaStream_t)stream);
}

int hdgc_mass_inverse(hdgc_ctx* c, double* out, void* stream) {
  if (!c || !out) return hdgc_set_err(HDGC_EINVAL, "null argument");
  CUDA_TRY(cudaMemcpyAsync(out, c->d_minv, sizeof(double) * c->nt, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return HDGC_OK;
}

static int maxspeed_affine(hdgc_ctx* c, const double* u, double* out, cudaStream_t st) {
  HDGC_K_SWITCH(c->k, launch_maxspeed<KK>(c, u, out, st));
}

int hdgc_max_speed(hdgc_ctx* c, const double* u, double* out_dev, void* stream) {
  if (!c || !u || !out_dev) return hdgc_set_err(HDGC_EINVAL, "null argument");
  if (c->dim == 3) return maxspeed3(c, u, out_dev, (cudaStream_t)stream);
  int rc = maxspeed_affine(c, u, out_dev, (cudaStream_t)stream);
  if (rc || c->n_curved == 0) return rc;
  const int th = 256, work = c->n_curved * c->nqv, nbs1 = c->k * (c->k + 1) / 2;
  const size_t off_vd = (size_t)c->nb * c->nb + (size_t)nbs1 * c->nb + c->nqv;   // Dims<K>::OFF_VD
  curved_maxspeed_kernel<<<(work + th - 1) / th, th, 0, (cudaStream_t)stream>>>(
      c->d_celems, c->n_curved, c->nbs, c->nb + nbs1, c->nqv, c->d_tab + off_vd, c->d_modal, c->d_cpiola,
      reinterpret_cast<unsigned long long*>(out_dev));
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

int hdgc_set_curved(hdgc_ctx* c, int32_t n, const int32_t* elems, const double* minv_blocks,
                    const double* itrans, const double* piola) {
  if (!c) return hdgc_set_err(HDGC_EINVAL, "null context");
  if (c->dim != 2) return hdgc_set_err(HDGC_EUNSUP, "curved elements: 2D contexts only");
  if (c->n_curved) return hdgc_set_err(HDGC_EINVAL, "curved elements already installed on this context");
  if (n < 0 || n > c->nt) return hdgc_set_err(HDGC_EINVAL, "n_curved=%d out of range", n);
  if (n == 0) return HDGC_OK;
  if (!elems || !minv_blocks || !itrans || !piola) return hdgc_set_err(HDGC_EINVAL, "null argument");
  for (int i = 0; i < n; ++i) {
    if (elems[i] < 0 || elems[i] >= c->nt) return hdgc_set_err(HDGC_EINVAL, "curved element %d out of range", elems[i]);
    if (i && elems[i] <= elems[i - 1]) return hdgc_set_err(HDGC_EINVAL, "curved element ids must ascend");
  }
  const size_t nbs2 = (size_t)c->nbs * c->nbs, nb2 = (size_t)c->nb * c->nb, pq = (size_t)c->nqv * 4;
  int rc;
  if ((rc = hdgc_dev_alloc(c, (void**)&c->d_celems, sizeof(int32_t) * n)) ||
      (rc = hdgc_dev_alloc(c, (void**)&c->d_cminv, sizeof(double) * n * nbs2)) ||
      (rc = hdgc_dev_alloc(c, (void**)&c->d_citrans, sizeof(double) * n * nb2)) ||
      (rc = hdgc_dev_alloc(c, (void**)&c->d_cpiola, sizeof(double) * n * pq)) ||
      (rc = hdgc_dev_alloc(c, (void**)&c->d_cres, sizeof(double) * n * c->nb)))
    return rc;
  CUDA_TRY(cudaMemcpy(c->d_celems, elems, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_cminv, minv_blocks, sizeof(double) * n * nbs2, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_citrans, itrans, sizeof(double) * n * nb2, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_cpiola, piola, sizeof(double) * n * pq, cudaMemcpyHostToDevice));
  mark_curved_kernel<<<(n + 127) / 128, 128>>>(c->d_celems, n, c->d_minv);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  c->n_curved = n;
  return HDGC_OK;
}

static int ensure_staging(hdgc_ctx* c, bool need_inflow) {
  const size_t vec = sizeof(double) * (size_t)c->nt * c->nb;
  int rc;
  if (!c->d_hu && (rc = hdgc_dev_alloc(c, (void**)&c->d_hu, vec))) return rc;
  if (!c->d_hw && (rc = hdgc_dev_alloc(c, (void**)&c->d_hw, vec))) return rc;
  if (!c->d_hr && (rc = hdgc_dev_alloc(c, (void**)&c->d_hr, vec))) return rc;
  if (need_inflow && !c->d_hin && c->nbf > 0 &&
      (rc = hdgc_dev_alloc(c, (void**)&c->d_hin, sizeof(double) * (size_t)c->nbf * c->nf * c->dim)))
    return rc;
  return HDGC_OK;
}

int hdgc_apply_v_host(hdgc_ctx* c, const double* u, const double* w, const double* inflow, double* r, void* stream) {
  if (!c || !u || !w || !r) return hdgc_set_err(HDGC_EINVAL, "null argument");
  int rc = ensure_staging(c, inflow != nullptr);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t vec = sizeof(double) * (size_t)c->nt * c->nb;
  CUDA_TRY(cudaMemcpyAsync(c->d_hu, u, vec, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->d_hw, w, vec, cudaMemcpyHostToDevice, st));
  const double* din = nullptr;
  if (inflow && c->nbf > 0) {
    CUDA_TRY(cudaMemcpyAsync(c->d_hin, inflow, sizeof(double) * (size_t)c->nbf * c->nf * c->dim, cudaMemcpyHostToDevice, st));
    din = c->d_hin;
  }
  if ((rc = apply_any(c, MODE_APPLY, c->d_hu, c->d_hw, din, c->d_hr, 0.0, false, st))) return rc;
  CUDA_TRY(cudaMemcpyAsync(r, c->d_hr, vec, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return HDGC_OK;
}

int hdgc_substeps_host(hdgc_ctx* c, const double* u, double* w, const double* inflow, double dt, int32_t nsteps,
                       void* stream) {
  if (!c || !u || !w) return hdgc_set_err(HDGC_EINVAL, "null argument");
  int rc = ensure_staging(c, inflow != nullptr);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t vec = sizeof(double) * (size_t)c->nt * c->nb;
  CUDA_TRY(cudaMemcpyAsync(c->d_hu, u, vec, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->d_hw, w, vec, cudaMemcpyHostToDevice, st));
  const double* din = nullptr;
  if (inflow && c->nbf > 0) {
    CUDA_TRY(cudaMemcpyAsync(c->d_hin, inflow, sizeof(double) * (size_t)c->nbf * c->nf * c->dim, cudaMemcpyHostToDevice, st));
    din = c->d_hin;
  }
  if ((rc = hdgc_substeps(c, c->d_hu, c->d_hw, din, dt, nsteps, stream))) return rc;
  CUDA_TRY(cudaMemcpyAsync(w, c->d_hw, vec, cudaMemcpyDeviceToHost, st));
  return hdgc_check_finite(c, stream);   // synchronises the stream
}

}  // extern "C"
