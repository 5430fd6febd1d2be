// context.cuh — device context, error plumbing and the per-order entry
// points shared by hdgconv.cu (C ABI) and the per-order translation units
// order_k*.cu (one per k, compiled in parallel).
#pragma once
#include "../../include/hdgconv.h"

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "common.cuh"

int hdgc_set_err(int code, const char* fmt, ...);

#define CUDA_TRY(x)                                                                           \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      return hdgc_set_err(HDGC_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
                          __LINE__);                                                          \
  } while (0)

// one captured substep batch (hdgc_substeps), keyed by its arguments
struct hdgc_graph {
  const double* u = nullptr;
  const double* w = nullptr;
  const double* inflow = nullptr;
  uint64_t dt_bits = 0;
  int nsteps = 0;
  cudaGraphExec_t exec = nullptr;
};
constexpr int HDGC_GRAPH_CACHE = 4;

struct hdgc_ctx {
  int dim = 2, k = 0, nb = 0, nbs = 0, nqv = 0, nf = 0;
  int nt = 0, nf_facets = 0, nbf = 0, nv = 0;
  double* d_tab = nullptr;      // packed tables (Dims<K> layout)
  int32_t* d_code = nullptr;    // (NT, 3) neighbour codes
  double* d_piola = nullptr;    // (4, NT) J/detJ
  double* d_minv = nullptr;     // (NT,) 2/detJ
  double* d_scratch = nullptr;  // (NT, nb) ping-pong / I u
  double* d_prep = nullptr;     // (NT, PREP) frozen-velocity data (sum-factorised variant)
  double* d_modal = nullptr;    // (NT, nb + nbs(k-1)) modal u_hat | div u_hat
  double* d_scratch2 = nullptr; // (NT, nb) r_V for apply_w (lazily allocated)
  double* d_sign = nullptr;     // (NT,) sign(detJ) (3D: sorted-vertex tets)
  double* d_ftab = nullptr;     // facet tables fw | fD (sum-factorised variant)
  double* d_afrag = nullptr;    // DMMA A fragments of [coef ; divm] (tile prep, k = 3..6)
  double* d_mprep = nullptr;    // modal frozen-velocity prep [tile][MP][16] (conv2d_sfm.cuh)
  bool modal = false;           // the sum-factorised variant uses the modal prep + conv2d_sfm_kernel
  // host-variant staging (lazily allocated)
  double* d_hu = nullptr;
  double* d_hw = nullptr;
  double* d_hr = nullptr;
  double* d_hin = nullptr;
  double* d_uext = nullptr;     // (NT, nb) extrapolated velocity (propagate, lazily allocated)
  double* d_rn = nullptr;       // (NT, dim) residual sums of squares (richardson)
  double* d_rpart = nullptr;    // (RED_CTAS,) Richardson reduction partials
  double* d_fpart = nullptr;    // Richardson CTA partials of the sum-factorised STAGE kernels
  int* d_ctl = nullptr;         // (4,) Richardson device control block (stop, iteration, blow-up, counter)
  double* d_norms = nullptr;    // (n_norms,) residual norm per iteration
  int n_norms = 0;
  int* h_ctl = nullptr;         // pinned (12,) control-block copies (two chunk slots + final)
  cudaEvent_t ev[2] = {nullptr, nullptr};
  hdgc_graph graphs[HDGC_GRAPH_CACHE];  // captured substep batches (LRU)
  int graph_next = 0;
  cudaStream_t cap_stream = nullptr;    // private stream the batches are captured on
  int64_t ndof = 0;             // global H(div) dof map (hdgc_set_dofmap)
  int32_t* d_dof = nullptr;     // (NT, nb) global dof of each local dof
  double* d_dfac = nullptr;     // (NT, nb) local = factor * global
  int32_t* d_inv = nullptr;     // (ndof, 2) flat local index T*nb+j (or -1), ascending
  double* d_invf = nullptr;     // (ndof, 2) factors of d_inv
  double* d_gl = nullptr;       // (NT, nb) gathered u_loc (apply_u)
  double* d_rw = nullptr;       // (NT, nb) r_W (apply_u)
  // curved elements (hdgc_set_curved): d_minv[T] = -(slot + 1) marks them
  int n_curved = 0;
  int32_t* d_celems = nullptr;  // (n_curved,) element ids, ascending
  double* d_cminv = nullptr;    // (n_curved, nbs, nbs) inverse mass blocks
  double* d_citrans = nullptr;  // (n_curved, nb, nb) I_T (L2 projection), I^T = I_T^T
  double* d_cpiola = nullptr;   // (n_curved, nqv, 4) J/detJ at the volume points
  double* d_cres = nullptr;     // (n_curved, nb) raw residual rows (update kernels -> fix-up)
  int* d_flag = nullptr;        // (1,) norm-blowup flag set by the update epilogues (StageParams::flag)
  int* h_flag = nullptr;        // pinned host copy of d_flag
  int64_t bytes = 0;
  int variant = 0;              // 0: thread-per-element (k <= 2), 1: sum-factorised (k >= 3)
  bool pdl = false;             // next update kernel may launch with PDL (set by hdgc_substeps only)
  double* d_tprep = nullptr;    // k <= 2: frozen-velocity rows of prep_thread2d_kernel (allocated on first use)
  bool tprep_valid = false;     // d_tprep holds the rows of the u last passed to prep_any
  bool tprep_on = false;        // the next thread-variant launch reads d_tprep (set by apply_any_)
  unsigned sweep = 0;           // launch counter of the sum-factorised update kernel (alternating tile sweeps)
  bool prep_dep = false;        // ... and it follows a prep kernel (stages the prep after griddepcontrol.wait)
};

int hdgc_dev_alloc(hdgc_ctx* c, void** p, size_t bytes);
// c->d_modal[T][r] = sum_j M[r][j] u[T][j] for r < nr (M row-major [nr][nb] at
// c->d_tab + off), all elements, on stream st (modal_rows_kernel).
int hdgc_modal_gemm(hdgc_ctx* c, const double* u, int nb, int nr, size_t off, cudaStream_t st);

namespace hdgc {
// per-order operations, explicitly instantiated in order_k<K>.cu
template <int K> int launch_elem(hdgc_ctx* c, int mode, const double* u, const double* w,
                                 const double* inflow, double* out, const StageParams& sp, cudaStream_t st);
template <int K> int launch_elem_prep(hdgc_ctx* c, const double* u, cudaStream_t st);
template <int K> int launch_transfer(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st);
template <int K> int launch_maxspeed(hdgc_ctx* c, const double* u, double* out, cudaStream_t st);
template <int K> int sf_prep(hdgc_ctx* c, const double* u, cudaStream_t st);
template <int K> int sf_main(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out,
                             const StageParams& sp, cudaStream_t st);
template <int K> int sf_setup(hdgc_ctx* c, const hdgc_tables_desc* t, const std::vector<double>& packed);

// 3D (tetrahedra), order3d_k<K>.cu
template <int K> int launch3_prep(hdgc_ctx* c, const double* u, cudaStream_t st);
template <int K> int launch3_main(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out,
                                  const StageParams& sp, cudaStream_t st);
template <int K> int launch3_transfer(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st);
template <int K> int launch3_maxspeed(hdgc_ctx* c, const double* u, double* out, cudaStream_t st);
template <int K> int launch3_setup(hdgc_ctx* c, const hdgc_tables_desc* t);

#define HDGC_DECLARE_ORDER3(K)                                                                     \
  extern template int launch3_prep<K>(hdgc_ctx*, const double*, cudaStream_t);                    \
  extern template int launch3_main<K>(hdgc_ctx*, int, const double*, const double*, double*, const StageParams&, \
                                      cudaStream_t);                                               \
  extern template int launch3_transfer<K>(hdgc_ctx*, int, const double*, double*, cudaStream_t);  \
  extern template int launch3_maxspeed<K>(hdgc_ctx*, const double*, double*, cudaStream_t);      \
  extern template int launch3_setup<K>(hdgc_ctx*, const hdgc_tables_desc*);

#define HDGC_DECLARE_ORDER(K)                                                                      \
  extern template int launch_elem<K>(hdgc_ctx*, int, const double*, const double*, const double*,  \
                                     double*, const StageParams&, cudaStream_t);                               \
  extern template int launch_transfer<K>(hdgc_ctx*, int, const double*, double*, cudaStream_t);    \
  extern template int launch_maxspeed<K>(hdgc_ctx*, const double*, double*, cudaStream_t);         \
  extern template int sf_prep<K>(hdgc_ctx*, const double*, cudaStream_t);                          \
  extern template int sf_main<K>(hdgc_ctx*, int, const double*, const double*, double*, const StageParams&, \
                                 cudaStream_t);                                                    \
  extern template int sf_setup<K>(hdgc_ctx*, const hdgc_tables_desc*, const std::vector<double>&); \
  extern template int launch_elem_prep<K>(hdgc_ctx*, const double*, cudaStream_t);
}  // namespace hdgc
