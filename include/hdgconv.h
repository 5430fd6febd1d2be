/*
 * hdgconv.h — C ABI of the B200 (sm_100a) fp64 upwind-DG convection apply.
 *
 * Drop-in boundary for the reference's convection entry point
 *   forms.apply_convection(u_conv, w, data) -> residual over V_h
 *   (operator PAPER.md:424-436)
 * and for the explicit substep loop that calls it
 *   timeloop.propagate_convection,
 * plus the transfer operators I / I^T.
 *
 * Conventions:
 *  - u_loc (NT, nb): element-local BDM_k coefficients in BDMBasis member
 *    order: edge e=0..2 x Legendre mode 0..k, then interior moments
 *    (polybasis.py:265-268, 315-354).
 *  - w, r (NT, nb): V_h coefficients, index c*nbs + m, c in {x,y}, m in
 *    dubiner_index(k) order (polybasis.py:174-176, 282-289).
 *  - inflow (NBF, nf, 2): exterior values on boundary facets, rows in
 *    boundary-facet order (facet index order of mesh2d.py:178-207), points
 *    of quad_interval(3k+1) along the owner's traversal.  NULL = interior
 *    trace everywhere (no inflow data).
 *  - all fp64, row-major, contiguous.
 *
 * Memory: every double* argument of the compute calls is a DEVICE pointer
 * owned by the caller, 16-byte aligned (rows move with 16-byte vector loads
 * and TMA bulk copies; misaligned pointers are rejected with HDGC_EINVAL), no
 * allocation in hot calls, except the *_host
 * variants, which take pageable or pinned HOST pointers and stage through
 * context-owned device buffers.  `stream` is a cudaStream_t (NULL = legacy
 * default stream); all calls are asynchronous on it except the *_host ones,
 * which synchronise the stream before returning.
 *
 * Errors: every call returns 0 on success, a negative HDGC_E* code on
 * failure; hdgc_last_error() returns a thread-local message.  No C++
 * exception crosses this boundary.
 *
 * Determinism: element-owned passes, no atomics, fixed summation order —
 * results are bitwise reproducible run to run on the same GPU.
 */
#ifndef HDGCONV_H
#define HDGCONV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDGC_OK 0
#define HDGC_EINVAL (-1)   /* bad argument / inconsistent descriptor */
#define HDGC_ECUDA (-2)    /* CUDA runtime error */
#define HDGC_ENOMEM (-3)   /* device allocation failed */
#define HDGC_EUNSUP (-4)   /* unsupported order / dimension */
#define HDGC_ENOCONV (-5)  /* Richardson iteration hit max_iter (result = last iterate) */
#define HDGC_EBLOWUP (-6)  /* norm blow-up: an explicit update produced non-finite values */

typedef struct hdgc_ctx hdgc_ctx;

/* Mesh topology + affine geometry, HOST arrays (copied at create).
 * Mirrors hdgflow.mesh2d.Mesh (mesh2d.py:86-150): CCW triangles, facets in
 * sorted-vertex-key order, facet_elems[:,1] = -1 on the boundary. */
typedef struct {
  int32_t dim;               /* 2 (triangles); 3 (tetrahedra) */
  int32_t n_vertices;
  int32_t n_elements;
  int32_t n_facets;
  const double* vertices;    /* (NV, dim) */
  const int64_t* elements;   /* (NT, dim+1) vertex ids */
  const int64_t* facet_elems;/* (NF, 2) */
  const int64_t* facet_local;/* (NF, 2) */
  const int32_t* facet_perm; /* reserved, must be NULL.  3D meshes must list every tet's vertex
                              * ids in ascending order (mesh3d.py does): a shared face then has the
                              * same vertex order, hence the same face parametrisation, on both
                              * sides, and no face permutation is needed.  Unsorted tets are
                              * rejected with HDGC_EINVAL. */
} hdgc_mesh_desc;

/* Reference-element tables, HOST arrays (copied at create), produced by the
 * host-side basis module (restating polybasis.py:47-378). */
typedef struct {
  int32_t k;                 /* polynomial order */
  int32_t nqv;               /* volume rule size, quad_triangle(3k-1) */
  int32_t nf;                /* facet rule size, quad_interval(3k+1) (2D) */
  const double* coef;        /* (nb, nb) BDM dual basis: raw -> member (polybasis.py:357-378) */
  const double* div_modal;   /* (nbs(k-1), nb) div of each BDM member in the Dubiner P_{k-1} basis */
  const double* vol_w;       /* (nqv) */
  const double* vol_D;       /* (nqv, nbs)   Dubiner values */
  const double* vol_G;       /* (nqv, nbs, dim) Dubiner reference gradients */
  const double* fac_w;       /* (nf) */
  const double* fac_L;       /* (nf, nfd) facet normal-trace basis at facet points */
  const double* fac_D;       /* (nfaces, nf, nbs) Dubiner on each reference facet */
  const double* fac_len;     /* (nfaces) reference facet measures |e_hat| */
  /* sum-factorisation tables on the collapsed volume rule (2D, k >= 3; else 0/NULL):
   * D_ij(xi_a, y_b) = A_i(a) B_ij(b); see basis.collapsed_tables */
  int32_t col_n;             /* points per direction, (3k+1)/2 */
  const double* col_A;       /* (n, k+1) P_i(2 xi_a - 1) */
  const double* col_Ad;      /* (n, k+1) d/dxi */
  const double* col_B;       /* (n, nbs) c_ij (1-y_b)^i P_j^(2i+1,0)(2 y_b - 1) */
  const double* col_Bd;      /* (n, nbs) d/dy at fixed xi */
  const double* col_xi;      /* (n) */
  const double* col_wa;      /* (n) */
  const double* col_wy;      /* (n) */
  const double* col_inv1my;  /* (n) 1/(1-y_b) */
  /* 3D sum-factorisation (tets): D_ijl(a,b,c) = A_i(a) B_ij(b) C_ijl(c), see
   * basis3d.collapsed_tables3; col_A/col_Ad/col_B/col_Bd hold the a- and
   * b-factors, col_B indexed by the pair (i,j) */
  const double* col_C;       /* (n, nbs) */
  const double* col_Cd;      /* (n, nbs) d/dc */
  const double* col_pf;      /* (n^3, 5) per point: w/t1, w a/t1, w/t2, w b/t2, w */
} hdgc_tables_desc;

typedef struct {
  int32_t dim, k, nb, nbs, nqv, nf;
  int32_t n_elements, n_facets, n_boundary_facets;
  int32_t volume_variant;    /* kernel variant chosen for this k */
  int64_t device_bytes;      /* context-owned device memory */
} hdgc_info;

/* Build a context: uploads tables, runs the on-device geometry/adjacency
 * precompute (Piola factors J/detJ, 2/detJ, neighbour codes, boundary slots).
 * The mesh is validated on the device: vertex ids in range, element ids and
 * local facet ids in range, every (element, local facet) in exactly one facet,
 * positive detJ (2D) / nonzero detJ and ascending vertex ids (3D); failures
 * return HDGC_EINVAL with the reason in hdgc_last_error(). */
int hdgc_create(const hdgc_mesh_desc* mesh, const hdgc_tables_desc* tables, hdgc_ctx** out);

/* The same from (mesh, dim = mesh->dim, k) alone: the library
 * carries the reference-element tables of every supported order (2D k = 1..8,
 * 3D k = 1..4), generated at build time by the package's basis modules
 * (restating polybasis.py:47-378, bit-identical to the reference's tables) —
 * a caller without Python needs only the mesh arrays.  HDGC_EUNSUP for other
 * (dim, k). */
int hdgc_create_k(const hdgc_mesh_desc* mesh, int32_t k, hdgc_ctx** out);
int hdgc_destroy(hdgc_ctx* ctx);
int hdgc_get_info(const hdgc_ctx* ctx, hdgc_info* info);

/* r = C^V(u; w).  r must not alias u, w or inflow. */
int hdgc_apply_v(hdgc_ctx* ctx, const double* u_loc, const double* w, const double* inflow,
                 double* r, void* stream);

/* r_w = I^T C^V(u; I u): the HDG-side operator C^U u, output in
 * element-local BDM-test layout (same layout as u_loc). */
int hdgc_apply_w(hdgc_ctx* ctx, const double* u_loc, const double* inflow, double* r_w,
                 void* stream);

/* nsteps forward-Euler substeps, u frozen, device-resident:
 *   w <- w - dt * (M^V)^{-1} C^V(u; w),  (M^V)^{-1} = 2/detJ per element. */
int hdgc_substeps(hdgc_ctx* ctx, const double* u_loc, double* w_inout, const double* inflow,
                  double dt, int32_t nsteps, void* stream);

/* Convection propagation Q^{t1 -> t1 + nsteps ds} (SPEC.md:429-437,
 * timeloop.propagate_convection), device-resident:
 *   scheme 0: forward Euler, 1: SSP-RK2 (Heun: v1 = v - ds M^-1 C(s) v,
 *   v' = v/2 + (v1 - ds M^-1 C(s + ds) v1)/2).
 * Convecting velocity at pseudo time s: u_cur if u_prev is NULL (frozen),
 * else the linear extrapolation u(s) = u_cur + (s - t_cur)/(t_cur - t_prev)
 * (u_cur - u_prev) of two stored divergence-free fields. */
int hdgc_propagate(hdgc_ctx* ctx, const double* u_prev, const double* u_cur, double t_prev, double t_cur,
                   double t1, double ds, int32_t nsteps, int32_t scheme, const double* inflow,
                   double* w_inout, void* stream);

/* Richardson / pseudo-time solve of v + tau (M^V)^{-1} C^V v = g (PAPER.md:671-687,
 * SPEC.md:456-464, timeloop.pseudo_time_solve):
 *   res_i = g - v_i - tau M^-1 C v_i,  v_{i+1} = v_i + ds res_i,
 * stopping at the first i with ||res_i||_2 <= rho ||res_0||_2 (v_inout <- v_i,
 * *iters = i).  Returns HDGC_ENOCONV when i reaches max_iter first (v_inout =
 * v_max_iter).  The stopping test runs on the device (a fixed-order,
 * deterministic reduction of the residual norm raises a stop flag that the
 * iterations queued after it honour), so the host does not wait per
 * iteration: it queues iterations in chunks and checks the flag once per
 * chunk, one chunk behind.  Returns HDGC_EBLOWUP on a non-finite norm. */
int hdgc_richardson(hdgc_ctx* ctx, const double* u_loc, const double* g, const double* inflow, double tau,
                    double ds, double rho, int32_t max_iter, double* v_inout, int32_t* iters,
                    double* res0, double* res_final, void* stream);

/* Global H(div) space (fespace.FESpace Hdiv(k)): install the
 * element -> global dof map, host arrays element_dofs (NT, nb) and factors
 * (NT, nb) (u_loc[T,j] = factors[T,j] u_glob[element_dofs[T,j]]; every global
 * dof used by one or two (T, j), 0 <= dof < ndof < 2^31).  Copied to the device;
 * replaces a previous map.  2D contexts only. */
int hdgc_set_dofmap(hdgc_ctx* ctx, int64_t ndof, const int64_t* element_dofs, const double* factors);
/* u_loc = gather(u_glob), (NT, nb) from (ndof,) */
int hdgc_gather(hdgc_ctx* ctx, const double* u_glob, double* u_loc, void* stream);
/* r_glob[d] = sum over the (T, j) of d of factors[T,j] r_loc[T,j]: the global
 * I^T assembly, per dof in a fixed order (no atomics, bitwise reproducible) */
int hdgc_scatter(hdgc_ctx* ctx, const double* r_loc, double* r_glob, void* stream);
/* C^U u in global numbering: scatter(I^T C^V(I u_loc; I u_loc)), u_loc = gather(u_glob)
 * (the convection right-hand side of the Stokes solve). */
int hdgc_apply_u(hdgc_ctx* ctx, const double* u_glob, const double* inflow, double* r_glob, void* stream);

/* Transfer operators: direction 0: out = I in (BDM -> V_h),
 * direction 1: out = I^T in (V_h functionals -> BDM-test layout). */
int hdgc_transfer(hdgc_ctx* ctx, int32_t direction, const double* in, double* out, void* stream);

/* (M^V)^{-1} diagonal scale per element, out (NT,) = 2/detJ;
 * on a curved element (hdgc_set_curved) the entry is -(slot + 1), its
 * (M^V)^{-1} being the full block minv_blocks[slot]. */
int hdgc_mass_inverse(hdgc_ctx* ctx, double* out, void* stream);

/* Curved elements (mesh2d.curve_boundary, MESH:555-615):
 * install, once per 2D context, the n elements carrying an isoparametric map
 * (ascending ids, HOST arrays, copied):
 *   minv_blocks (n, nbs, nbs)  inverse V_h mass blocks, M_T = int D_m D_n detJ
 *                              (same block for both components);
 *   itrans      (n, nb, nb)    I_T, the element L2 projection BDM -> V_h
 *                              (rows c*nbs+m, columns BDM members); I^T = I_T^T;
 *   piola       (n, nqv, 4)    J/detJ at the volume points (max_speed).
 * The convection apply itself is unchanged (geometry-free reference form, exact
 * with Piola velocities and pulled-back test functions); substeps, propagate
 * and richardson apply the block inverse, transfer / apply_w / apply_u use I_T,
 * max_speed the per-point Piola factor.  2D only (HDGC_EUNSUP in 3D). */
int hdgc_set_curved(hdgc_ctx* ctx, int32_t n, const int32_t* elems, const double* minv_blocks,
                    const double* itrans, const double* piola);

/* max over elements x volume points of |J u_hat / detJ| into *out_dev (device
 * double), for the substep size dt = 0.1 h / (k^2 max|u|) (BASELINE cfg2). */
int hdgc_max_speed(hdgc_ctx* ctx, const double* u_loc, double* out_dev, void* stream);

/* End-to-end variants on HOST buffers: H2D of the inputs, compute, D2H of
 * the result, all on `stream`, synchronised before return. */
int hdgc_apply_v_host(hdgc_ctx* ctx, const double* u_loc, const double* w, const double* inflow,
                      double* r, void* stream);
int hdgc_substeps_host(hdgc_ctx* ctx, const double* u_loc, double* w_inout, const double* inflow,
                       double dt, int32_t nsteps, void* stream);

/* Norm-blowup guard: every update kernel (substeps, propagate,
 * richardson) sets a context flag when it writes a non-finite value.  This
 * call synchronises `stream`, and returns HDGC_EBLOWUP (clearing the flag) if
 * any update since the last check blew up, else HDGC_OK.  hdgc_substeps_host
 * runs it before returning; hdgc_richardson returns HDGC_EBLOWUP on a
 * non-finite residual norm. */
int hdgc_check_finite(hdgc_ctx* ctx, void* stream);

const char* hdgc_last_error(void);
const char* hdgc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HDGCONV_H */
