// Shared compile-time dimensions and parameter blocks for the 2D
// convection kernels (sm_100a, fp64).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hdgc {

// Per-order constants.  The volume rule is quad_triangle(3k-1) (exact for the
// degree 3k-1 volume integrand), the facet rule quad_interval(3k+1) (pinned,
// SPEC.md:157); see basis.volume_rule / basis.facet_rule.
template <int K>
struct Dims {
  static constexpr int NE = K + 1;                       // Legendre modes per edge
  static constexpr int NBS = (K + 1) * (K + 2) / 2;      // scalar P_k
  static constexpr int NB = 2 * NBS;                     // [P_k]^2 = BDM_k
  static constexpr int NBS1 = K * (K + 1) / 2;           // scalar P_{k-1} (divergence space)
  static constexpr int NQV = K == 1 ? 3 : (K == 2 ? 7 : ((3 * K + 1) / 2) * ((3 * K + 1) / 2));
  static constexpr int NF = (3 * K + 3) / 2;
  // table offsets (doubles) in the packed device table
  static constexpr int OFF_COEF = 0;
  static constexpr int OFF_DIVM = OFF_COEF + NB * NB;
  static constexpr int OFF_VW = OFF_DIVM + NBS1 * NB;
  static constexpr int OFF_VD = OFF_VW + NQV;
  static constexpr int OFF_VG = OFF_VD + NQV * NBS;
  static constexpr int OFF_FW = OFF_VG + NQV * NBS * 2;
  static constexpr int OFF_FL = OFF_FW + NF;
  static constexpr int OFF_FD = OFF_FL + NF * NE;
  static constexpr int OFF_FLEN = OFF_FD + 3 * NF * NBS;
  static constexpr int TAB = OFF_FLEN + 4;               // padded to keep 16-B alignment
};

inline int dims_nqv(int k) {
  return k == 1 ? 3 : (k == 2 ? 7 : ((3 * k + 1) / 2) * ((3 * k + 1) / 2));
}
inline int dims_nf(int k) { return (3 * k + 3) / 2; }
inline int dims_nbs(int k) { return (k + 1) * (k + 2) / 2; }
inline int dims_tab(int k) {
  const int nbs = dims_nbs(k), nb = 2 * nbs, nqv = dims_nqv(k), nf = dims_nf(k);
  return nb * nb + (k * (k + 1) / 2) * nb + nqv + nqv * nbs + nqv * nbs * 2 + nf + nf * (k + 1) + 3 * nf * nbs + 4;
}

// Output modes of the element kernel.
enum : int {
  MODE_APPLY = 0,    // r = C^V(u; w)
  MODE_SUBSTEP = 1,  // w_out = w + c (2/detJ) C^V(u; w)  (forward Euler: c = -dt)
  MODE_APPLY_IT = 2, // r_w = I^T C^V(u; w)
  MODE_STAGE = 3,    // w_out = a w + b x + c (2/detJ) C^V(u; w), optional residual norms (StageParams)
};

// Epilogues of the update modes:
//   MODE_SUBSTEP: out = w + c minv r          (forward Euler / Heun stage 1: c = -dt)
//   MODE_STAGE:   out = a w + b x + c minv r,
//                 res = x - w - tau minv r, rn[T * dim + comp] = sum_m res^2 (rn optional)
// Heun's second stage: a = b = 1/2, c = -dt/2, x = w^n; Richardson
// (PAPER.md:679-685): a = 1 - ds, b = ds, c = -ds tau, x = g*.
// Curved elements (hdgc_set_curved): their mass is a full block, flagged by a
// negative minv[T] = -(slot + 1).  The update kernels then store the raw
// residual row into cres[slot] and curved_fixup_kernel applies the block
// inverse afterwards (the kernels' own output for those rows is overwritten).
// Norm-blowup guard ("instability shows as norm blowup caught by
// a guard"): the update epilogues sum their output row and set *flag when the
// sum is not finite (one DADD per output value; the atomic only fires on a
// blow-up).  hdgc_check_finite reads and clears the flag.
struct StageParams {
  const double* __restrict__ x = nullptr;
  double* __restrict__ rn = nullptr;
  double* __restrict__ cres = nullptr;   // (n_curved, NB) raw residual rows of curved elements
  int* __restrict__ flag = nullptr;      // blow-up flag (context-owned), set on non-finite output
  // device-side Richardson stop (hdgc_richardson): when *stop != 0 the update
  // kernel returns at entry without touching its output (the iteration has
  // converged on the device; later queued iterations are no-ops)
  const int* stop = nullptr;
  // sum-factorised kernels (no curved elements): per-CTA residual partials
  // (rich_cta_partial) instead of per-(element, component) sums into rn
  double* rpart = nullptr;
  double a = 1.0, b = 0.0, c = 0.0, tau = 0.0;
};

// Richardson residual norm, part 1 (sum-factorised STAGE kernels): one whole
// warp of every CTA sums its lanes' squared residuals in a fixed xor-tree
// order and stores the CTA partial; richardson_final_kernel (launched with PDL
// right after) adds the partials in index order and takes the stop decision.
__device__ __forceinline__ double warp_sum_fixed(double a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}
__device__ __forceinline__ void rich_cta_partial(const StageParams& st, double acc, int slot) {
  acc = warp_sum_fixed(acc);
  if ((threadIdx.x & 31) == 0) st.rpart[slot] = acc;
}

__device__ __forceinline__ bool stage_stopped(const StageParams& st) {
  if (st.stop == nullptr) return false;
  int v;
  asm volatile("ld.global.relaxed.gpu.b32 %0, [%1];\n" : "=r"(v) : "l"(st.stop) : "memory");
  return v != 0;
}
// the same flag as a plain L2 load the compiler may schedule early and consume
// late (call after griddepcontrol.wait: the flag is the previous kernel's output)
__device__ __forceinline__ int stage_stop_flag(const StageParams& st) { return st.stop ? __ldcg(st.stop) : 0; }

__device__ __forceinline__ void guard_finite(int* flag, double rowsum) {
  if (flag != nullptr && !isfinite(rowsum)) atomicOr(flag, 1);
}

// Per-element neighbour code: >= 0: (neighbour element << 2) | neighbour local
// edge; < 0: boundary facet, slot = -1 - code (row of the inflow array).
struct ElemParams {
  const double* __restrict__ tab;     // packed reference tables (Dims<K> layout)
  const double* __restrict__ u;       // (NT, NB) BDM coefficients
  const double* __restrict__ w;       // (NT, NB) V_h coefficients
  const double* __restrict__ inflow;  // (NBF, NF, 2) or nullptr
  const int32_t* __restrict__ code;   // (NT, 3)
  const double* __restrict__ piola;   // (4, NT) SoA: J/detJ row-major (00, 01, 10, 11)
  const double* __restrict__ minv;    // (NT,) 2/detJ
  const double* __restrict__ prep = nullptr;   // frozen-velocity rows (prep_thread2d_kernel) or nullptr
  double* __restrict__ out;           // (NT, NB)
  StageParams st;
  int nt;
};

// FP64 tensor-core MMA (SASS DMMA), D (8x8) += A (8x4, row) B (4x8, col).
// Fragments (lane l): a = A[l/4][l%4], b = B[l%4][l/4], d0/d1 = D[l/4][2(l%4) + 0/1].
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Host side: A fragments of an (nr x nb) row-major matrix M for dmma_m8n8k4,
// tile (mt, ks) lane l at [(mt * ks_n + ks) * 32 + l] = M[8 mt + l/4][4 ks + l%4]
// (zero-padded to 8-row / 4-column multiples).
inline void dmma_a_fragments(const double* M, int nr, int nb, double* out) {
  const int mt_n = (nr + 7) / 8, ks_n = (nb + 3) / 4;
  for (int mt = 0; mt < mt_n; ++mt)
    for (int ks = 0; ks < ks_n; ++ks)
      for (int l = 0; l < 32; ++l) {
        const int i = mt * 8 + l / 4, j = ks * 4 + l % 4;
        out[(mt * ks_n + ks) * 32 + l] = (i < nr && j < nb) ? M[(size_t)i * nb + j] : 0.0;
      }
}

// --- TMA bulk copies + mbarrier (sm_90+ PTX; SASS UBLKCP / SYNCS)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// L2 prefetch of a contiguous global range (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// HDGC_DEBUG builds (tools/debug_check.py; compute-sanitizer is not available
// on the GPU pool): every kernel with dynamic shared memory starts with
// hdgc_debug_prologue, which (1) poisons the whole dynamic smem with NaN, so a
// read of smem nobody wrote turns the output non-finite, and (2) delays the
// CTA and then each warp by a pseudo-random amount, which reshuffles the CTA
// schedule and skews the warps of a CTA against each other, so a missing
// barrier / mbarrier / PDL wait shows up as output that differs from the
// release build.  HDGC_ASSERT bounds-checks neighbour / slot indices (device
// assert: the kernel traps, the host sees a CUDA error).  Release builds: no-ops.
#ifdef HDGC_DEBUG
#include <cassert>
#define HDGC_ASSERT(x) assert(x)
__device__ __forceinline__ unsigned hdgc_hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ void hdgc_debug_prologue(double* smem, int n_doubles) {
  for (int i = threadIdx.x; i < n_doubles; i += blockDim.x) smem[i] = __longlong_as_double(0x7ff8dead0000beefLL);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // before any TMA writes the same smem
  __syncthreads();
  __nanosleep(hdgc_hash(blockIdx.x * 2654435761u + 17u) % 4000u);
  __nanosleep(hdgc_hash(blockIdx.x * 40503u + (threadIdx.x >> 5) * 977u + 3u) % 3000u);
}
#else
#define HDGC_ASSERT(x) ((void)0)
__device__ __forceinline__ void hdgc_debug_prologue(double*, int) {}
#endif

// Programmatic dependent launch (PDL) between consecutive update kernels of a
// substep batch (hdgc_substeps): kernel s+1 is launched with the
// programmatic-stream-serialisation attribute, so its CTAs start while kernel
// s drains its last wave, stage everything that does not depend on w (prep
// tile, facet tables, neighbour codes, frozen-velocity work) and block in
// pdl_wait() until kernel s has completed and its writes are visible.  Both
// instructions are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Host side: launch kern<<<grid, block, smem, st>>>(p), with the PDL attribute
// when pdl is set (the caller guarantees the previous kernel on st is an
// update kernel of the same batch and nothing before pdl_wait() reads what it
// writes).
template <class... P, class... A>
inline cudaError_t launch_maybe_pdl(void (*kern)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                                    bool pdl, const A&... p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, p...);
}

}  // namespace hdgc
