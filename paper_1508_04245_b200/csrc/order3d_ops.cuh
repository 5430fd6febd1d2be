// order3d_ops.cuh — per-order launchers of the 3D kernels (included by order3d_k<K>.cu).
#pragma once
#include "context.cuh"
#include "conv3d.cuh"

namespace hdgc {

static inline unsigned grid3_for(long long work, int threads) { return (unsigned)((work + threads - 1) / threads); }

template <int K>
int launch3_prep(hdgc_ctx* c, const double* u, cudaStream_t st) {
  Prep3Params p;
  p.tab = c->d_tab;
  p.u = u;
  p.sgn = c->d_sign;
  p.prep = c->d_prep;
  p.nt = c->nt;
  prep3d_kernel<K><<<grid3_for(c->nt, 128), 128, 0, st>>>(p);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

template <int K>
int launch3_main(hdgc_ctx* c, int mode, const double* w, const double* inflow, double* out, double dt,
                 cudaStream_t st) {
  Conv3Params p;
  p.tab = c->d_tab;
  p.prep = c->d_prep;
  p.w = w;
  p.inflow = inflow;
  p.code = c->d_code;
  p.minv = c->d_minv;
  p.out = out;
  p.dt = dt;
  p.nt = c->nt;
  const unsigned blocks = grid3_for(c->nt, Dims3<K>::EPB);
  if (mode == MODE_SUBSTEP) conv3d_kernel<K, MODE_SUBSTEP><<<blocks, Dims3<K>::THREADS, 0, st>>>(p);
  else conv3d_kernel<K, MODE_APPLY><<<blocks, Dims3<K>::THREADS, 0, st>>>(p);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

template <int K>
int launch3_transfer(hdgc_ctx* c, int dir, const double* in, double* out, cudaStream_t st) {
  const long long work = (long long)c->nt * Dims3<K>::NB;
  if (dir == 0) transfer3d_kernel<K, false><<<grid3_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, in, out);
  else transfer3d_kernel<K, true><<<grid3_for(work, 256), 256, 0, st>>>(c->d_tab, c->d_piola, c->nt, in, out);
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

template <int K>
int launch3_maxspeed(hdgc_ctx* c, const double* u, double* out, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
  maxspeed3d_kernel<K><<<grid3_for(c->nt, 128), 128, 0, st>>>(c->d_tab, c->d_piola, c->nt, u,
                                                             reinterpret_cast<unsigned long long*>(out));
  CUDA_TRY(cudaGetLastError());
  return HDGC_OK;
}

}  // namespace hdgc

#define HDGC_INSTANTIATE_ORDER3(K)                                                                  \
  namespace hdgc {                                                                                  \
  template int launch3_prep<K>(hdgc_ctx*, const double*, cudaStream_t);                             \
  template int launch3_main<K>(hdgc_ctx*, int, const double*, const double*, double*, double, cudaStream_t); \
  template int launch3_transfer<K>(hdgc_ctx*, int, const double*, double*, cudaStream_t);           \
  template int launch3_maxspeed<K>(hdgc_ctx*, const double*, double*, cudaStream_t);                \
  }
