// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA-core) and DMMA
// (warp-level mma.sync f64 tensor-core shapes). Prints one JSON object.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C 2 regs
template <int CH>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 1;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

// Do DMMA and DFMA share one FP64 pipe?  Even warps run m8n8k4 DMMA chains,
// odd warps DFMA chains (8x the iterations: 512 vs 64 flops per warp
// instruction); the combined rate tells whether the two overlap.
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  double s = 0;
  if (((threadIdx.x >> 5) & 1) == 0) {
    double av = threadIdx.x * 1e-3, bv = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < 8 * iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
  }
  if (s == 1234.5) out[0] = s;
}

template <typename F>
static float time_it(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d", p.name, sms);
  const int threads = 256;
  for (int occ : {4, 8}) {
    int blocks = sms * occ;
    int iters = 20000;
    float ms = time_it([&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_occ%d_tflops\": %.3f", occ, flops / ms / 1e9);
  }
  {
    int blocks = sms * 8; int iters = 4000;
    float ms = time_it([&] { dmma_m8n8k4<8><<<blocks, threads>>>(out, iters); }, 5);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * blocks * (threads / 32);
    printf(", \"dmma_m8n8k4_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    int blocks = sms * 8; int iters = 2000;
    float ms = time_it([&] { dmma_m16n8k4<8><<<blocks, threads>>>(out, iters); }, 5);
    double flops = 2.0 * 16 * 8 * 4 * 8.0 * iters * blocks * (threads / 32);
    printf(", \"dmma_m16n8k4_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    int blocks = sms * 8; int iters = 1000;
    float ms = time_it([&] { dmma_m16n8k8<8><<<blocks, threads>>>(out, iters); }, 5);
    double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * blocks * (threads / 32);
    printf(", \"dmma_m16n8k8_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    int blocks = sms * 8; int iters = 2000;
    float ms = time_it([&] { mixed_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    // half the warps: 8 DMMA x 512 flops per iteration; the other half: 8 x 8 DFMA x 64 flops
    const double warps = (double)blocks * (threads / 32) / 2;
    double flops = warps * iters * 8 * 512.0 + warps * 8.0 * iters * 8 * 64.0;
    printf(", \"mixed_dmma_dfma_tflops\": %.3f", flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
