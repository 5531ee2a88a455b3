// FP64 ceiling microbenchmarks for B200 (sm_100a): DFMA (SIMT) and DMMA (mma.sync m8n8k4 f64).
// MEASURED_PEAKS.json carries no FP64 figure, so the roofline
// denominator for polya_schur is measured here.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int TILES>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[TILES][2];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  // DFMA: 8 chains x 4 warps-per-scheduler worth of threads
  for (int bpsm : {2, 4, 8}) {
    int iters = 20000; int threads = 256; int blocks = sms * bpsm;
    dfma_kernel<8><<<blocks, threads>>>(out, 100, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf(", \"dfma_tflops_bpsm%d\": %.3f", bpsm, flops / (best * 1e-3) / 1e12);
  }
  for (int wpsm : {4, 8, 16}) {
    int iters = 20000; int threads = 128; int blocks = sms * wpsm / 4;
    dmma_kernel<4><<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); dmma_kernel<4><<<blocks, threads>>>(out, iters);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256 * 4 * (double)iters * (threads / 32) * blocks;
    printf(", \"dmma_tflops_wpsm%d\": %.3f", wpsm, flops / (best * 1e-3) / 1e12);
  }
  // long sustained DMMA run (~2 s) for the clock-under-load figure
  {
    int iters = 400000; int threads = 128; int blocks = sms * 2;
    CK(cudaEventRecord(e0)); dmma_kernel<4><<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 256 * 4 * (double)iters * (threads / 32) * blocks;
    printf(", \"dmma_tflops_sustained\": %.3f, \"dmma_sustained_ms\": %.1f", flops / (ms * 1e-3) / 1e12, ms);
  }
  {
    int iters = 400000; int threads = 256; int blocks = sms * 4;
    CK(cudaEventRecord(e0)); dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf(", \"dfma_tflops_sustained\": %.3f, \"dfma_sustained_ms\": %.1f", flops / (ms * 1e-3) / 1e12, ms);
  }
  printf("}\n");
  return 0;
}
