// tma_gather_probe2.cu -- K4 v26's producer pattern on its own: 32 lanes each issue one tile::gather4
// (operand, k-half, k-pair, row pair) into one 8 KB stage; the stage is checked against stage_byte().
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__host__ __device__ constexpr int stage_byte(int t, int x, int y) {
  return 2048 * (t >> 2) + 512 * (x >> 1) + 128 * (t & 3) + 64 * (x & 1) + 16 * ((y >> 1) ^ (t & 3)) + 8 * (y & 1);
}
__device__ __forceinline__ unsigned sptr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, double* out, int np, int off, int single) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sptr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sptr(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sptr(&bar[0])), "r"(single >= 0 ? 0 : 4096));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sptr(&bar[1])), "r"(single >= 0 ? 0 : 4096));
    }
    __syncwarp();
    const int op = lane >> 4, thalf = (lane >> 3) & 1, t0 = 4 * thalf + 2 * ((lane >> 2) & 1), pr = lane & 3;
    // operand op, k-term t: matrix 2 t + op, rows 8..15 of it (chunk 1), columns 8..15
    const int ra = (2 * t0 + op) * np + 8 + 2 * pr, rb = (2 * (t0 + 1) + op) * np + 8 + 2 * pr;
    const unsigned dst = sptr(sm) + off + op * 4096 + (2048 * (t0 >> 2) + 512 * pr + 128 * (t0 & 3));
    if (single >= 0 && lane != single) return;
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
        "l"(&tmap), "r"(8), "r"(ra), "r"(ra + 1), "r"(rb), "r"(rb + 1), "r"(sptr(&bar[thalf]))
        : "memory");
  }
  if (single >= 0) { __syncthreads(); if (threadIdx.x == 0) { unsigned ns = 0; for (int i = 0; i < 1000000; ++i) ns += i; if (ns == 7) out[0] = ns; } return; }
  for (int b = 0; b < 2; ++b)
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(sptr(&bar[b])) : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<double*>(sm + off)[i];
}

int main(int argc, char** argv) {
  const int np = 16, nm = 16;
  std::vector<double> h((size_t)nm * np * np);
  for (int m = 0; m < nm; ++m)
    for (int r = 0; r < np; ++r)
      for (int c = 0; c < np; ++c) h[((size_t)m * np + r) * np + c] = m * 10000 + r * 100 + c;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 1024 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)np, (cuuint64_t)nm * np};
  cuuint64_t strides[1] = {(cuuint64_t)np * 8};
  cuuint32_t box[2] = {8, 1}, es[2] = {1, 1};
  CUresult r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  int rc = 0;
  for (int l = 0; l < 32; ++l) {
    probe<<<1, 160, 20480>>>(tm, o, np, 0, l);
    cudaError_t e = cudaDeviceSynchronize();
    const int op = l >> 4, thalf = (l >> 3) & 1, t0 = 4 * thalf + 2 * ((l >> 2) & 1), pr = l & 3;
    printf("lane %2d dst %5d: %s\n", l, op * 4096 + (2048 * (t0 >> 2) + 512 * pr + 128 * (t0 & 3)), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  for (int off : {0, 8192}) {
    cudaMemset(o, 0xff, 1024 * 8);
    probe<<<1, 160, 20480>>>(tm, o, np, off, -1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("off %d kernel: %s\n", off, cudaGetErrorString(e)); return 1; }
    std::vector<double> ho(1024);
    cudaMemcpy(ho.data(), o, 1024 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int op = 0; op < 2; ++op)
      for (int t = 0; t < 8; ++t)
        for (int x = 0; x < 8; ++x)
          for (int y = 0; y < 8; ++y) {
            const double want = (2 * t + op) * 10000 + (8 + x) * 100 + 8 + y;
            if (ho[(op * 4096 + stage_byte(t, x, y)) / 8] != want) ++bad;
          }
    printf("off %d: %s (%d mismatches)\n", off, bad ? "FAIL" : "PASS", bad);
    rc |= bad != 0;
  }
  return rc;
}
