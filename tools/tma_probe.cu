// tma_probe.cu -- checks the shared-memory layout of a 3-D TMA load (box 8 x 8 x 1 of FP64, SWIZZLE_64B)
// at 128-byte-aligned destinations that are not 512-byte aligned: K4 v25 relies on the 16-byte chunk
// index being XORed with bits 7-8 of the ABSOLUTE shared address (so tiles at 640-byte strides get
// different XOR phases).  Prints the observed chunk permutation per tile and row and checks it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ unsigned sptr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, double* out, int ntiles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sptr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sptr(&bar)), "r"(ntiles * 512));
    for (int t = 0; t < ntiles; ++t) {
      // tile t: matrix t, rows 8..15, cols 16..23
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
              sptr(sm + 640 * t)),
          "l"(&tmap), "r"(16), "r"(8), "r"(t), "r"(sptr(&bar))
          : "memory");
    }
  }
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(sptr(&bar)) : "memory");
  for (int i = threadIdx.x; i < ntiles * 80; i += blockDim.x) out[i] = reinterpret_cast<double*>(sm)[i];
}

int main() {
  const int np = 32, nm = 4;
  std::vector<double> h((size_t)nm * np * np);
  for (int m = 0; m < nm; ++m)
    for (int r = 0; r < np; ++r)
      for (int c = 0; c < np; ++c) h[((size_t)m * np + r) * np + c] = m * 10000 + r * 100 + c;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, nm * 80 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(o, 0, nm * 80 * 8);
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) { printf("no entry point\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)np, (cuuint64_t)np, (cuuint64_t)nm};
  cuuint64_t strides[2] = {(cuuint64_t)np * 8, (cuuint64_t)np * np * 8};
  cuuint32_t box[3] = {8, 8, 1}, es[3] = {1, 1, 1};
  CUresult r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  probe<<<1, 128, 8192>>>(tm, o, nm);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<double> ho(nm * 80);
  cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int t = 0; t < nm; ++t) {
    for (int x = 0; x < 8; ++x) {
      printf("tile %d row %d:", t, x);
      for (int y = 0; y < 8; ++y) {
        // predicted position: byte 640 t + 64 x + 8 y with chunk (bits 4-5) ^= bits 7-8 of the address
        const unsigned lin = 640 * t + 64 * x + 8 * y;
        const unsigned sw = lin ^ (((lin >> 7) & 3) << 4);
        const double want = t * 10000 + (8 + x) * 100 + (16 + y);
        const double got = ho[sw / 8];
        printf(" %s", got == want ? "ok" : "XX");
        bad += got != want;
      }
      printf("\n");
    }
  }
  printf("%s (%d mismatches)\n", bad ? "FAIL" : "PASS: swizzle = chunk ^ address bits 7-8", bad);
  if (bad)   // where each element actually landed (double index within the tile's 640-byte slot)
    for (int t = 0; t < nm; ++t)
      for (int x = 0; x < 8; ++x) {
        printf("tile %d row %d at:", t, x);
        for (int y = 0; y < 8; ++y) {
          const double want = t * 10000 + (8 + x) * 100 + (16 + y);
          int at = -1;
          for (int i = 0; i < nm * 80; ++i) if (ho[i] == want) at = i;
          printf(" %d", at - 80 * t);
        }
        printf("\n");
      }
  return bad != 0;
}
