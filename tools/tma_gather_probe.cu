// tma_gather_probe.cu -- checks TMA tile::gather4 on sm_100a for K4's stage layout: a 2-D tensor map
// over the arena viewed as [nmats*np rows][np columns] FP64, box 8 columns x 1 row, 64-byte swizzle;
// one gather4 brings 4 arbitrary rows (two rows of two k-terms) = 256 bytes into shared memory at a
// 128-byte-aligned address, the 16-byte chunk index XORed with address bits 7-8.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ unsigned sptr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, double* out, int np) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sptr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sptr(&bar)), "r"(4 * 256));
    for (int q = 0; q < 4; ++q) {
      // gather q: matrix q rows 2, 3 and matrix q+1 rows 2, 3 (columns 8..15), into sm + 128 q + 512 (q>>1)... simple: 256 q
      const int r0 = q * np + 2, r1 = q * np + 3, r2 = (q + 1) * np + 2, r3 = (q + 1) * np + 3;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(
              sptr(sm + 256 * q + 128 * (q >= 2 ? 4 : 0))),
          "l"(&tmap), "r"(8), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sptr(&bar))
          : "memory");
    }
  }
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(sptr(&bar)) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = reinterpret_cast<double*>(sm)[i];
}

int main() {
  const int np = 16, nm = 6;
  std::vector<double> h((size_t)nm * np * np);
  for (int m = 0; m < nm; ++m)
    for (int r = 0; r < np; ++r)
      for (int c = 0; c < np; ++c) h[((size_t)m * np + r) * np + c] = m * 10000 + r * 100 + c;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 256 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(o, 0xff, 256 * 8);
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
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096);
  probe<<<1, 128, 4096>>>(tm, o, np);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<double> ho(256);
  cudaMemcpy(ho.data(), o, 256 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int qq = 0; qq < 4; ++qq)
    for (int rr = 0; rr < 4; ++rr)
      for (int y = 0; y < 8; ++y) {
        const int m = qq + (rr >> 1), row = 2 + (rr & 1);
        const double want = m * 10000 + row * 100 + 8 + y;
        const unsigned lin = 256 * qq + 128 * (qq >= 2 ? 4 : 0) + 64 * rr + 8 * y;
        const unsigned sw = lin ^ (((lin >> 7) & 3) << 4);
        if (sw / 8 >= 256 || ho[sw / 8] != want) ++bad;
      }
  printf("%s (%d mismatches)\n", bad ? "FAIL" : "PASS: gather4 rows at 64-byte pitch, chunk ^ address bits 7-8", bad);
  if (bad)
    for (int i = 0; i < 256; ++i) printf("%d:%g%s", i, ho[i], i % 8 == 7 ? "\n" : " ");
  return bad != 0;
}
