// Probe: TMA tile::gather4 of four 512-byte rows of a 2D f32 tensor into
// shared memory (diagnostic for a TMA producer in the fused backward).
// Usage: gather4_probe <box_rows>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int r0, int r1, int r2, int r3) {
  __shared__ __align__(128) float buf[4 * 128];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4 * 512) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"((unsigned)__cvta_generic_to_shared(buf)),
        "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
        : "memory");
  }
  unsigned ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(b) : "memory");
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int box_rows = argc > 1 ? atoi(argv[1]) : 1;
  const int R = 1000, C = 256;  // tensor: R rows x C cols f32, box 128 cols
  float* h = (float*)malloc(R * C * 4);
  for (int i = 0; i < R * C; ++i) h[i] = (float)i;
  float *d, *out;
  cudaMalloc(&d, R * C * 4);
  cudaMalloc(&out, 512 * 4);
  cudaMemcpy(d, h, R * C * 4, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode(box_rows=%d) = %d\n", box_rows, (int)cr);
  if (cr != CUDA_SUCCESS) return 1;
  const int rows[4] = {7, 999, 3, 7};
  probe<<<1, 128>>>(map, out, rows[0], rows[1], rows[2], rows[3]);
  cudaError_t e = cudaDeviceSynchronize();
  float r[512];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int k = 0; k < 4; ++k)
    for (int j = 0; j < 128; ++j)
      if (r[k * 128 + j] != (float)(rows[k] * C + j)) ++bad;
  printf("kernel: %s, mismatches %d (r[0]=%g r[128]=%g)\n", cudaGetErrorString(e), bad, r[0], r[128]);
  return e != cudaSuccess || bad;
}
