// L2 probe 2 (development tool): cp.async gathers of random 512-byte rows from
// a W-MB working set, interleaved (1 per `every` gathers) with a read-modify-
// write of a *unique* 512-byte row from a large array (the weight-row update
// of the TBE backward).  Variants: RMW via cp.async+st (kernel-like) or via
// ld.cs/st.cs (streaming).  Run under ncu for L2 hit rate and DRAM bytes.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

template <int RMW_MODE>
__global__ void probe(const float4* __restrict__ base, long rows, long stride_vec, int iters, int every,
                      float4* __restrict__ big, long big_rows, float4* __restrict__ sink) {
  __shared__ float4 ring[8][8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  unsigned x = 12345u ^ (unsigned)(warp * 2654435761u);
  float4 acc = make_float4(0, 0, 0, 0);
  long u = warp;  // unique-row cursor (interleaved across warps: sequential sweep)
  for (int i = 0; i < iters + 7; ++i) {
    if (i < iters) {
      x = x * 1664525u + 1013904223u;
      const long r = (long)(x % (unsigned)rows);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&ring[w][i & 7][lane]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(base + r * stride_vec + lane));
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 7;");
    if (i >= 7) {
      float4 v = ring[w][(i - 7) & 7][lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (RMW_MODE >= 0 && i % every == 0) {
      float4* p = big + (u % big_rows) * 32 + lane;
      u += nwarps;
      if (RMW_MODE == 0) {
        float4 v = *p;
        v.x += acc.x;
        *p = v;
      } else {
        float4 v = __ldcs(p);
        v.x += acc.x;
        __stcs(p, v);
      }
    }
  }
  if (acc.x == 12345.f) sink[0] = acc;
}

int main(int argc, char** argv) {
  const long mb = argc > 1 ? atol(argv[1]) : 16;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;  // -1 none, 0 normal RMW, 1 streaming RMW
  const int every = argc > 3 ? atoi(argv[3]) : 2;
  float4 *base, *big, *sink;
  cudaMalloc(&base, 4L << 30);
  cudaMalloc(&big, 8L << 30);
  cudaMalloc(&sink, 64);
  cudaMemset(base, 0, 4L << 30);
  cudaMemset(big, 0, 8L << 30);
  const long rows = (mb << 20) / 512, sv = 32768 / 16;
  const int blocks = 148 * 6, threads = 256, iters = 2000;
  auto k = mode < 0 ? probe<-1> : mode == 0 ? probe<0> : probe<1>;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<blocks, threads>>>(base, rows, sv, iters, every, big, (8L << 30) / 512, sink);
  cudaEventRecord(a);
  k<<<blocks, threads>>>(base, rows, sv, iters, every, big, (8L << 30) / 512, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double g = (double)blocks * threads / 32 * iters * 512;
  printf("ws %ld MB mode %d every %d: %.3f ms, gather %.0f GB/s\n", mb, mode, every, ms, g / (ms * 1e-3) / 1e9);
  return 0;
}
