// L2 residency probe (development tool): random 512-byte row gathers from a
// working set of S bytes, rows either contiguous or strided (as a table's
// column slice of the (B, sum D) upstream gradient), with and without a
// concurrent stream of unique 1 KB read+write traffic (the weight rows).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gather(const float4* __restrict__ base, long rows, long stride_vec, int iters,
                       float4* __restrict__ sink, const float4* __restrict__ stream_src,
                       float4* __restrict__ stream_dst, long stream_rows, unsigned seed) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  unsigned x = seed ^ (unsigned)(warp * 2654435761u);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const long r = (long)(x % (unsigned)rows);
    float4 v = __ldcg(base + r * stride_vec + lane);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    if (stream_src && (i % 2 == 0)) {  // ~1 KB unique traffic per 2.4 gathers
      const long s = (warp * (long)iters + i) % stream_rows;
      float4 w = __ldcs(stream_src + s * 32 + lane);
      w.x += 1.f;
      __stcs(stream_dst + s * 32 + lane, w);
    }
  }
  if (acc.x == 12345.f) sink[0] = acc;
}

// same access pattern, rows staged with cp.async.cg into a per-warp smem ring
__global__ void gather_cpasync(const float4* __restrict__ base, long rows, long stride_vec, int iters,
                               float4* __restrict__ sink, const float4* __restrict__ stream_src,
                               float4* __restrict__ stream_dst, long stream_rows, unsigned seed) {
  __shared__ float4 ring[8][8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  unsigned x = seed ^ (unsigned)(warp * 2654435761u);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters + 7; ++i) {
    if (i < iters) {
      x = x * 1664525u + 1013904223u;
      const long r = (long)(x % (unsigned)rows);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&ring[w][i & 7][lane]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(base + r * stride_vec + lane));
      if (stream_src && (i % 2 == 0)) {
        const long s = (warp * (long)iters + i) % stream_rows;
        float4 v = __ldcs(stream_src + s * 32 + lane);
        v.x += 1.f;
        __stcs(stream_dst + s * 32 + lane, v);
      }
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 7;");
    if (i >= 7) {
      float4 v = ring[w][(i - 7) & 7][lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x == 12345.f) sink[0] = acc;
}

int main() {
  const long big = 4L << 30;  // 4 GB stream buffers
  float4 *base, *sink, *ss, *sd;
  cudaMalloc(&base, 8L << 30);
  cudaMalloc(&sink, 64);
  cudaMalloc(&ss, big);
  cudaMalloc(&sd, big);
  cudaMemset(base, 0, 8L << 30);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 8, threads = 256, iters = 400;
  const long gathers = (long)blocks * threads / 32 * iters;
  printf("working_set_MB stride_bytes stream GB/s(gather bytes) \n");
  for (int mode = 0; mode < 2; ++mode)
  for (int withstream = 0; withstream < 2; ++withstream)
    for (long mb : {16L, 32L, 64L, 128L}) {
      for (long stride_bytes : {32768L}) {
        const long rows = (mb << 20) / 512;
        const long sv = stride_bytes / 16;
        if (rows * stride_bytes > (8L << 30)) continue;
        auto k = mode ? gather_cpasync : gather;
        k<<<blocks, threads>>>(base, rows, sv, iters, sink, withstream ? ss : nullptr, sd, big / 512, 1);
        cudaEventRecord(a);
        k<<<blocks, threads>>>(base, rows, sv, iters, sink, withstream ? ss : nullptr, sd, big / 512, 7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s %6ld %6ld %d %8.1f\n", mode ? "cpasync" : "ldg    ", mb, stride_bytes, withstream, gathers * 512.0 / (ms * 1e-3) / 1e9);
      }
    }
  return 0;
}
