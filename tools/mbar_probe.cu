// Probe: which mbarrier + cp.async completion patterns run on this sm_100a
// part (diagnostic for the warp-specialised backward).  Usage: mbar_probe <mode>
//   0: cp.async.mbarrier.arrive (inc) + mbarrier.arrive, count 32
//   1: cp.async.mbarrier.arrive.noinc only, count 32
//   2: cp.async.wait_all + mbarrier.arrive, count 32
//   3: mode 0 with the try_wait loop in the producer on an `empty` barrier
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const float4* src, float* out, int mode, int rounds, int off, int small) {
  extern __shared__ __align__(16) unsigned char dyn[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(dyn);
  float4 (*buf)[32] = reinterpret_cast<float4 (*)[32]>(dyn + off);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[i])), "r"(32) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[2 + i])), "r"(1) : "memory");
    }
  }
  __syncthreads();
  if (warp == 1) {  // producer
    unsigned ph = 1;
    for (int r = 0; r < rounds; ++r) {
      const int s = r & 1;
      if (mode == 3 || r >= 2) {
        unsigned ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(ok) : "r"(sa(&bar[2 + s])), "r"(ph) : "memory");
      }
      if (small)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa(&buf[s][lane])), "l"(src + r * 32 + lane));
      else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(&buf[s][lane])), "l"(src + r * 32 + lane));
      if (mode == 0 || mode == 3) {
        asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(sa(&bar[s])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[s])) : "memory");
      } else if (mode == 1) {
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&bar[s])) : "memory");
      } else {
        asm volatile("cp.async.wait_all;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[s])) : "memory");
      }
      if (s == 1) ph ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 0) {  // consumer
    unsigned ph = 0;
    float acc = 0.f;
    for (int r = 0; r < rounds; ++r) {
      const int s = r & 1;
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
      acc += buf[s][lane].x;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[2 + s])) : "memory");
      if (s == 1) ph ^= 1;
    }
    out[lane] = acc;
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int off = argc > 2 ? atoi(argv[2]) : 64;
  const int small = argc > 3 ? atoi(argv[3]) : 0;
  const int smem = 220 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 64;
  float4* src;
  float* out;
  cudaMalloc(&src, rounds * 32 * sizeof(float4));
  cudaMalloc(&out, 32 * sizeof(float));
  float4* h = (float4*)malloc(rounds * 32 * sizeof(float4));
  for (int i = 0; i < rounds * 32; ++i) h[i] = make_float4(1.f, 0.f, 0.f, 0.f);
  cudaMemcpy(src, h, rounds * 32 * sizeof(float4), cudaMemcpyHostToDevice);
  probe<<<1, 64, smem>>>(src, out, mode, rounds, off, small);
  cudaError_t e = cudaDeviceSynchronize();
  float r[32];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  printf("mode %d off %d small %d: %s acc=%g (want %d)\n", mode, off, small, cudaGetErrorString(e), r[0], rounds);
  return e != cudaSuccess;
}
