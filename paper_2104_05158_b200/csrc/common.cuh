// Shared device helpers for libneob200 (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "neo_tbe.h"

namespace neo {

constexpr int kWarp = 32;

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// thread-local message for neo_last_error()
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// element conversion (all round-to-nearest-even)

template <typename T> struct Elem;
template <> struct Elem<float> {
  __device__ __forceinline__ static float to_f(float v) { return v; }
  __device__ __forceinline__ static double to_d(float v) { return v; }
  __device__ __forceinline__ static float from_f(float v) { return v; }
  __device__ __forceinline__ static float from_d(double v) { return __double2float_rn(v); }
};
template <> struct Elem<double> {
  __device__ __forceinline__ static float to_f(double v) { return __double2float_rn(v); }
  __device__ __forceinline__ static double to_d(double v) { return v; }
  __device__ __forceinline__ static double from_f(float v) { return v; }
  __device__ __forceinline__ static double from_d(double v) { return v; }
};
template <> struct Elem<__half> {
  __device__ __forceinline__ static float to_f(__half v) { return __half2float(v); }
  __device__ __forceinline__ static double to_d(__half v) { return __half2float(v); }
  __device__ __forceinline__ static __half from_f(float v) { return __float2half_rn(v); }
  __device__ __forceinline__ static __half from_d(double v) { return __double2half(v); }
};
template <> struct Elem<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static double to_d(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_d(double v) {
    return __float2bfloat16_rn(__double2float_rn(v));
  }
};

template <typename Acc, typename T>
__device__ __forceinline__ Acc to_acc(T v) {
  if constexpr (sizeof(Acc) == 8) return Elem<T>::to_d(v);
  else return Elem<T>::to_f(v);
}
template <typename T, typename Acc>
__device__ __forceinline__ T from_acc(Acc v) {
  if constexpr (sizeof(Acc) == 8) return Elem<T>::from_d(v);
  else return Elem<T>::from_f(v);
}

// 16-byte vector of VEC elements of T
template <typename T, int VEC>
struct alignas(sizeof(T) * VEC) Vec {
  T v[VEC];
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void record_bad_index(neo_error* err, int64_t pos) {
  if (err) atomicMin(reinterpret_cast<unsigned long long*>(&err->position),
                     static_cast<unsigned long long>(pos));
}

// resolves a recorded first-bad position into (value, table); no-op when clean
void launch_error_finalize(neo_error* err, const void* indices, int32_t index_dtype,
                           const int64_t* offsets, int64_t B, int32_t T, cudaStream_t s);

// generic vector load of VEC elements of T (2..32 bytes) from an aligned
// address through the read-only path
template <typename T, int VEC>
__device__ __forceinline__ Vec<T, VEC> ld_vec(const T* p) {
  constexpr int kBytes = sizeof(T) * VEC;
  Vec<T, VEC> r;
  if constexpr (kBytes == 32) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 a = __ldg(q), b = __ldg(q + 1);
    reinterpret_cast<uint4*>(&r)[0] = a;
    reinterpret_cast<uint4*>(&r)[1] = b;
  } else if constexpr (kBytes == 16) {
    *reinterpret_cast<uint4*>(&r) = __ldg(reinterpret_cast<const uint4*>(p));
  } else if constexpr (kBytes == 8) {
    *reinterpret_cast<uint2*>(&r) = __ldg(reinterpret_cast<const uint2*>(p));
  } else if constexpr (kBytes == 4) {
    *reinterpret_cast<unsigned*>(&r) = __ldg(reinterpret_cast<const unsigned*>(p));
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.v[e] = p[e];
  }
  return r;
}

// generic vector store of VEC elements
template <typename T, int VEC>
__device__ __forceinline__ void st_vec(T* p, const Vec<T, VEC>& r) {
  constexpr int kBytes = sizeof(T) * VEC;
  if constexpr (kBytes == 32) {
    reinterpret_cast<uint4*>(p)[0] = reinterpret_cast<const uint4*>(&r)[0];
    reinterpret_cast<uint4*>(p)[1] = reinterpret_cast<const uint4*>(&r)[1];
  } else if constexpr (kBytes == 16) {
    *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&r);
  } else if constexpr (kBytes == 8) {
    *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(&r);
  } else if constexpr (kBytes == 4) {
    *reinterpret_cast<unsigned*>(p) = *reinterpret_cast<const unsigned*>(&r);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) p[e] = r.v[e];
  }
}

__host__ __device__ inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// sub-warp width for a row of `chunks` vector chunks: the smallest power of
// two >= chunks (capped at 32); 32/S rows are gathered per warp instruction
__device__ __forceinline__ int subwarp_width(int chunks) {
  if (chunks >= kWarp) return kWarp;
  int s = 1;
  while (s < chunks) s <<= 1;
  return s;
}

}  // namespace neo
