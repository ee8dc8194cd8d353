// Sparse optimizer row updates shared by the fused backward and
// neo_apply_row_updates (embedding.py:212-267).
#pragma once
#include "common.cuh"

namespace neo {

// numpy pairwise summation of x_i = g_i * g_i (numpy/_core/src/umath/
// loops_utils.h.src pairwise_sum, block 128, 8 accumulators), the order the
// reference's np.mean(g * g, axis=1) uses (embedding.py:229)
static __device__ __noinline__ double pairwise_sumsq(const double* g, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, __dmul_rn(g[i], g[i]));
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(g[j], g[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(g[i + j], g[i + j]));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn(g[i], g[i]));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sumsq(g, n2), pairwise_sumsq(g + n2, n - n2));
}

// Target-row state prefetched at segment start so the HBM latency of the
// weight row and its moment overlaps the bag-id -> upstream gather chain.
// Covers rows of up to kPf*32 elements (all of c1..c3); wider rows read in place.
constexpr int kPf = 4;
template <typename W, typename Acc>
struct RowPrefetch {
  W w[kPf];
  Acc m[kPf];   // element-wise AdaGrad state
  Acc mrow;     // row-wise AdaGrad state
  bool valid;
};

template <typename W, typename Acc>
__device__ __forceinline__ void prefetch_row(bool enable, const W* wbase, const Acc* mbase,
                                             int optim, int64_t row, int32_t D, int lane,
                                             RowPrefetch<W, Acc>& pf) {
  pf.valid = enable && D <= kPf * kWarp;
  if (!pf.valid) return;
  const W* w = wbase + row * D;
#pragma unroll
  for (int i = 0; i < kPf; ++i) {
    const int j = lane + i * kWarp;
    pf.w[i] = j < D ? w[j] : W(0);
  }
  pf.mrow = Acc(0);
  if (optim == NEO_OPT_ROWWISE_ADAGRAD) {
    pf.mrow = mbase[row];
  } else if (optim == NEO_OPT_ADAGRAD) {
    const Acc* m = mbase + row * D;
#pragma unroll
    for (int i = 0; i < kPf; ++i) {
      const int j = lane + i * kWarp;
      pf.m[i] = j < D ? m[j] : Acc(0);
    }
  }
}

// one optimizer step on element j of the row (w_j, g_j; m_j for AdaGrad)
template <typename Acc>
__device__ __forceinline__ Acc sgd_step(Acc w, Acc g, double lr) {
  if constexpr (sizeof(Acc) == 8) return __dsub_rn(w, __dmul_rn(lr, g));
  else return w - (float)lr * g;
}
template <typename Acc>
__device__ __forceinline__ Acc rowwise_step(Acc w, Acc g, double lr, Acc denom) {
  if constexpr (sizeof(Acc) == 8) return __dsub_rn(w, __ddiv_rn(__dmul_rn(lr, g), denom));
  else return w - (float)lr * g / denom;
}
template <typename Acc>
__device__ __forceinline__ Acc adagrad_step(Acc w, Acc g, double lr, double eps, Acc& m) {
  if constexpr (sizeof(Acc) == 8) {
    m = __dadd_rn(m, __dmul_rn(g, g));
    return __dsub_rn(w, __ddiv_rn(__dmul_rn(lr, g), __dadd_rn(__dsqrt_rn(m), eps)));
  } else {
    m = m + g * g;
    return w - (float)lr * g / (sqrtf(m) + (float)eps);
  }
}

// Apply exactly one optimizer step to row `row` (embedding.py:212-254) from
// the aggregated gradient row g (shared memory, D elements, accumulator type).
template <typename W, typename Acc>
__device__ __forceinline__ void update_row(W* wbase, Acc* mom, int optim, double lr, double eps,
                                           int64_t row, int32_t D, const Acc* g, int lane,
                                           const RowPrefetch<W, Acc>& pf) {
  constexpr bool kExact = sizeof(Acc) == 8;
  W* w = wbase + row * D;
  if (optim != NEO_OPT_SGD) {
    bool nz = false;
    for (int j = lane; j < D; j += kWarp) nz |= (g[j] != Acc(0));
    if (!__any_sync(0xffffffffu, nz)) return;  // embedding.py:225-228
  }
  Acc denom = Acc(1);
  if (optim == NEO_OPT_ROWWISE_ADAGRAD) {
    const Acc m0 = pf.valid ? pf.mrow : mom[row];
    Acc m;
    if constexpr (kExact) {
      double mm = 0.0;
      if (lane == 0) mm = __dadd_rn(m0, __ddiv_rn(pairwise_sumsq((const double*)g, D), (double)D));
      m = __shfl_sync(0xffffffffu, mm, 0);
      denom = __dadd_rn(__dsqrt_rn(m), eps);
    } else {
      float ss = 0.f;
      for (int j = lane; j < D; j += kWarp) ss += g[j] * g[j];
      ss = warp_sum(ss);
      m = m0 + ss / (float)D;
      denom = sqrtf(m) + (float)eps;
    }
    if (lane == 0) mom[row] = m;
  }
  if (pf.valid) {
#pragma unroll
    for (int i = 0; i < kPf; ++i) {
      const int j = lane + i * kWarp;
      if (j >= D) break;
      const Acc wj = to_acc<Acc>(pf.w[i]);
      Acc r;
      if (optim == NEO_OPT_SGD) r = sgd_step<Acc>(wj, g[j], lr);
      else if (optim == NEO_OPT_ROWWISE_ADAGRAD) r = rowwise_step<Acc>(wj, g[j], lr, denom);
      else {
        Acc m = pf.m[i];
        r = adagrad_step<Acc>(wj, g[j], lr, eps, m);
        mom[row * D + j] = m;
      }
      w[j] = from_acc<W, Acc>(r);
    }
  } else {
    for (int j = lane; j < D; j += kWarp) {
      const Acc wj = to_acc<Acc>(w[j]);
      Acc r;
      if (optim == NEO_OPT_SGD) r = sgd_step<Acc>(wj, g[j], lr);
      else if (optim == NEO_OPT_ROWWISE_ADAGRAD) r = rowwise_step<Acc>(wj, g[j], lr, denom);
      else {
        Acc m = mom[row * D + j];
        r = adagrad_step<Acc>(wj, g[j], lr, eps, m);
        mom[row * D + j] = m;
      }
      w[j] = from_acc<W, Acc>(r);
    }
  }
}

}  // namespace neo
