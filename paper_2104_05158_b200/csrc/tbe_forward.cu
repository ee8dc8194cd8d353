// TBE forward: sum/mean pooling of embedding rows per (table, bag).
//
// Reference semantics: embedding.py:136-151 (forward_pooled: out[s] = sum of
// values[idx] over the bag, empty bag -> 0, accumulation sequential in buffer
// order via np.add.at) and embedding.py:154-168 (fused_forward: per-table
// outputs concatenated along columns in table order).
//
// B200 mapping: one warp per (table, bag).  The warp stages the bag's row ids
// in its own shared-memory slice (one coalesced load per 32 ids, range-checked
// on the way in), then walks them, gathering each row with 16-byte
// ld.global.nc vector loads — a row of D=128 fp32 is exactly one 512-byte
// warp-wide load.  Narrow rows (D*e < 512 B) are packed several per warp
// instruction (sub-warps of S lanes, R = 32/S rows per instruction) and the
// partial sums are folded with shuffles at the end; rows wider than one warp
// load are covered by column passes over the staged ids.  U rows are in
// flight per lane to cover HBM latency.  Accumulation is f32 for F32/F16
// storage; F64 storage accumulates in f64 one row at a time in buffer order,
// which reproduces np.add.at bit for bit.
#include <climits>

#include "common.cuh"

namespace neo {

constexpr int kFwdWarps = 8;   // warps per CTA
// scatter destination of the current launch (set by neo_tbe_forward_scatter
// around the dispatch; host-side, per thread)
static thread_local const uint64_t* g_out_ptrs = nullptr;
// forward grid cap in CTAs per SM (0 = one CTA per 8 bags, uncapped); process-wide
static int g_fwd_ctas_per_sm = 0;
static thread_local int64_t g_rows_per_dst = 1;
constexpr int kFwdStage = 64;  // row ids staged per warp per pass
constexpr int kFwdUnroll = 8;  // row gathers in flight per lane

template <typename W, typename Idx, typename Out, int VEC>
__device__ __forceinline__ void fwd_bag(const W* __restrict__ wt, int32_t D, int64_t H,
                                        const Idx* __restrict__ indices, int64_t start,
                                        int64_t end, Idx* s_idx, int pooling, Out* orow,
                                        neo_error* err, int lane) {
  constexpr bool kExact = sizeof(W) == 8;  // f64 oracle-order mode
  using Acc = typename std::conditional<kExact, double, float>::type;
  constexpr int U = kFwdUnroll;
  const int chunks = D / VEC;
  const int S = kExact ? kWarp : subwarp_width(chunks);
  const int R = kWarp / S;
  const int sub = lane / S;
  const int sl = lane % S;
  const int64_t len = end - start;
  const bool single_stage = len <= kFwdStage;

  for (int cbase = 0; cbase < chunks; cbase += S) {  // column passes
    const int ch = cbase + sl;
    const bool col_live = ch < chunks;
    Acc acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = Acc(0);

    for (int64_t base = start; base < end; base += kFwdStage) {
      const int n = (int)min64(kFwdStage, end - base);
      if (cbase == 0 || !single_stage) {
        __syncwarp();
        for (int i = lane; i < n; i += kWarp) {
          Idx v = indices[base + i];
          if (v < 0 || (int64_t)v >= H) {
            if (cbase == 0) record_bad_index(err, base + i);
            v = Idx(-1);
          }
          s_idx[i] = v;
        }
        __syncwarp();
      }
      for (int j = 0; j < n; j += R * U) {
        Vec<W, VEC> v[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = j + u * R + sub;
          const int64_t row = r < n ? (int64_t)s_idx[r] : -1;
          live[u] = row >= 0;
          if (live[u] && col_live) {
            v[u] = ld_vec<W, VEC>(wt + row * D + (int64_t)ch * VEC);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) v[u].v[e] = W(0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (kExact && !live[u]) continue;  // exact sequence of adds
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] += to_acc<Acc>(v[u].v[e]);
        }
      }
    }
    if (!kExact) {  // fold the R sub-warp partial sums
      for (int o = S; o < kWarp; o <<= 1) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
      }
    }
    if (sub == 0 && col_live) {
      Vec<Out, VEC> o;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        Acc a = acc[e];
        if (pooling == NEO_POOL_MEAN) a = len > 0 ? a / (Acc)len : Acc(0);
        o.v[e] = from_acc<Out, Acc>(a);
      }
      st_vec<Out, VEC>(orow + (int64_t)ch * VEC, o);
    }
  }
}

template <typename W, typename Idx, typename Out>
__global__ void __launch_bounds__(kFwdWarps * kWarp)
tbe_forward_kernel(int32_t T, int64_t B, const int64_t* __restrict__ row_offsets,
                   const int32_t* __restrict__ dim_offsets, const uint64_t* __restrict__ weights,
                   const Idx* __restrict__ indices, const int64_t* __restrict__ offsets,
                   int pooling, Out* __restrict__ out, int64_t out_stride, neo_error* err,
                   const uint64_t* __restrict__ out_ptrs, int64_t rows_per_dst) {
  constexpr int kVec = 16 / sizeof(W);
  __shared__ Idx s_idx[kFwdWarps][kFwdStage];
  const int warp = threadIdx.x / kWarp;
  const int lane = threadIdx.x % kWarp;
  // grid-stride over bags: the grid may be capped (neo_set_forward_residency)
  // so that a side-stream kernel (the backward's key build + sort) can
  // co-reside with this DRAM-bound gather
  for (int64_t bag = (int64_t)blockIdx.x * kFwdWarps + warp; bag < (int64_t)T * B;
       bag += (int64_t)gridDim.x * kFwdWarps) {
  const int32_t t = (int32_t)(bag / B);
  const int64_t b = bag - (int64_t)t * B;
  const int32_t doff = dim_offsets[t];
  const int32_t D = dim_offsets[t + 1] - doff;
  const int64_t H = row_offsets[t + 1] - row_offsets[t];
  const W* wt = reinterpret_cast<const W*>(weights[t]);
  // out_ptrs: row b goes to destination b / rows_per_dst (e.g. the peer GPU's
  // receive buffer: the pooled all-to-all is performed by this store)
  Out* obase = out;
  int64_t orow_i = b;
  if (out_ptrs) {
    const int64_t d = b / rows_per_dst;
    obase = reinterpret_cast<Out*>(out_ptrs[d]);
    orow_i = b - d * rows_per_dst;
  }
  Out* orow = obase + orow_i * out_stride + doff;
  const bool vec = (D % kVec) == 0 && aligned16(wt) && (doff % kVec) == 0 &&
                   (out_stride % kVec) == 0 &&
                   ((reinterpret_cast<uintptr_t>(obase) % (sizeof(Out) * kVec)) == 0);
  if (vec)
    fwd_bag<W, Idx, Out, kVec>(wt, D, H, indices, offsets[bag], offsets[bag + 1], s_idx[warp],
                               pooling, orow, err, lane);
  else
    fwd_bag<W, Idx, Out, 1>(wt, D, H, indices, offsets[bag], offsets[bag + 1], s_idx[warp],
                            pooling, orow, err, lane);
  __syncwarp();
  }
}

template <typename W, typename Idx, typename Out>
static int launch_fwd(dim3 grid, cudaStream_t s, int32_t T, int64_t B, const int64_t* ro,
                      const int32_t* dof, const uint64_t* w, const void* idx, const int64_t* off,
                      int pooling, void* out, int64_t os, neo_error* err) {
  tbe_forward_kernel<W, Idx, Out><<<grid, kFwdWarps * kWarp, 0, s>>>(
      T, B, ro, dof, w, (const Idx*)idx, off, pooling, (Out*)out, os, err, g_out_ptrs, g_rows_per_dst);
  return check_launch("neo_tbe_forward");
}

template <typename W, typename Idx>
static int launch_fwd_out(int32_t out_dtype, dim3 grid, cudaStream_t s, int32_t T, int64_t B,
                          const int64_t* ro, const int32_t* dof, const uint64_t* w,
                          const void* idx, const int64_t* off, int pooling, void* out,
                          int64_t os, neo_error* err) {
  if constexpr (sizeof(W) == 8) {
    if (out_dtype != NEO_F64) return fail(NEO_E_ARG, "F64 tables pool into F64 outputs");
    return launch_fwd<W, Idx, double>(grid, s, T, B, ro, dof, w, idx, off, pooling, out, os, err);
  } else {
    switch (out_dtype) {
      case NEO_F32:
        return launch_fwd<W, Idx, float>(grid, s, T, B, ro, dof, w, idx, off, pooling, out, os,
                                         err);
      case NEO_F16:
        return launch_fwd<W, Idx, __half>(grid, s, T, B, ro, dof, w, idx, off, pooling, out, os,
                                          err);
      case NEO_BF16:
        return launch_fwd<W, Idx, __nv_bfloat16>(grid, s, T, B, ro, dof, w, idx, off, pooling,
                                                 out, os, err);
      default:
        return fail(NEO_E_ARG, "neo_tbe_forward: output dtype must be F32, F16 or BF16");
    }
  }
}

template <typename W>
static int launch_fwd_idx(int32_t index_dtype, int32_t out_dtype, dim3 grid, cudaStream_t s,
                          int32_t T, int64_t B, const int64_t* ro, const int32_t* dof,
                          const uint64_t* w, const void* idx, const int64_t* off, int pooling,
                          void* out, int64_t os, neo_error* err) {
  if (index_dtype == NEO_I32)
    return launch_fwd_out<W, int32_t>(out_dtype, grid, s, T, B, ro, dof, w, idx, off, pooling,
                                      out, os, err);
  return launch_fwd_out<W, int64_t>(out_dtype, grid, s, T, B, ro, dof, w, idx, off, pooling, out,
                                    os, err);
}

}  // namespace neo

extern "C" int neo_set_forward_residency(int32_t ctas_per_sm) {
  if (ctas_per_sm < 0) return neo::fail(NEO_E_ARG, "neo_set_forward_residency: negative");
  neo::g_fwd_ctas_per_sm = ctas_per_sm;
  return NEO_OK;
}

extern "C" int neo_tbe_forward(int32_t num_tables, int64_t batch, const int64_t* row_offsets,
                               const int32_t* dim_offsets, int32_t max_dim,
                               const uint64_t* weights, int32_t weight_dtype,
                               const void* indices, int32_t index_dtype, const int64_t* offsets,
                               int32_t pooling, void* out, int32_t out_dtype, int64_t out_stride,
                               neo_error* err, void* stream) {
  using namespace neo;
  if (num_tables < 0 || batch < 0 || max_dim < 0 || out_stride < 0)
    return fail(NEO_E_ARG, "neo_tbe_forward: negative size");
  if (num_tables == 0 || batch == 0) return NEO_OK;
  if (!row_offsets || !dim_offsets || !weights || !offsets || !out)
    return fail(NEO_E_ARG, "neo_tbe_forward: null pointer");
  if (index_dtype != NEO_I32 && index_dtype != NEO_I64)
    return fail(NEO_E_ARG, "neo_tbe_forward: index dtype must be I32 or I64");
  if (pooling != NEO_POOL_SUM && pooling != NEO_POOL_MEAN)
    return fail(NEO_E_ARG, "neo_tbe_forward: pooling must be SUM or MEAN");
  const int64_t bags = (int64_t)num_tables * batch;
  const int64_t blocks = (bags + kFwdWarps - 1) / kFwdWarps;
  if (blocks > INT_MAX) return fail(NEO_E_ARG, "neo_tbe_forward: too many bags");
  int64_t gblocks = blocks;
  if (g_fwd_ctas_per_sm > 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t cap = (int64_t)sms * g_fwd_ctas_per_sm;
    if (gblocks > cap) gblocks = cap;
  }
  const dim3 grid((unsigned)gblocks);
  cudaStream_t s = as_stream(stream);
  int rc;
  switch (weight_dtype) {
    case NEO_F32:
      rc = launch_fwd_idx<float>(index_dtype, out_dtype, grid, s, num_tables, batch, row_offsets,
                                 dim_offsets, weights, indices, offsets, pooling, out, out_stride,
                                 err);
      break;
    case NEO_F16:
      rc = launch_fwd_idx<__half>(index_dtype, out_dtype, grid, s, num_tables, batch, row_offsets,
                                  dim_offsets, weights, indices, offsets, pooling, out,
                                  out_stride, err);
      break;
    case NEO_F64:
      rc = launch_fwd_idx<double>(index_dtype, out_dtype, grid, s, num_tables, batch, row_offsets,
                                  dim_offsets, weights, indices, offsets, pooling, out,
                                  out_stride, err);
      break;
    default:
      return fail(NEO_E_ARG, "neo_tbe_forward: weight dtype must be F32, F16 or F64");
  }
  if (rc != NEO_OK) return rc;
  launch_error_finalize(err, indices, index_dtype, offsets, batch, num_tables, s);
  return check_launch("neo_tbe_forward(finalize)");
}

extern "C" int neo_tbe_forward_scatter(int32_t num_tables, int64_t batch, const int64_t* row_offsets,
                                       const int32_t* dim_offsets, int32_t max_dim,
                                       const uint64_t* weights, int32_t weight_dtype,
                                       const void* indices, int32_t index_dtype,
                                       const int64_t* offsets, int32_t pooling,
                                       const uint64_t* out_ptrs, int64_t rows_per_dst,
                                       int32_t out_dtype, int64_t out_stride, neo_error* err,
                                       void* stream) {
  using namespace neo;
  if (!out_ptrs || rows_per_dst < 1)
    return fail(NEO_E_ARG, "neo_tbe_forward_scatter: out_ptrs and rows_per_dst >= 1 required");
  g_out_ptrs = out_ptrs;
  g_rows_per_dst = rows_per_dst;
  // `out` is unused when out_ptrs is set; pass a non-null placeholder
  const int rc = neo_tbe_forward(num_tables, batch, row_offsets, dim_offsets, max_dim, weights,
                                 weight_dtype, indices, index_dtype, offsets, pooling,
                                 const_cast<uint64_t*>(out_ptrs), out_dtype, out_stride, err, stream);
  g_out_ptrs = nullptr;
  g_rows_per_dst = 1;
  return rc;
}
