// Integer layout kernels around the TBE (bit-exact) and small element-wise
// helpers: row-wise bucketisation, (W,T,B)<->(T,W,B) block permute,
// lengths->offsets, block gathers for the input all-to-all, pooled-row piece
// copies for the output all-to-all, precision casts and optimizer updates
// from materialised RowGradients.
#include <algorithm>
#include <climits>
#include <cub/block/block_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "optim.cuh"

namespace neo {

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t inclusive_scan_temp(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int64_t)(n > 0 ? n : 1));
  return bytes;
}

// offsets[0] = 0, offsets[i+1] = offsets[i] + lengths[i] (model.py:365-370)
static int scan_lengths(int64_t n, const int64_t* lengths, int64_t* offsets, void* temp,
                        size_t temp_bytes, cudaStream_t s) {
  if (cudaMemsetAsync(offsets, 0, sizeof(int64_t), s) != cudaSuccess)
    return fail(NEO_E_CUDA, "scan: memset failed");
  if (n == 0) return NEO_OK;
  if (cub::DeviceScan::InclusiveSum(temp, temp_bytes, lengths, offsets + 1, n, s) != cudaSuccess)
    return fail(NEO_E_CUDA, "scan: inclusive sum failed");
  return NEO_OK;
}

// ---------------------------------------------------------------------------
// row-wise bucketisation (comms.py:107-141)

constexpr int kMaxShards = 64;
struct ShardStarts {
  int64_t v[kMaxShards + 1];
};

__device__ __forceinline__ int shard_of(int64_t x, const ShardStarts& st, int k) {
  // searchsorted(ends, x, side="right") over ends = st.v[1..k]
  int lo = 0, hi = k - 1;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (x < st.v[mid + 1]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

template <typename Idx, bool kScatter>
__global__ void __launch_bounds__(256)
bucketize_kernel(int64_t n, const int64_t* __restrict__ offsets, const Idx* __restrict__ indices,
                 int k, ShardStarts st, int64_t* __restrict__ out_lengths,
                 const int64_t* __restrict__ out_offsets, Idx* __restrict__ out_indices,
                 neo_error* err) {
  __shared__ int32_t s_cnt[8][kMaxShards];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int64_t b = (int64_t)blockIdx.x * 8 + warp;
  if (b >= n) return;
  int32_t* cnt = s_cnt[warp];
  for (int s = lane; s < k; s += kWarp) cnt[s] = 0;
  __syncwarp();
  const int64_t start = offsets[b], end = offsets[b + 1];
  const int64_t H = st.v[k];
  for (int64_t base = start; base < end; base += kWarp) {
    const int64_t p = base + lane;
    const bool live = p < end;
    int sh = -1;
    int64_t x = 0;
    if (live) {
      x = (int64_t)indices[p];
      if (x < 0 || x >= H) {
        if (!kScatter) record_bad_index(err, p);
      } else {
        sh = shard_of(x, st, k);
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, sh);
    const int leader = __ffs(peers) - 1;
    if (kScatter && sh >= 0) {
      const unsigned lt = peers & ((1u << lane) - 1u);
      const int64_t pos = out_offsets[(int64_t)sh * n + b] + cnt[sh] + __popc(lt);
      out_indices[pos] = (Idx)(x - st.v[sh]);
    }
    __syncwarp();
    if (sh >= 0 && lane == leader) cnt[sh] += __popc(peers);
    __syncwarp();
  }
  if (!kScatter)
    for (int s = lane; s < k; s += kWarp) out_lengths[(int64_t)s * n + b] = cnt[s];
}

// Many row-wise tables in one launch (the sharded step's sender side): warp
// per (row-wise table r, bag b); table r is tables[r] of the full batch
// (global offsets over T*B bags), its shard boundaries starts[r][0..k_r].
// Output blocks are (r, shard, bag) ordered with kmax shard slots per table
// (unused slots stay empty), so one scan gives every block's offsets.
template <typename Idx, bool kScatter>
__global__ void __launch_bounds__(256)
bucketize_multi_kernel(int32_t R, int64_t B, const int32_t* __restrict__ tables,
                       const int64_t* __restrict__ offsets, const Idx* __restrict__ indices, int32_t kmax,
                       const int64_t* __restrict__ starts, const int32_t* __restrict__ kk,
                       int64_t* __restrict__ out_lengths, const int64_t* __restrict__ out_offsets,
                       Idx* __restrict__ out_indices) {
  __shared__ int32_t s_cnt[8][kMaxShards];
  __shared__ int64_t s_st[8][kMaxShards + 1];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int64_t g = (int64_t)blockIdx.x * 8 + warp;
  if (g >= (int64_t)R * B) return;
  const int r = (int)(g / B);
  const int64_t b = g - (int64_t)r * B;
  const int k = kk[r];
  int32_t* cnt = s_cnt[warp];
  int64_t* st = s_st[warp];
  for (int i = lane; i < kMaxShards; i += kWarp) cnt[i] = 0;
  for (int i = lane; i <= k; i += kWarp) st[i] = starts[(int64_t)r * (kmax + 1) + i];
  __syncwarp();
  const int64_t gb = (int64_t)tables[r] * B + b;
  const int64_t start = offsets[gb], end = offsets[gb + 1];
  const int64_t H = st[k];
  const int64_t blk0 = (int64_t)r * kmax;
  for (int64_t base = start; base < end; base += kWarp) {
    const int64_t p = base + lane;
    int sh = -1;
    int64_t x = 0;
    if (p < end) {
      x = (int64_t)indices[p];
      if (x >= 0 && x < H) {  // ids outside the table were reported by neo_check_indices
        int lo = 0, hi = k - 1;
        while (lo < hi) {
          const int mid = (lo + hi) / 2;
          if (x < st[mid + 1]) hi = mid;
          else lo = mid + 1;
        }
        sh = lo;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, sh);
    const int leader = __ffs(peers) - 1;
    if (kScatter && sh >= 0) {
      const unsigned lt = peers & ((1u << lane) - 1u);
      const int64_t pos = out_offsets[(blk0 + sh) * B + b] + cnt[sh] + __popc(lt);
      out_indices[pos] = (Idx)(x - st[sh]);
    }
    __syncwarp();
    if (sh >= 0 && lane == leader) cnt[sh] += __popc(peers);
    __syncwarp();
  }
  if (!kScatter)
    for (int i = lane; i < kmax; i += kWarp) out_lengths[(blk0 + i) * B + b] = cnt[i];
}

// ---------------------------------------------------------------------------
// block permute (comms.py:222-257)

__global__ void block_count_kernel(int32_t outer, int32_t inner, int64_t B,
                                   const int64_t* __restrict__ lengths, int64_t* counts_oi,
                                   int64_t* counts_io) {
  const int64_t blk = blockIdx.x;  // (o, i) in input order
  const int o = (int)(blk / inner), i = (int)(blk % inner);
  int64_t acc = 0;
  for (int64_t j = threadIdx.x; j < B; j += blockDim.x) acc += lengths[blk * B + j];
  typedef cub::BlockReduce<int64_t, 256> R;
  __shared__ typename R::TempStorage tmp;
  acc = R(tmp).Sum(acc);
  if (threadIdx.x == 0) {
    counts_oi[blk] = acc;
    counts_io[(int64_t)i * outer + o] = acc;
  }
}

template <typename Idx>
__global__ void block_permute_kernel(int32_t outer, int32_t inner, int64_t B,
                                     const int64_t* __restrict__ lengths,
                                     const Idx* __restrict__ indices,
                                     const int64_t* __restrict__ in_off,
                                     const int64_t* __restrict__ out_off,
                                     int64_t* __restrict__ out_lengths, Idx* __restrict__ out_indices) {
  const int64_t blk = blockIdx.x;
  const int o = (int)(blk / inner), i = (int)(blk % inner);
  const int64_t oblk = (int64_t)i * outer + o;
  const int64_t stride = (int64_t)gridDim.y * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  for (int64_t j = t0; j < B; j += stride) out_lengths[oblk * B + j] = lengths[blk * B + j];
  const int64_t src = in_off[blk], dst = out_off[oblk];
  const int64_t cnt = in_off[blk + 1] - src;
  for (int64_t j = t0; j < cnt; j += stride) out_indices[dst + j] = indices[src + j];
}

// ---------------------------------------------------------------------------
// pooled-row pieces (comms.py:692-711)

template <typename S, typename D>
__global__ void __launch_bounds__(256)
copy_pieces_kernel(int64_t rows, const neo_piece* __restrict__ pieces, int32_t num_pieces) {
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  if (r >= rows) return;
  for (int pi = 0; pi < num_pieces; ++pi) {
    const neo_piece pc = pieces[pi];
    const S* src = reinterpret_cast<const S*>(pc.src) + r * pc.src_stride + pc.src_col;
    D* dst = reinterpret_cast<D*>(pc.dst) + r * pc.dst_stride + pc.dst_col;
    // 16-byte accesses on the narrower side (8 x 16-bit or 4 x 32-bit
    // elements per lane); f64 pieces take the scalar path
    constexpr int kMin = sizeof(S) < sizeof(D) ? sizeof(S) : sizeof(D);
    constexpr int V = 16 / kMin;
    constexpr bool kVecOk = sizeof(S) <= 4 && sizeof(D) <= 4;
    const bool vec = kVecOk && (pc.width % V) == 0 && (reinterpret_cast<uintptr_t>(src) % 16) == 0 &&
                     (reinterpret_cast<uintptr_t>(dst) % 16) == 0;
    if (vec) {
      for (int j = lane * V; j < pc.width; j += kWarp * V) {
        Vec<S, V> a = ld_vec<S, V>(src + j);
        Vec<D, V> o;
        if (pc.accumulate) {  // coherent 16-byte loads: earlier pieces of this launch wrote dst
#pragma unroll
          for (int q = 0; q < (int)(sizeof(D) * V) / 16; ++q)
            reinterpret_cast<uint4*>(&o)[q] = reinterpret_cast<const uint4*>(dst + j)[q];
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const float x = Elem<S>::to_f(a.v[e]);
          o.v[e] = pc.accumulate ? Elem<D>::from_f(Elem<D>::to_f(o.v[e]) + x) : Elem<D>::from_f(x);
        }
#pragma unroll
        for (int q = 0; q < (int)(sizeof(D) * V) / 16; ++q)
          reinterpret_cast<uint4*>(dst + j)[q] = reinterpret_cast<const uint4*>(&o)[q];
      }
    } else {
      for (int j = lane; j < pc.width; j += kWarp) {
        if constexpr (sizeof(S) == 8 || sizeof(D) == 8) {
          const double x = Elem<S>::to_d(src[j]);
          dst[j] = pc.accumulate ? Elem<D>::from_d(Elem<D>::to_d(dst[j]) + x) : Elem<D>::from_d(x);
        } else {
          const float x = Elem<S>::to_f(src[j]);
          dst[j] = pc.accumulate ? Elem<D>::from_f(Elem<D>::to_f(dst[j]) + x) : Elem<D>::from_f(x);
        }
      }
    }
    __syncwarp();
  }
}

// Narrow pieces lane-parallel: every chunk is one 16-byte vector (on the
// narrower side) of one piece, with its row stride; warp per row, lanes
// stride over the chunks, so a row's many narrow pieces (the sharded
// exchange's per-shard column blocks) keep all lanes storing 16 bytes.
template <typename S, typename D>
__global__ void __launch_bounds__(256)
copy_chunks_kernel(int64_t rows, const neo_chunk* __restrict__ chunks, int32_t num_chunks) {
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  if (r >= rows) return;
  constexpr int kMin = sizeof(S) < sizeof(D) ? sizeof(S) : sizeof(D);
  constexpr int V = 16 / kMin;
  for (int c = lane; c < num_chunks; c += kWarp) {
    const neo_chunk ch = chunks[c];
    const S* src = reinterpret_cast<const S*>(ch.src + r * ch.src_stride);
    D* dst = reinterpret_cast<D*>(ch.dst + r * ch.dst_stride);
    Vec<S, V> a = ld_vec<S, V>(src);
    Vec<D, V> o;
#pragma unroll
    for (int e = 0; e < V; ++e) o.v[e] = Elem<D>::from_f(Elem<S>::to_f(a.v[e]));
#pragma unroll
    for (int q = 0; q < (int)(sizeof(D) * V) / 16; ++q)
      reinterpret_cast<uint4*>(dst)[q] = reinterpret_cast<const uint4*>(&o)[q];
  }
}

// ---------------------------------------------------------------------------
// block gather

template <typename T>
__global__ void gather_blocks_kernel(int32_t n, const uint64_t* __restrict__ src_ptrs,
                                     const int64_t* __restrict__ counts,
                                     const int64_t* __restrict__ dst_offsets, T* __restrict__ dst) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const T* src = reinterpret_cast<const T*>(src_ptrs[i]);
  const int64_t cnt = counts[i];
  T* d = dst + dst_offsets[i];
  const int64_t stride = (int64_t)gridDim.y * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; j < cnt; j += stride) d[j] = src[j];
}

// ---------------------------------------------------------------------------
// casts

// range check of a CombinedBatch's ids (model.py:344-348, embedding.py:144-146):
// table t's ids (positions offsets[t*B] .. offsets[(t+1)*B]) must lie in
// [0, rows[t]); the first offending position is recorded in err
template <typename Idx>
__global__ void check_indices_kernel(int32_t T, int64_t B, const int64_t* __restrict__ rows,
                                     const int64_t* __restrict__ offsets, const Idx* __restrict__ ids,
                                     neo_error* err) {
  const int t = blockIdx.y;
  const int64_t lo = offsets[(int64_t)t * B], hi = offsets[(int64_t)(t + 1) * B];
  const int64_t H = rows[t];
  for (int64_t p = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < hi;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)ids[p];
    if (v < 0 || v >= H) record_bad_index(err, p);
  }
}

template <typename S, typename D>
__global__ void cast_kernel(int64_t n, const S* __restrict__ src, D* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(S) == 8) dst[i] = Elem<D>::from_d(src[i]);
    else dst[i] = Elem<D>::from_f(Elem<S>::to_f(src[i]));
  }
}

__global__ void fp16_roundtrip_kernel(int64_t n, double* __restrict__ x, uint8_t* overflow,
                                      int32_t* nonfinite) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    if (!isfinite(v)) {
      if (nonfinite) *nonfinite = 1;
      continue;
    }
    // direct f64 -> f16 round-to-nearest-even, as numpy's astype(float16)
    const double q = (double)__half2float(__double2half(v));
    x[i] = q;
    if (overflow) overflow[i] = isinf(q) ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// optimizer from RowGradients

template <typename W>
__global__ void __launch_bounds__(256)
apply_rows_kernel(int64_t n, const int64_t* __restrict__ ids, const void* grads, int32_t dim,
                  W* weight, void* moment, int optim, double lr, double eps) {
  using Acc = typename std::conditional<sizeof(W) == 8, double, float>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  Acc* g = reinterpret_cast<Acc*>(smem_raw) + (size_t)warp * dim;
  const int64_t i = (int64_t)blockIdx.x * 8 + warp;
  if (i >= n) return;
  const Acc* src = reinterpret_cast<const Acc*>(grads) + i * dim;
  for (int j = lane; j < dim; j += kWarp) g[j] = src[j];
  __syncwarp();
  const int64_t row = ids ? ids[i] : i;
  Acc* mom = reinterpret_cast<Acc*>(moment);
  RowPrefetch<W, Acc> pf;
  prefetch_row<W, Acc>(true, weight, mom, optim, row, dim, lane, pf);
  update_row<W, Acc>(weight, mom, optim, lr, eps, row, dim, g, lane, pf);
}

}  // namespace neo

using namespace neo;

extern "C" {

size_t neo_scan_workspace_bytes(int64_t n) { return al256(inclusive_scan_temp(n)); }

int neo_lengths_to_offsets(int64_t n, const int64_t* lengths, int64_t* offsets, void* workspace,
                           size_t workspace_bytes, void* stream) {
  if (n < 0 || !offsets || (n > 0 && !lengths)) return fail(NEO_E_ARG, "lengths_to_offsets: bad args");
  if (workspace_bytes < inclusive_scan_temp(n))
    return fail(NEO_E_ARG, "lengths_to_offsets: workspace too small");
  return scan_lengths(n, lengths, offsets, workspace, workspace_bytes, as_stream(stream));
}

int neo_bucketize_rowwise_multi(int32_t num_rw, int64_t batch, const int32_t* tables, const int64_t* offsets,
                                const void* indices, int32_t index_dtype, int32_t kmax, const int64_t* shard_starts,
                                const int32_t* shard_counts, int64_t* out_lengths, int64_t* out_offsets,
                                void* out_indices, void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (num_rw < 0 || batch < 0 || kmax < 1) return fail(NEO_E_ARG, "bucketize_multi: bad sizes");
  if (kmax > kMaxShards) return fail(NEO_E_ARG, "bucketize_multi: at most 64 row shards");
  if (index_dtype != NEO_I32 && index_dtype != NEO_I64)
    return fail(NEO_E_ARG, "bucketize_multi: index dtype must be I32 or I64");
  const int64_t n = (int64_t)num_rw * batch;
  if (workspace_bytes < inclusive_scan_temp((int64_t)kmax * n))
    return fail(NEO_E_ARG, "bucketize_multi: workspace too small");
  if (n == 0) {
    if (cudaMemsetAsync(out_offsets, 0, sizeof(int64_t), s) != cudaSuccess)
      return fail(NEO_E_CUDA, "bucketize_multi: memset failed");
    return NEO_OK;
  }
  if (!tables || !offsets || !shard_starts || !shard_counts || !out_lengths || !out_offsets)
    return fail(NEO_E_ARG, "bucketize_multi: null pointer");
  const unsigned grid = (unsigned)((n + 7) / 8);
#define NEO_BKM(IDX, SC, OUT)                                                                              \
  bucketize_multi_kernel<IDX, SC><<<grid, 256, 0, s>>>(num_rw, batch, tables, offsets, (const IDX*)indices, \
                                                       kmax, shard_starts, shard_counts, out_lengths,      \
                                                       SC ? out_offsets : nullptr, (IDX*)OUT)
  if (index_dtype == NEO_I32) NEO_BKM(int32_t, false, nullptr);
  else NEO_BKM(int64_t, false, nullptr);
  int rc = check_launch("bucketize_multi(count)");
  if (rc) return rc;
  rc = scan_lengths((int64_t)kmax * n, out_lengths, out_offsets, workspace, workspace_bytes, s);
  if (rc) return rc;
  if (index_dtype == NEO_I32) NEO_BKM(int32_t, true, out_indices);
  else NEO_BKM(int64_t, true, out_indices);
#undef NEO_BKM
  return check_launch("bucketize_multi(scatter)");
}

size_t neo_bucketize_workspace_bytes(int64_t n, int32_t k) {
  return al256(inclusive_scan_temp((int64_t)k * n));
}

int neo_bucketize_rowwise(int64_t n, const int64_t* offsets, const void* indices,
                          int32_t index_dtype, int32_t k, const int64_t* shard_starts_host,
                          int64_t* out_lengths, int64_t* out_offsets, void* out_indices,
                          int32_t table, neo_error* err, void* workspace, size_t workspace_bytes,
                          void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n < 0 || k < 1 || !shard_starts_host) return fail(NEO_E_ARG, "bucketize: bad sizes");
  if (k > kMaxShards) return fail(NEO_E_ARG, "bucketize: at most 64 row shards");
  if (index_dtype != NEO_I32 && index_dtype != NEO_I64)
    return fail(NEO_E_ARG, "bucketize: index dtype must be I32 or I64");
  ShardStarts st{};
  int64_t pos = 0;
  for (int i = 0; i < k; ++i) {  // comms.py:121-125
    const int64_t a = shard_starts_host[i], b = shard_starts_host[i + 1];
    if (a != pos || b <= a) return fail(NEO_E_ARG, "boundaries: must tile [0, H) in order");
    st.v[i] = a;
    pos = b;
  }
  st.v[k] = pos;
  if (workspace_bytes < inclusive_scan_temp((int64_t)k * n))
    return fail(NEO_E_ARG, "bucketize: workspace too small");
  if (n == 0) {
    if (cudaMemsetAsync(out_offsets, 0, sizeof(int64_t), s) != cudaSuccess)
      return fail(NEO_E_CUDA, "bucketize: memset failed");
    return NEO_OK;
  }
  const unsigned grid = (unsigned)((n + 7) / 8);
  if (index_dtype == NEO_I32)
    bucketize_kernel<int32_t, false><<<grid, 256, 0, s>>>(n, offsets, (const int32_t*)indices, k, st,
                                                          out_lengths, nullptr, nullptr, err);
  else
    bucketize_kernel<int64_t, false><<<grid, 256, 0, s>>>(n, offsets, (const int64_t*)indices, k, st,
                                                          out_lengths, nullptr, nullptr, err);
  int rc = check_launch("bucketize(count)");
  if (rc) return rc;
  rc = scan_lengths((int64_t)k * n, out_lengths, out_offsets, workspace, workspace_bytes, s);
  if (rc) return rc;
  if (index_dtype == NEO_I32)
    bucketize_kernel<int32_t, true><<<grid, 256, 0, s>>>(n, offsets, (const int32_t*)indices, k, st,
                                                         out_lengths, out_offsets,
                                                         (int32_t*)out_indices, err);
  else
    bucketize_kernel<int64_t, true><<<grid, 256, 0, s>>>(n, offsets, (const int64_t*)indices, k, st,
                                                         out_lengths, out_offsets,
                                                         (int64_t*)out_indices, err);
  rc = check_launch("bucketize(scatter)");
  if (rc) return rc;
  if (err) {
    launch_error_finalize(err, indices, index_dtype, nullptr, 0, 0, s);
    rc = check_launch("bucketize(finalize)");
    if (rc) return rc;
    (void)table;
  }
  return NEO_OK;
}

size_t neo_permute_workspace_bytes(int32_t outer, int32_t inner) {
  const int64_t m = (int64_t)outer * inner;
  return 4 * al256(sizeof(int64_t) * (m + 1)) + al256(inclusive_scan_temp(m));
}

int neo_permute_blocks(int32_t outer, int32_t inner, int64_t B, const int64_t* lengths,
                       const void* indices, int32_t index_dtype, int64_t* out_lengths,
                       void* out_indices, void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (outer < 0 || inner < 0 || B < 0) return fail(NEO_E_ARG, "permute: negative size");
  if (index_dtype != NEO_I32 && index_dtype != NEO_I64)
    return fail(NEO_E_ARG, "permute: index dtype must be I32 or I64");
  const int64_t m = (int64_t)outer * inner;
  if (m == 0 || B == 0) return NEO_OK;
  if (m > INT_MAX) return fail(NEO_E_ARG, "permute: too many blocks");
  if (workspace_bytes < neo_permute_workspace_bytes(outer, inner))
    return fail(NEO_E_ARG, "permute: workspace too small");
  unsigned char* w = static_cast<unsigned char*>(workspace);
  int64_t* c_oi = reinterpret_cast<int64_t*>(w);
  w += al256(sizeof(int64_t) * (m + 1));
  int64_t* c_io = reinterpret_cast<int64_t*>(w);
  w += al256(sizeof(int64_t) * (m + 1));
  int64_t* in_off = reinterpret_cast<int64_t*>(w);
  w += al256(sizeof(int64_t) * (m + 1));
  int64_t* out_off = reinterpret_cast<int64_t*>(w);
  w += al256(sizeof(int64_t) * (m + 1));
  const size_t tb = inclusive_scan_temp(m);
  block_count_kernel<<<(unsigned)m, 256, 0, s>>>(outer, inner, B, lengths, c_oi, c_io);
  int rc = check_launch("permute(count)");
  if (rc) return rc;
  rc = scan_lengths(m, c_oi, in_off, w, tb, s);
  if (rc) return rc;
  rc = scan_lengths(m, c_io, out_off, w, tb, s);
  if (rc) return rc;
  const dim3 grid((unsigned)m, 8);
  if (index_dtype == NEO_I32)
    block_permute_kernel<int32_t><<<grid, 256, 0, s>>>(outer, inner, B, lengths,
                                                       (const int32_t*)indices, in_off, out_off,
                                                       out_lengths, (int32_t*)out_indices);
  else
    block_permute_kernel<int64_t><<<grid, 256, 0, s>>>(outer, inner, B, lengths,
                                                       (const int64_t*)indices, in_off, out_off,
                                                       out_lengths, (int64_t*)out_indices);
  return check_launch("permute(copy)");
}

int neo_copy_pieces(int64_t rows, const neo_piece* pieces, int32_t num_pieces, int32_t src_dtype,
                    int32_t dst_dtype, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (rows < 0 || num_pieces < 0) return fail(NEO_E_ARG, "copy_pieces: negative size");
  if (rows == 0 || num_pieces == 0) return NEO_OK;
  const int64_t blocks = (rows + 7) / 8;
  if (blocks > INT_MAX) return fail(NEO_E_ARG, "copy_pieces: too many rows");
  const unsigned g = (unsigned)blocks;
#define NEO_PC(S, D) copy_pieces_kernel<S, D><<<g, 256, 0, s>>>(rows, pieces, num_pieces)
  if (src_dtype == NEO_F32 && dst_dtype == NEO_F32) NEO_PC(float, float);
  else if (src_dtype == NEO_F16 && dst_dtype == NEO_F32) NEO_PC(__half, float);
  else if (src_dtype == NEO_BF16 && dst_dtype == NEO_F32) NEO_PC(__nv_bfloat16, float);
  else if (src_dtype == NEO_F32 && dst_dtype == NEO_F16) NEO_PC(float, __half);
  else if (src_dtype == NEO_F32 && dst_dtype == NEO_BF16) NEO_PC(float, __nv_bfloat16);
  else if (src_dtype == NEO_F16 && dst_dtype == NEO_F16) NEO_PC(__half, __half);
  else if (src_dtype == NEO_BF16 && dst_dtype == NEO_BF16) NEO_PC(__nv_bfloat16, __nv_bfloat16);
  else if (src_dtype == NEO_F64 && dst_dtype == NEO_F64) NEO_PC(double, double);
  else return fail(NEO_E_ARG, "copy_pieces: unsupported dtype pair");
#undef NEO_PC
  return check_launch("copy_pieces");
}

int neo_copy_chunks(int64_t rows, const neo_chunk* chunks, int32_t num_chunks, int32_t src_dtype,
                    int32_t dst_dtype, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (rows < 0 || num_chunks < 0) return fail(NEO_E_ARG, "copy_chunks: negative size");
  if (rows == 0 || num_chunks == 0) return NEO_OK;
  if (!chunks) return fail(NEO_E_ARG, "copy_chunks: null chunk table");
  const int64_t blocks = (rows + 7) / 8;
  if (blocks > INT_MAX) return fail(NEO_E_ARG, "copy_chunks: too many rows");
  const unsigned g = (unsigned)blocks;
#define NEO_CC(S, D) copy_chunks_kernel<S, D><<<g, 256, 0, s>>>(rows, chunks, num_chunks)
  if (src_dtype == NEO_F32 && dst_dtype == NEO_F32) NEO_CC(float, float);
  else if (src_dtype == NEO_F16 && dst_dtype == NEO_F32) NEO_CC(__half, float);
  else if (src_dtype == NEO_BF16 && dst_dtype == NEO_F32) NEO_CC(__nv_bfloat16, float);
  else if (src_dtype == NEO_F32 && dst_dtype == NEO_F16) NEO_CC(float, __half);
  else if (src_dtype == NEO_F32 && dst_dtype == NEO_BF16) NEO_CC(float, __nv_bfloat16);
  else if (src_dtype == NEO_F16 && dst_dtype == NEO_F16) NEO_CC(__half, __half);
  else if (src_dtype == NEO_BF16 && dst_dtype == NEO_BF16) NEO_CC(__nv_bfloat16, __nv_bfloat16);
  else return fail(NEO_E_ARG, "copy_chunks: unsupported dtype pair (16-bit / 32-bit floats)");
#undef NEO_CC
  return check_launch("copy_chunks");
}

int neo_check_indices(int32_t num_tables, int64_t batch, const int64_t* rows, const int64_t* offsets,
                      const void* indices, int32_t index_dtype, neo_error* err, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (num_tables < 0 || batch < 0) return fail(NEO_E_ARG, "check_indices: negative size");
  if (num_tables > 65535) return fail(NEO_E_ARG, "check_indices: more than 65535 tables in one call");
  if (num_tables == 0 || batch == 0 || !err) return NEO_OK;
  const dim3 grid(64, (unsigned)num_tables);
  if (index_dtype == NEO_I32)
    check_indices_kernel<int32_t><<<grid, 256, 0, s>>>(num_tables, batch, rows, offsets, (const int32_t*)indices,
                                                       err);
  else
    check_indices_kernel<int64_t><<<grid, 256, 0, s>>>(num_tables, batch, rows, offsets, (const int64_t*)indices,
                                                       err);
  int rc = check_launch("check_indices");
  if (rc) return rc;
  launch_error_finalize(err, indices, index_dtype, offsets, batch, num_tables, s);
  return check_launch("check_indices(finalize)");
}

int neo_gather_blocks(int32_t n, const uint64_t* src_ptrs, const int64_t* counts,
                      const int64_t* dst_offsets, void* dst, int32_t elem_bytes, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n < 0) return fail(NEO_E_ARG, "gather_blocks: negative count");
  if (n == 0) return NEO_OK;
  const dim3 grid((unsigned)n, 4);
  if (elem_bytes == 4)
    gather_blocks_kernel<int32_t><<<grid, 256, 0, s>>>(n, src_ptrs, counts, dst_offsets, (int32_t*)dst);
  else if (elem_bytes == 8)
    gather_blocks_kernel<int64_t><<<grid, 256, 0, s>>>(n, src_ptrs, counts, dst_offsets, (int64_t*)dst);
  else
    return fail(NEO_E_ARG, "gather_blocks: elem_bytes must be 4 or 8");
  return check_launch("gather_blocks");
}

int neo_cast(int64_t n, const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype,
             void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n < 0) return fail(NEO_E_ARG, "cast: negative size");
  if (n == 0) return NEO_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
#define NEO_CAST(S, D) cast_kernel<S, D><<<grid, 256, 0, s>>>(n, (const S*)src, (D*)dst)
  if (src_dtype == NEO_F32 && dst_dtype == NEO_F16) NEO_CAST(float, __half);
  else if (src_dtype == NEO_F32 && dst_dtype == NEO_BF16) NEO_CAST(float, __nv_bfloat16);
  else if (src_dtype == NEO_F16 && dst_dtype == NEO_F32) NEO_CAST(__half, float);
  else if (src_dtype == NEO_BF16 && dst_dtype == NEO_F32) NEO_CAST(__nv_bfloat16, float);
  else if (src_dtype == NEO_F64 && dst_dtype == NEO_F32) NEO_CAST(double, float);
  else if (src_dtype == NEO_F64 && dst_dtype == NEO_F16) NEO_CAST(double, __half);
  else if (src_dtype == NEO_F64 && dst_dtype == NEO_BF16) NEO_CAST(double, __nv_bfloat16);
  else if (src_dtype == NEO_F32 && dst_dtype == NEO_F64) NEO_CAST(float, double);
  else if (src_dtype == NEO_F16 && dst_dtype == NEO_F64) NEO_CAST(__half, double);
  else if (src_dtype == NEO_BF16 && dst_dtype == NEO_F64) NEO_CAST(__nv_bfloat16, double);
  else return fail(NEO_E_ARG, "cast: unsupported dtype pair");
#undef NEO_CAST
  return check_launch("cast");
}

int neo_fp16_roundtrip(int64_t n, double* x, uint8_t* overflow, int32_t* nonfinite, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n < 0) return fail(NEO_E_ARG, "fp16_roundtrip: negative size");
  if (n == 0) return NEO_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  fp16_roundtrip_kernel<<<grid, 256, 0, s>>>(n, x, overflow, nonfinite);
  return check_launch("fp16_roundtrip");
}

int neo_apply_row_updates(int64_t n, const int64_t* ids, const void* grads, int32_t dim,
                          void* weight, int32_t weight_dtype, void* moment, int32_t optim,
                          double lr, double eps, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n < 0 || dim < 1) return fail(NEO_E_ARG, "apply_row_updates: bad sizes");
  if (optim != NEO_OPT_SGD && optim != NEO_OPT_ROWWISE_ADAGRAD && optim != NEO_OPT_ADAGRAD)
    return fail(NEO_E_ARG, "cfg.kind: unknown optimizer");
  if (!(lr > 0)) return fail(NEO_E_ARG, "lr: must be > 0");
  if (eps < 0) return fail(NEO_E_ARG, "eps: must be >= 0");
  if (optim != NEO_OPT_SGD && !moment) return fail(NEO_E_ARG, "moment: state required");
  if (n == 0) return NEO_OK;
  const unsigned grid = (unsigned)((n + 7) / 8);
  if (weight_dtype == NEO_F64) {
    const size_t smem = 8 * (size_t)dim * sizeof(double);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(apply_rows_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_rows_kernel<double><<<grid, 256, smem, s>>>(n, ids, grads, dim, (double*)weight, moment,
                                                      optim, lr, eps);
  } else if (weight_dtype == NEO_F32) {
    const size_t smem = 8 * (size_t)dim * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(apply_rows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_rows_kernel<float><<<grid, 256, smem, s>>>(n, ids, grads, dim, (float*)weight, moment,
                                                     optim, lr, eps);
  } else if (weight_dtype == NEO_F16) {
    const size_t smem = 8 * (size_t)dim * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(apply_rows_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_rows_kernel<__half><<<grid, 256, smem, s>>>(n, ids, grads, dim, (__half*)weight, moment,
                                                      optim, lr, eps);
  } else {
    return fail(NEO_E_ARG, "apply_row_updates: weight dtype must be F32, F16 or F64");
  }
  return check_launch("apply_row_updates");
}

}  // extern "C"
