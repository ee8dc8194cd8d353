// TBE backward fused with the sparse optimizer.
//
// Reference semantics:
//   embedding.py:175-192 backward_sort_aggregate — ids = unique(indices)
//     ascending; grads[r] = sum over r's occurrences (duplicates counted per
//     occurrence) of upstream[sample], summed in buffer order (np.add.at).
//   embedding.py:212-232 apply_rowwise_adagrad — rows with an identically
//     zero gradient are skipped; m_r += mean_j g_rj^2 (numpy pairwise sum);
//     w_rj -= (lr * g_rj) / (sqrt(m_r) + eps).
//   embedding.py:235-254 apply_adagrad / apply_sgd; embedding.py:270-281
//     fused_backward_update = aggregate, then exactly ONE optimizer
//     application per touched row.
//
// B200 mapping (one launch sequence for all T tables of a group):
//   1. key build: warp per bag writes (key = row_offsets[t] + id, bag) pairs
//      for its occurrences (coalesced), range-checking ids;
//   2. stable LSD radix sort of the pairs on ceil(log2(total_rows+1)) bits
//      (keys are table-major, so each table's rows are contiguous and each
//      table's upstream slice stays L2-resident while its rows are updated);
//   3. segment heads (key[i] != key[i-1]) compacted into segment starts;
//   4. persistent segment kernel: one warp per touched row sums the upstream
//      rows of its occurrences in sorted (= buffer) order into a warp-private
//      shared-memory row, then applies the optimizer to the weight row and
//      its moment in place.  No dense gradient is ever materialised.
// F64 tables run the identical sequence with f64 accumulation, numpy's
// pairwise order for the row mean and no FMA contraction, so results are
// bit-identical to the reference.
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include <cuda.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "common.cuh"
#include "optim.cuh"
#include "bwd_common.cuh"

namespace neo {

constexpr int kBwdWarps = 8;
constexpr int kBwdUnroll = 8;


static inline int key_bits_for(int64_t total_rows) {
  // sentinel key == total_rows marks an invalid id; it must be representable
  int bits = 1;
  while (bits < 64 && (uint64_t(1) << bits) <= (uint64_t)total_rows) ++bits;
  return bits;
}

// ---------------------------------------------------------------------------
// 1. key build

template <typename Idx, typename Key>
__global__ void __launch_bounds__(256)
build_keys_kernel(int32_t T, int64_t B, const int64_t* __restrict__ row_offsets,
                  const Idx* __restrict__ indices, const int64_t* __restrict__ offsets,
                  Key* __restrict__ keys, int32_t* __restrict__ bags, Key sentinel,
                  neo_error* err) {
  // persistent warps, 4 consecutive bags per step: their ids form one
  // contiguous range walked with independent (coalesced) loads
  constexpr int kBags = 4;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int64_t nb = (int64_t)T * B;
  const int64_t base0 = offsets[0];
  for (int64_t b0 = ((int64_t)blockIdx.x * 8 + warp) * kBags; b0 < nb; b0 += (int64_t)gridDim.x * 8 * kBags) {
    const int n = (int)min64(kBags, nb - b0);
    const int64_t o = lane <= n ? offsets[b0 + lane] : 0;
    const int64_t start = __shfl_sync(0xffffffffu, o, 0), end = __shfl_sync(0xffffffffu, o, n);
    const int64_t o1 = n > 1 ? __shfl_sync(0xffffffffu, o, 1) : end;
    const int64_t o2 = n > 2 ? __shfl_sync(0xffffffffu, o, 2) : end;
    const int64_t o3 = n > 3 ? __shfl_sync(0xffffffffu, o, 3) : end;
    const int32_t t0 = (int32_t)(b0 / B);
    for (int64_t p = start + lane; p < end; p += kWarp) {
      const int64_t bag = b0 + (p >= o1) + (p >= o2) + (p >= o3);
      int32_t t = t0;
      while (bag >= (int64_t)(t + 1) * B) ++t;
      const int64_t rbase = row_offsets[t];
      const int64_t H = row_offsets[t + 1] - rbase;
      const int64_t v = (int64_t)indices[p];
      Key k;
      if (v < 0 || v >= H) {
        record_bad_index(err, p);
        k = sentinel;
      } else {
        k = (Key)(rbase + v);
      }
      keys[p - base0] = k;
      bags[p - base0] = (int32_t)bag;
    }
  }
}

// 3. segment heads
template <typename Key>
struct HeadFlag {
  const Key* keys;
  __device__ __forceinline__ bool operator()(const int32_t& i) const {
    return i == 0 || keys[i] != keys[i - 1];
  }
};

// ---------------------------------------------------------------------------
// 4. segment reduce + optimizer



// aggregate the segment's upstream rows into g (warp-private smem row)
template <typename G, typename Acc, int VEC>
__device__ __forceinline__ void aggregate_row(const SegParams& p, const G* __restrict__ grad,
                                              int32_t t, int32_t D, int32_t doff, int64_t s0,
                                              int64_t s1, Acc* g, int lane) {
  constexpr bool kExact = sizeof(Acc) == 8;
  constexpr int U = kBwdUnroll;
  const int chunks = D / VEC;
  const int S = kExact ? kWarp : subwarp_width(chunks);
  const int R = kWarp / S;
  const int sub = lane / S, sl = lane % S;
  const int64_t bag_base = (int64_t)t * p.B;
  for (int cbase = 0; cbase < chunks; cbase += S) {
    const int ch = cbase + sl;
    const bool col_live = ch < chunks;
    Acc acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = Acc(0);
    for (int64_t j0 = s0; j0 < s1; j0 += kWarp) {
      const int m = (int)min64(kWarp, s1 - j0);
      const int32_t mybag = lane < m ? p.bags[j0 + lane] : 0;
      for (int jj = 0; jj < m; jj += R * U) {
        Vec<G, VEC> v[U];
        bool live[U];
        Acc scale[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = jj + u * R + sub;
          const int32_t bg = __shfl_sync(0xffffffffu, mybag, r < m ? r : 0);
          live[u] = r < m;
          const int64_t b = (int64_t)bg - bag_base;
          scale[u] = Acc(1);
          if (p.pooling == NEO_POOL_MEAN && live[u]) {
            const int64_t len = p.offsets[bg + 1] - p.offsets[bg];
            scale[u] = Acc(1) / (Acc)len;
          }
          if (live[u] && col_live) {
            v[u] = ld_vec<G, VEC>(grad + b * p.grad_stride + doff + (int64_t)ch * VEC);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) v[u].v[e] = G(0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (kExact && !live[u]) continue;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            Acc x = to_acc<Acc>(v[u].v[e]);
            if (p.pooling == NEO_POOL_MEAN) x = x * scale[u];
            acc[e] += x;
          }
        }
      }
    }
    if (!kExact) {
      for (int o = S; o < kWarp; o <<= 1) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
      }
    }
    if (sub == 0 && col_live) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) g[ch * VEC + e] = acc[e];
    }
  }
  __syncwarp();
}

template <typename W, typename G, typename Key>
__global__ void __launch_bounds__(kBwdWarps * kWarp)
tbe_segment_kernel(SegParams p) {
  constexpr bool kExact = sizeof(W) == 8;
  using Acc = typename std::conditional<kExact, double, float>::type;
  constexpr int kVec = 16 / sizeof(W);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  Acc* g = reinterpret_cast<Acc*>(smem_raw) + (size_t)warp * p.max_dim;
  const G* grad = reinterpret_cast<const G*>(p.grad);
  const Key* keys = reinterpret_cast<const Key*>(p.keys);
  const int64_t U = *p.num_segs;
  const int64_t nwarps = (int64_t)gridDim.x * kBwdWarps;
  for (int64_t seg = (int64_t)blockIdx.x * kBwdWarps + warp; seg < U; seg += nwarps) {
    const int64_t s0 = p.seg_starts[seg];
    const int64_t s1 = seg + 1 < U ? (int64_t)p.seg_starts[seg + 1] : p.N;
    const uint64_t key = (uint64_t)keys[s0];
    if (key >= (uint64_t)p.total_rows) continue;  // invalid ids sort last
    const int32_t t = (int32_t)(p.bags[s0] / p.B);
    const int64_t row = (int64_t)key - p.row_offsets[t];
    const int32_t doff = p.dim_offsets[t];
    const int32_t D = p.dim_offsets[t + 1] - doff;
    W* wbase = reinterpret_cast<W*>(p.weights[t]);
    Acc* mbase = p.moments ? reinterpret_cast<Acc*>(p.moments[t]) : nullptr;
    RowPrefetch<W, Acc> pf;
    prefetch_row<W, Acc>(p.mode == NEO_BWD_UPDATE, wbase, mbase, p.optim, row, D, lane, pf);
    const bool vec = (D % kVec) == 0 && (doff % kVec) == 0 && (p.grad_stride % kVec) == 0 &&
                     (reinterpret_cast<uintptr_t>(grad) % min(16, (int)sizeof(G) * kVec)) == 0;
    if (vec) aggregate_row<G, Acc, kVec>(p, grad, t, D, doff, s0, s1, g, lane);
    else aggregate_row<G, Acc, 1>(p, grad, t, D, doff, s0, s1, g, lane);

    if (p.mode == NEO_BWD_UPDATE) {
      update_row<W, Acc>(wbase, mbase, p.optim, p.lr, p.eps, row, D, g, lane, pf);
    } else if (p.mode == NEO_BWD_AGGREGATE) {
      Acc* og = reinterpret_cast<Acc*>(p.out_grads) + seg * p.max_dim;
      for (int j = lane; j < D; j += kWarp) og[j] = g[j];
      if (lane == 0) p.out_ids[seg] = (int64_t)key;
    } else {  // DENSE
      Acc* dg = reinterpret_cast<Acc*>(p.dense_grads[t]) + row * D;
      for (int j = lane; j < D; j += kWarp) dg[j] = g[j];
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// 4'. fast path: streamed segment walk (f32/f16 tables, rows of <= 32 16-byte
// vectors, SUM pooling, UPDATE mode).
//
// Each warp owns a chunk of 32 consecutive sorted (key, bag) entries and
// every segment that STARTS in it (walking past the chunk end for the last
// one); segment boundaries come from one coalesced key load + a shuffle.  The
// warp runs two cursors over that entry stream: a producer LEAD entries ahead
// issues cp.async copies of each entry's upstream row (and, at a segment
// head, of the segment's weight row and moment) into per-warp shared-memory
// rings, one commit group per entry; the consumer waits for the group of its
// entry, accumulates the row, and at the next head applies the optimizer to
// the staged weight row and stores it.  Every lane only ever reads the bytes
// it copied itself, so no warp barrier guards the rings, and LEAD rows per
// warp stay in flight without occupying registers.  Accumulation order is the
// sorted (= buffer) order.

constexpr int kLead = 7;               // entries in flight per warp
constexpr int kGRing = kLead + 1;      // upstream-row slots
constexpr int kWRing = kLead + 3;      // open-segment slots (>= kLead + 2)
constexpr int kStreamWarps = 4;        // warps per CTA

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
// L2 residency control: the upstream slice of the table being updated is
// re-read ~L times (once per occurrence) and must stay in L2, while weight
// rows, moments and the sorted (key, bag) stream are touched once.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async_hint(void* smem, const void* gmem, int bytes, uint64_t pol) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "l"(pol));
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "l"(pol));
  else
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void st_v4_hint(void* gmem, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(gmem), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }


template <typename W, typename G, int VPL>
struct alignas(16) StreamSmem {
  static constexpr int kVec = 16 / sizeof(W);
  static constexpr int kGBytes = kVec * sizeof(G);  // upstream bytes per lane per row vector
  unsigned char g[kGRing][kWarp][kGBytes * VPL];
  unsigned char w[kWRing][kWarp][16 * VPL];
  float mr[kWRing];               // row-wise moment
};

// Lane-parallel metadata of a 32-entry window: lane l describes entry base+l.
struct Window {
  int64_t base;
  uint64_t key;
  unsigned heads;   // bit l: entry base+l starts a segment
  unsigned live;    // bit l: entry is a valid row id (< total_rows, < N)
  uint32_t gofs;    // upstream element offset of this lane's entry (row * stride + column offset)
  uint64_t wptr;    // weight row
  uint64_t mptr;    // moment (row-wise scalar / element-wise row)
  int32_t D;        // table dim of this lane's entry
  int32_t vec;      // 16-byte vector path usable for this entry's table
  int32_t tt;       // table of this lane's entry (-1: invalid)
  uint32_t grow;    // upstream row (bag within the table)
  int32_t dcol;     // upstream column offset of the table
};

template <typename W, typename G, typename Key, int OPT>
__device__ __forceinline__ void load_window(const SegParams& p, int64_t base, uint64_t prev_key, int lane,
                                            Window& w) {
  constexpr int kVec = 16 / sizeof(W);
  const unsigned full = 0xffffffffu;
  const Key* keys = reinterpret_cast<const Key*>(p.keys);
  const int64_t j = base + lane;
  w.base = base;
  const bool in = j < p.N;
  w.key = in ? (uint64_t)__ldcs(keys + j) : ~0ull;
  const int32_t bag = in ? __ldcs(p.bags + j) : 0;
  uint64_t pv = __shfl_up_sync(full, w.key, 1);
  if (lane == 0) pv = prev_key;
  w.heads = __ballot_sync(full, w.key != pv);
  const bool ok = in && w.key < (uint64_t)p.total_rows;
  w.live = __ballot_sync(full, ok);
  w.gofs = 0;
  w.wptr = w.mptr = 0;
  w.D = 0;
  w.vec = 0;
  w.tt = -1;
  w.grow = 0;
  w.dcol = 0;
  if (ok) {
    const int32_t t = bag / (int32_t)p.B;
    w.tt = t;
    w.grow = (uint32_t)(bag - t * (int32_t)p.B);
    w.dcol = p.dim_offsets[t];
    const int64_t row = (int64_t)w.key - p.row_offsets[t];
    const int32_t doff = p.dim_offsets[t];
    const int32_t D = p.dim_offsets[t + 1] - doff;
    const G* grad = reinterpret_cast<const G*>(p.grad);
    const W* wbase = reinterpret_cast<const W*>(p.weights[t]);
    w.D = D;
    w.vec = (D % kVec) == 0 && aligned16(wbase) && (doff % kVec) == 0 && (p.grad_stride % kVec) == 0 &&
            (reinterpret_cast<uintptr_t>(grad) % min(16, (int)(sizeof(G) * kVec))) == 0;
    w.gofs = (uint32_t)(((int64_t)bag - (int64_t)t * p.B) * p.grad_stride + doff);
    w.wptr = reinterpret_cast<uint64_t>(wbase + row * D);
    if (OPT == NEO_OPT_ROWWISE_ADAGRAD || OPT == NEO_OPT_ADAGRAD) {
      float* mb = reinterpret_cast<float*>(p.moments[t]);
      w.mptr = reinterpret_cast<uint64_t>(OPT == NEO_OPT_ROWWISE_ADAGRAD ? mb + row : mb + row * D);
    }
  }
}

constexpr int kChunk = 128;  // sorted entries owned per warp task (4 windows)

// element index of (vector v of lane, element e): the vector path gives lane
// contiguous 16-byte vectors lane, lane+32, ...; the scalar path strides by 32
__device__ __forceinline__ int elem_index(bool vec, int lane, int v, int e, int kVec) {
  return vec ? (lane + v * kWarp) * kVec + e : lane + (v * kVec + e) * kWarp;
}

// Hot rows (skewed ids): a 128-entry chunk whose entries all belong to ONE
// row (no segment boundary inside, and it does not start the row) gets its
// upstream partial sum precomputed here, in entry order, by its own warp.
// The streamed kernel then folds such partials into the row's gradient in
// chunk order instead of walking the row's occurrences on a single warp, so
// a row touched 1e5 times costs ~1e3 partial loads, not 1e5 serial gathers.
template <typename W, typename G, typename Key, int VPL>
__global__ void __launch_bounds__(256)
hot_chunk_kernel(SegParams p) {
  constexpr int kVec = 16 / sizeof(W);
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const Key* keys = reinterpret_cast<const Key*>(p.keys);
  const G* grad = reinterpret_cast<const G*>(p.grad);
  const int64_t nchunks = (p.N + kChunk - 1) / kChunk;
  for (int64_t c = (int64_t)blockIdx.x * 8 + warp; c < nchunks; c += (int64_t)gridDim.x * 8) {
    const int64_t c0 = c * kChunk;
    bool bf = false;
    if (c0 > 0 && c0 + kChunk <= p.N) {
      const uint64_t k0 = (uint64_t)keys[c0];
      bf = k0 < (uint64_t)p.total_rows && (uint64_t)keys[c0 - 1] == k0 && (uint64_t)keys[c0 + kChunk - 1] == k0;
    }
    int32_t slot = -1;
    if (bf) {
      unsigned sl = 0;
      if (lane == 0) sl = atomicAdd(p.pool_counter, 1u);
      sl = __shfl_sync(full, sl, 0);
      slot = sl < (unsigned)p.pool_cap ? (int32_t)sl : -1;
    }
    if (slot >= 0) {
      const int32_t t = p.bags[c0] / (int32_t)p.B;
      const int32_t doff = p.dim_offsets[t];
      const int32_t D = p.dim_offsets[t + 1] - doff;
      const bool vec = (D % kVec) == 0 && aligned16(reinterpret_cast<const void*>(p.weights[t])) &&
                       (doff % kVec) == 0 && (p.grad_stride % kVec) == 0 &&
                       (reinterpret_cast<uintptr_t>(grad) % min(16, (int)(sizeof(G) * kVec))) == 0;
      float acc[VPL][kVec];
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int e = 0; e < kVec; ++e) acc[v][e] = 0.f;
      for (int q = 0; q < kChunk; q += kWarp) {
        const int32_t qb = p.bags[c0 + q + lane];
#pragma unroll 4
        for (int e2 = 0; e2 < kWarp; ++e2) {
          const int32_t bag = __shfl_sync(full, qb, e2);
          const G* src = grad + ((int64_t)bag - (int64_t)t * p.B) * p.grad_stride + doff;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if (vec) {
              if ((lane + v * kWarp) * kVec < D) {
                Vec<G, kVec> x = ld_vec<G, kVec>(src + (lane + v * kWarp) * kVec);
#pragma unroll
                for (int e = 0; e < kVec; ++e) acc[v][e] += Elem<G>::to_f(x.v[e]);
              }
            } else {
#pragma unroll
              for (int e = 0; e < kVec; ++e) {
                const int j = lane + (v * kVec + e) * kWarp;
                if (j < D) acc[v][e] += Elem<G>::to_f(src[j]);
              }
            }
          }
        }
      }
      float* dst = p.pool + (int64_t)slot * p.max_dim;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int e = 0; e < kVec; ++e) {
          const int j = elem_index(vec, lane, v, e, kVec);
          if (j < D) dst[j] = acc[v][e];
        }
    }
    if (lane == 0) p.chunk_slot[c] = slot;
  }
}


template <typename W, typename G, typename Key, int OPT, bool FULL, int VPL>
__global__ void __launch_bounds__(kStreamWarps * kWarp, VPL == 1 ? 6 : 3)
tbe_stream_update_kernel(SegParams p) {
  using SM = StreamSmem<W, G, VPL>;
  constexpr int kVec = SM::kVec;
  constexpr int kGB = SM::kGBytes;
  const unsigned full = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  SM& sm = reinterpret_cast<SM*>(smem_raw)[warp];
  const Key* keys = reinterpret_cast<const Key*>(p.keys);
  const int64_t N = p.N;
  const int64_t nchunks = (N + kChunk - 1) / kChunk;
  const float lr = (float)p.lr, eps = (float)p.eps;
  const G* gbase = reinterpret_cast<const G*>(p.grad);
#ifndef NEO_L2_HINTS
#define NEO_L2_HINTS 2
#endif
  // 0: no hints; 1: evict_first weights + evict_last upstream; 2: evict_last upstream only
  const uint64_t pol_stream = NEO_L2_HINTS == 1 ? l2_evict_first() : l2_evict_normal();
  const uint64_t pol_keep = NEO_L2_HINTS == 0 ? l2_evict_normal() : l2_evict_last();

  // Dynamic chunk scheduling: warps claim chunks from a global counter (one
  // claim in flight ahead), so all warps stay on the same frontier of the
  // sorted stream and the upstream slice they share stays L2-resident (a
  // static grid stride lets warps drift apart over hundreds of chunks).
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(p.chunk_counter);
  __shared__ long long s_claim[kStreamWarps];
  for (;;) {
    __syncwarp();
    if (lane == 0) s_claim[warp] = (long long)atomicAdd(counter, 1ull);
    __syncwarp();
    const int64_t chunk = s_claim[warp];
    if (chunk >= nchunks) break;
    const int64_t c0 = chunk * kChunk;
    // first segment start at or after c0 (scan the chunk's windows)
    Window pw;
    uint64_t prev = c0 > 0 ? (uint64_t)keys[c0 - 1] : ~0ull;
    int e0 = -1;
    for (int k = 0; k < kChunk / kWarp; ++k) {
      if (c0 + k * kWarp >= N) break;
      load_window<W, G, Key, OPT>(p, c0 + k * kWarp, prev, lane, pw);
      if (pw.heads) {
        e0 = k * kWarp + __ffs(pw.heads) - 1;
        break;
      }
      prev = __shfl_sync(full, pw.key, kWarp - 1);
    }
    if (e0 < 0 || !((pw.live >> (e0 & (kWarp - 1))) & 1u)) continue;
    Window cw = pw;  // the consumer's window (the producer's, or the one before it)
    // producer: runs kLead entries ahead, issuing one cp.async group per entry
    int pe = e0;
    int pend = -1;  // range end once known: first head at/after c0+kChunk, first invalid entry, or N
    int64_t cont_chunk = -1;  // first hot chunk the last segment continues into
    int pslot = -1;
    int pD = 0, pvec = 0;

    auto produce = [&]() {
      if (pend < 0) {
        int l = pe - (int)(pw.base - c0);
        if (l == kWarp) {  // slide to the next window
          const int64_t nb = pw.base + kWarp;
#ifndef NEO_HOT_CHUNKS
#define NEO_HOT_CHUNKS 1
#endif
          if (NEO_HOT_CHUNKS && nb % kChunk == 0 && nb < p.N && p.chunk_slot[nb / kChunk] >= 0) {
            // the row continues through a hot chunk: its partials are folded in below
            pend = pe;
            cont_chunk = nb / kChunk;
            cp_commit();
            return;
          }
          const uint64_t last = __shfl_sync(full, pw.key, kWarp - 1);
          load_window<W, G, Key, OPT>(p, nb, last, lane, pw);
          l = 0;
        }
        const bool head = (pw.heads >> l) & 1u;
        if (!((pw.live >> l) & 1u) || (head && pe >= kChunk)) {
          pend = pe;
        } else {
          if (head) {  // new segment: stage its weight row (+ row-wise moment)
            pslot = pslot + 1 == kWRing ? 0 : pslot + 1;
            if (!FULL) {
              pD = __shfl_sync(full, pw.D, l);
              pvec = __shfl_sync(full, pw.vec, l);
            }
            const W* wrow = reinterpret_cast<const W*>(__shfl_sync(full, pw.wptr, l));
            if (FULL || pvec) {
#pragma unroll
              for (int v = 0; v < VPL; ++v)
                if (FULL || (lane + v * kWarp) * kVec < pD)
                  cp_async_hint(&sm.w[pslot][lane][16 * v], wrow + (lane + v * kWarp) * kVec, 16, pol_stream);
            } else {  // unaligned table: synchronous strided staging (own lane's slice)
              W* ws = reinterpret_cast<W*>(&sm.w[pslot][lane][0]);
#pragma unroll
              for (int e = 0; e < kVec * VPL; ++e) {
                const int j = lane + e * kWarp;
                ws[e] = j < pD ? wrow[j] : W(0);
              }
            }
            if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
              const uint64_t mp = __shfl_sync(full, pw.mptr, l);
              if (lane == 0) cp_async_hint(&sm.mr[pslot], reinterpret_cast<const float*>(mp), 4, pol_stream);
            }
          }
          const int gs = pe & (kGRing - 1);
          const G* grow = gbase + __shfl_sync(full, pw.gofs, l);
          if (FULL || pvec) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              if (FULL || (lane + v * kWarp) * kVec < pD) {
                const G* src = grow + (lane + v * kWarp) * kVec;
                unsigned char* dst = &sm.g[gs][lane][kGB * v];
                if constexpr (kGB == 32) {
                  cp_async_hint(dst, src, 16, pol_keep);
                  cp_async_hint(dst + 16, src + kVec / 2, 16, pol_keep);
                } else {
                  cp_async_hint(dst, src, kGB, pol_keep);
                }
              }
            }
          } else {
            G* gsm = reinterpret_cast<G*>(&sm.g[gs][lane][0]);
#pragma unroll
            for (int e = 0; e < kVec * VPL; ++e) {
              const int j = lane + e * kWarp;
              gsm[e] = j < pD ? grow[j] : G(0);
            }
          }
          ++pe;
        }
      }
      cp_commit();
    };

    // consumer state: current segment (registers) and its accumulator
    float acc[VPL * kVec];
#pragma unroll
    for (int e = 0; e < VPL * kVec; ++e) acc[e] = 0.f;
    int cslot = -1;
    uint64_t cw_w = 0, cw_m = 0;
    int cD = 0, cvec = 0;
    float cinvD = 0.f;
    uint64_t cseg_key = 0;

    auto live_at = [&](int v, int e) -> bool {  // element (v, e) of this lane is inside the row
      if (FULL) return true;
      return elem_index(cvec, lane, v, e, kVec) < cD;
    };

    auto finalize = [&]() {  // exactly one optimizer step for the row (embedding.py:212-254)
      if (!FULL) {
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
          for (int e = 0; e < kVec; ++e)
            if (!live_at(v, e)) acc[v * kVec + e] = 0.f;
      }
      bool nz = false;
#pragma unroll
      for (int e = 0; e < VPL * kVec; ++e) nz |= acc[e] != 0.f;
      if (OPT == NEO_OPT_SGD || __any_sync(full, nz)) {
        const W* wsm = reinterpret_cast<const W*>(&sm.w[cslot][lane][0]);
        float scale = lr;
        if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
          float ss = 0.f;
#pragma unroll
          for (int e = 0; e < VPL * kVec; ++e) ss += acc[e] * acc[e];
          ss = warp_sum(ss);
          const float m = __shfl_sync(full, sm.mr[cslot], 0) + ss * cinvD;
          if (lane == 0) *reinterpret_cast<float*>(cw_m) = m;
          scale = __fdividef(lr, __fsqrt_rn(m) + eps);
        }
        W* wrow = reinterpret_cast<W*>(cw_w);
        float* mrow = reinterpret_cast<float*>(cw_m);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          W out[kVec];
          float mo[kVec];
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            const float w = Elem<W>::to_f(wsm[v * kVec + e]);
            const float a = acc[v * kVec + e];
            if (OPT == NEO_OPT_ADAGRAD) {  // element-wise state read here (not staged)
              const int j = elem_index(cvec, lane, v, e, kVec);
              const float mj = (FULL || j < cD ? mrow[j] : 0.f) + a * a;
              mo[e] = mj;
              out[e] = Elem<W>::from_f(w - __fdividef(lr * a, __fsqrt_rn(mj) + eps));
            } else {
              out[e] = Elem<W>::from_f(w - a * scale);
            }
          }
          if (FULL || cvec) {
            if (FULL || (lane + v * kWarp) * kVec < cD) {
              Vec<W, kVec> o;
#pragma unroll
              for (int e = 0; e < kVec; ++e) o.v[e] = out[e];
              st_v4_hint(wrow + (lane + v * kWarp) * kVec, *reinterpret_cast<const uint4*>(&o), pol_stream);
              if (OPT == NEO_OPT_ADAGRAD) {
#pragma unroll
                for (int e = 0; e < kVec; ++e) mrow[(lane + v * kWarp) * kVec + e] = mo[e];
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
              const int j = lane + (v * kVec + e) * kWarp;
              if (j < cD) {
                wrow[j] = out[e];
                if (OPT == NEO_OPT_ADAGRAD) mrow[j] = mo[e];
              }
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < VPL * kVec; ++e) acc[e] = 0.f;
    };

#pragma unroll 1
    for (int i = 0; i < kLead; ++i) produce();  // fill the pipeline
    int ce = e0;
#pragma unroll 1
    while (true) {
      const int wstart = (int)(cw.base - c0);
      bool stop = false;
#pragma unroll 1
      for (; ce < wstart + kWarp; ++ce) {
        produce();
        if (pend >= 0 && ce >= pend) {
          stop = true;
          break;
        }
        cp_wait<kLead>();
        const int l = ce - wstart;
        if ((cw.heads >> l) & 1u) {
          if (cslot >= 0) finalize();
          cslot = cslot + 1 == kWRing ? 0 : cslot + 1;
          cw_w = __shfl_sync(full, cw.wptr, l);
          cseg_key = __shfl_sync(full, cw.key, l);
          if (OPT != NEO_OPT_SGD) cw_m = __shfl_sync(full, cw.mptr, l);
          if (FULL) {
            cD = kWarp * kVec * VPL;
            cvec = 1;
            cinvD = 1.0f / (float)(kWarp * kVec * VPL);
          } else {
            cD = __shfl_sync(full, cw.D, l);
            cvec = __shfl_sync(full, cw.vec, l);
            cinvD = __frcp_rn((float)cD);
          }
        }
        const G* gsm = reinterpret_cast<const G*>(&sm.g[ce & (kGRing - 1)][lane][0]);
#pragma unroll
        for (int e = 0; e < VPL * kVec; ++e) acc[e] += Elem<G>::to_f(gsm[e]);
      }
      if (stop || (pend >= 0 && ce >= pend)) break;  // range may end exactly at a window edge
      cw = pw;  // the producer is already in the next window
    }
    if (cont_chunk >= 0 && cslot >= 0) {
      // fold the hot chunks' partials (chunk order), then walk the row's tail
      int64_t c = cont_chunk;
      const int64_t nchunks_all = (N + kChunk - 1) / kChunk;
      for (; c < nchunks_all; ++c) {
        const int32_t slot = p.chunk_slot[c];
        if (slot < 0) break;
        const float* src = p.pool + (int64_t)slot * p.max_dim;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            const int j = elem_index(cvec, lane, v, e, kVec);
            if (j < cD) acc[v * kVec + e] += src[j];
          }
      }
      for (int64_t e0 = c * kChunk; e0 < N; ++e0) {
        if ((uint64_t)keys[e0] != cseg_key) break;
        const int32_t bag = p.bags[e0];
        const int32_t t = bag / (int32_t)p.B;
        const G* src = gbase + ((int64_t)bag - (int64_t)t * p.B) * p.grad_stride + p.dim_offsets[t];
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            const int j = elem_index(cvec, lane, v, e, kVec);
            if (j < cD) acc[v * kVec + e] += Elem<G>::to_f(src[j]);
          }
      }
    }
    if (cslot >= 0) finalize();
    cp_wait<0>();
  }
}

#include "tbe_pipe.cuh"

// backward fast-path variant: the warp-specialised pipeline (default) or the
// single-warp streamed walk (NEO_BWD_VARIANT=stream, kept for A/B runs)
static bool use_pipe_variant() {
  const char* v = std::getenv("NEO_BWD_VARIANT");
  return !(v && std::strcmp(v, "stream") == 0);
}

typedef CUresult (*TensorMapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2D map over the upstream gradient (B rows x grad_stride columns), box = one
// row of `cols` elements: gather4 then stages four upstream rows per instruction
template <typename G>
static bool encode_upstream_map(const SegParams& p, int cols, CUtensorMap* map) {
  static TensorMapEncodeFn enc = [] {
    TensorMapEncodeFn f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (TensorMapEncodeFn) nullptr;
    return f;
  }();
  if (!enc || cols > 256 || (reinterpret_cast<uintptr_t>(p.grad) & 15) || ((p.grad_stride * sizeof(G)) & 15))
    return false;
  const CUtensorMapDataType dt = sizeof(G) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : std::is_same<G, __half>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                  : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  cuuint64_t dims[2] = {(cuuint64_t)p.grad_stride, (cuuint64_t)p.B};
  cuuint64_t strides[1] = {(cuuint64_t)p.grad_stride * sizeof(G)};
  cuuint32_t box[2] = {(cuuint32_t)cols, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(map, dt, 2, const_cast<void*>(p.grad), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

static bool use_pipe_tma() {
  const char* v = std::getenv("NEO_PIPE_TMA");
  return v && std::strcmp(v, "1") == 0;
}

template <typename W, typename G, typename Key, int OPT, int VPL>
static int launch_pipe(SegParams p, cudaStream_t s, int sms) {
  using Cfg = PipeCfg<W, G, OPT, VPL>;
  CUtensorMap gmap;
  std::memset(&gmap, 0, sizeof(gmap));
  p.tma = 0;
  if ((p.flags & NEO_BWD_FLAG_FULL_ROWS) && use_pipe_tma() &&
      encode_upstream_map<G>(p, kWarp * Cfg::kVec * VPL, &gmap))
    p.tma = 1;
  auto kern = tbe_pipe_update_kernel<W, G, Key, OPT, false, VPL>;
  if (p.flags & NEO_BWD_FLAG_FULL_ROWS) kern = tbe_pipe_update_kernel<W, G, Key, OPT, true, VPL>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve pipeline shared memory");
  const int64_t tasks = (p.N + NEO_PIPE_CHUNK - 1) / NEO_PIPE_CHUNK;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 2 * Cfg::P * kWarp, Cfg::kSmem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > (tasks + Cfg::P - 1) / Cfg::P) grid = (tasks + Cfg::P - 1) / Cfg::P;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, 2 * Cfg::P * kWarp, Cfg::kSmem, s>>>(p, gmap);
  return check_launch("neo_tbe_backward(pipe)");
}

// ---------------------------------------------------------------------------
template <typename W, typename G, typename Key, int OPT, int VPL>
static int launch_stream_vpl(const SegParams& p, cudaStream_t s) {
  // guard-free instantiation when every row is exactly 32 lanes x one vector
  auto kern = tbe_stream_update_kernel<W, G, Key, OPT, false, VPL>;
  if constexpr (VPL == 1) {
    if (p.flags & NEO_BWD_FLAG_FULL_ROWS) kern = tbe_stream_update_kernel<W, G, Key, OPT, true, 1>;
  }
  const size_t smem = sizeof(StreamSmem<W, G, VPL>) * kStreamWarps;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve shared memory");
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStreamWarps * kWarp, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t chunks = (p.N + kChunk - 1) / kChunk;
  const int64_t max_blocks = (chunks + kStreamWarps - 1) / kStreamWarps;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > max_blocks) grid = max_blocks;
  if (grid < 1) grid = 1;
  if (cudaMemsetAsync(p.chunk_counter, 0, 2 * sizeof(int64_t), s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: counter reset failed");
  {
    const int64_t hb = (chunks + 7) / 8;
    const unsigned hgrid = (unsigned)(hb < (int64_t)sms * 16 ? (hb > 0 ? hb : 1) : (int64_t)sms * 16);
    hot_chunk_kernel<W, G, Key, VPL><<<hgrid, 256, 0, s>>>(p);
    const int rc = check_launch("neo_tbe_backward(hot chunks)");
    if (rc) return rc;
  }
  if ((p.flags & NEO_BWD_FLAG_ALIGNED) && use_pipe_variant()) return launch_pipe<W, G, Key, OPT, VPL>(p, s, sms);
  kern<<<(unsigned)grid, kStreamWarps * kWarp, smem, s>>>(p);
  return check_launch("neo_tbe_backward(stream)");
}

template <typename W, typename G, typename Key, int OPT>
static int launch_stream_opt(const SegParams& p, cudaStream_t s) {
  // rows of up to 32 lanes x 1 or 2 sixteen-byte vectors
  if (p.max_dim <= kWarp * (16 / (int)sizeof(W))) return launch_stream_vpl<W, G, Key, OPT, 1>(p, s);
  return launch_stream_vpl<W, G, Key, OPT, 2>(p, s);
}

template <typename W, typename G, typename Key>
static int launch_stream(const SegParams& p, cudaStream_t s) {
  switch (p.optim) {
    case NEO_OPT_SGD: return launch_stream_opt<W, G, Key, NEO_OPT_SGD>(p, s);
    case NEO_OPT_ROWWISE_ADAGRAD: return launch_stream_opt<W, G, Key, NEO_OPT_ROWWISE_ADAGRAD>(p, s);
    default: return launch_stream_opt<W, G, Key, NEO_OPT_ADAGRAD>(p, s);
  }
}

// DENSE mode on the pipelined walk (f32 tables): each touched row's
// aggregated gradient is stored into dense_grads[t] (passed as the "weights")
template <typename G, typename Key>
static int launch_dense_pipe(SegParams p, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.weights = p.dense_grads;
  p.moments = nullptr;
  if (cudaMemsetAsync(p.chunk_counter, 0, 2 * sizeof(int64_t), s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: counter reset failed");
  const int64_t chunks = (p.N + kChunk - 1) / kChunk;
  const int64_t hb = (chunks + 7) / 8;
  const unsigned hgrid = (unsigned)(hb < (int64_t)sms * 16 ? (hb > 0 ? hb : 1) : (int64_t)sms * 16);
  const bool wide = p.max_dim > kWarp * 4;
  if (wide) hot_chunk_kernel<float, G, Key, 2><<<hgrid, 256, 0, s>>>(p);
  else hot_chunk_kernel<float, G, Key, 1><<<hgrid, 256, 0, s>>>(p);
  const int rc = check_launch("neo_tbe_backward(hot chunks)");
  if (rc) return rc;
  return wide ? launch_pipe<float, G, Key, NEO_OPT_NONE, 2>(p, s, sms) : launch_pipe<float, G, Key, NEO_OPT_NONE, 1>(p, s, sms);
}

template <typename Key>
__global__ void count_valid_kernel(const Key* keys, const int32_t* seg_starts,
                                   const int64_t* num_segs, int64_t total_rows, int64_t* out) {
  const int64_t U = *num_segs;
  int64_t c = U;
  if (U > 0 && (uint64_t)keys[seg_starts[U - 1]] >= (uint64_t)total_rows) c = U - 1;
  *out = c;
}

// ---------------------------------------------------------------------------

template <typename Key>
static size_t cub_temp_bytes(int64_t N) {
  size_t sort_bytes = 0, sel_bytes = 0;
  cub::DoubleBuffer<Key> kb(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, (int)N, 0, sizeof(Key) * 8);
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::If(nullptr, sel_bytes, it, (int32_t*)nullptr, (int64_t*)nullptr, (int)N,
                        HeadFlag<Key>{nullptr});
  return sort_bytes > sel_bytes ? sort_bytes : sel_bytes;
}

static inline int64_t hot_chunks(int64_t N) { return (N + 127) / 128; }

// PREPARE/APPLY split: which half of the double buffer holds the sorted
// pairs of a prepared workspace (host-side; no device sync)
static std::mutex g_prep_mu;
static std::unordered_map<const void*, int> g_prep_sel;

template <typename Key>
static size_t workspace_for(int64_t N, int64_t max_dim) {
  size_t b = 0;
  b += 2 * align256(sizeof(Key) * N);      // key double buffer
  b += 2 * align256(sizeof(int32_t) * N);  // bag double buffer
  b += align256(sizeof(int32_t) * N);      // segment starts
  b += align256(sizeof(int64_t) * 4);      // segment count, chunk counter, pool counter
  b += align256(sizeof(int32_t) * hot_chunks(N));                       // hot-chunk slots
  b += align256(sizeof(float) * hot_chunks(N) * (max_dim > 0 ? max_dim : 1));  // hot partials
  b += align256(cub_temp_bytes<Key>(N));
  return b;
}

static bool use_wide_keys(int64_t total_rows) { return total_rows >= (int64_t)UINT32_MAX; }

template <typename W, typename G, typename Key>
static int launch_segments(const SegParams& p, cudaStream_t s) {
  using Acc = typename std::conditional<sizeof(W) == 8, double, float>::type;
  const size_t smem = (size_t)kBwdWarps * p.max_dim * sizeof(Acc);
  auto kern = tbe_segment_kernel<W, G, Key>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return fail(NEO_E_ARG, "neo_tbe_backward: max_dim too large for shared memory");
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBwdWarps * kWarp, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t max_blocks = (p.N + kBwdWarps - 1) / kBwdWarps;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > max_blocks) grid = max_blocks;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kBwdWarps * kWarp, smem, s>>>(p);
  return check_launch("neo_tbe_backward(segments)");
}

template <typename Key>
static int run_backward(SegParams p, int32_t weight_dtype, int32_t grad_dtype,
                        const void* indices, int32_t index_dtype, void* workspace,
                        size_t ws_bytes, int64_t* out_count, neo_error* err, cudaStream_t s) {
  const int64_t N = p.N;
  if (ws_bytes < workspace_for<Key>(N, p.max_dim))
    return fail(NEO_E_ARG, "neo_tbe_backward: workspace too small");
  unsigned char* w = static_cast<unsigned char*>(workspace);
  Key* k0 = reinterpret_cast<Key*>(w);
  w += align256(sizeof(Key) * N);
  Key* k1 = reinterpret_cast<Key*>(w);
  w += align256(sizeof(Key) * N);
  int32_t* v0 = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * N);
  int32_t* v1 = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * N);
  int32_t* starts = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * N);
  int64_t* nseg = reinterpret_cast<int64_t*>(w);
  w += align256(sizeof(int64_t) * 4);
  p.chunk_slot = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * hot_chunks(N));
  p.pool = reinterpret_cast<float*>(w);
  p.pool_cap = hot_chunks(N);
  w += align256(sizeof(float) * hot_chunks(N) * (p.max_dim > 0 ? p.max_dim : 1));
  void* temp = w;
  size_t temp_bytes = cub_temp_bytes<Key>(N);

  const bool prepare_only = (p.flags & NEO_BWD_FLAG_PREPARE) != 0;
  const bool apply_only = (p.flags & NEO_BWD_FLAG_APPLY) != 0;
  const int wvec = weight_dtype == NEO_F16 ? 8 : 4;
  const bool fast = weight_dtype != NEO_F64 && p.mode == NEO_BWD_UPDATE && p.pooling == NEO_POOL_SUM &&
                    p.max_dim <= 2 * kWarp * wvec && !out_count &&
                    p.B * p.grad_stride < (int64_t(1) << 32);  // 32-bit upstream offsets
  const bool dense_fast = weight_dtype == NEO_F32 && p.mode == NEO_BWD_DENSE && p.pooling == NEO_POOL_SUM &&
                          (p.flags & NEO_BWD_FLAG_ALIGNED) && p.max_dim <= 2 * kWarp * 4 && !out_count &&
                          p.B * p.grad_stride < (int64_t(1) << 32) && use_pipe_variant();
  if ((prepare_only || apply_only) && !fast)
    return fail(NEO_E_ARG, "neo_tbe_backward: PREPARE/APPLY need the streamed UPDATE path");
  int rc = NEO_OK;
  cub::DoubleBuffer<Key> kbuf(k0, k1);
  cub::DoubleBuffer<int32_t> vbuf(v0, v1);
  if (apply_only) {
    std::lock_guard<std::mutex> lk(g_prep_mu);
    auto it = g_prep_sel.find(workspace);
    if (it == g_prep_sel.end()) return fail(NEO_E_ARG, "neo_tbe_backward: APPLY on an unprepared workspace");
    kbuf.selector = vbuf.selector = it->second;
    g_prep_sel.erase(it);
  } else {
  const int64_t bags = (int64_t)p.T * p.B;
  int kb_dev = 0, kb_sms = 0;
  cudaGetDevice(&kb_dev);
  cudaDeviceGetAttribute(&kb_sms, cudaDevAttrMultiProcessorCount, kb_dev);
  const int64_t kb_want = (bags + 8 * 4 - 1) / (8 * 4);
  const unsigned kb_blocks = (unsigned)(kb_want < (int64_t)kb_sms * 8 ? (kb_want > 0 ? kb_want : 1) : (int64_t)kb_sms * 8);
  const Key sentinel = (Key)p.total_rows;
  if (index_dtype == NEO_I32)
    build_keys_kernel<int32_t, Key><<<kb_blocks, 256, 0, s>>>(
        p.T, p.B, p.row_offsets, (const int32_t*)indices, p.offsets, k0, v0, sentinel, err);
  else
    build_keys_kernel<int64_t, Key><<<kb_blocks, 256, 0, s>>>(
        p.T, p.B, p.row_offsets, (const int64_t*)indices, p.offsets, k0, v0, sentinel, err);
  rc = check_launch("neo_tbe_backward(keys)");
  if (rc) return rc;

  const int bits = key_bits_for(p.total_rows);
  if (cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kbuf, vbuf, (int)N, 0, bits, s) !=
      cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: radix sort failed");
  if (prepare_only) {
    std::lock_guard<std::mutex> lk(g_prep_mu);
    g_prep_sel[workspace] = kbuf.selector;
    launch_error_finalize(err, indices, index_dtype, p.offsets, p.B, p.T, s);
    return check_launch("neo_tbe_backward(prepare)");
  }
  }  // !apply_only
  const Key* keys = kbuf.Current();
  p.keys = keys;
  p.bags = vbuf.Current();
  p.chunk_counter = nseg + 1;
  p.pool_counter = reinterpret_cast<unsigned*>(nseg + 2);
  if (dense_fast) {
    switch (grad_dtype) {
      case NEO_F32: rc = launch_dense_pipe<float, Key>(p, s); break;
      case NEO_BF16: rc = launch_dense_pipe<__nv_bfloat16, Key>(p, s); break;
      case NEO_F16: rc = launch_dense_pipe<__half, Key>(p, s); break;
      default: return fail(NEO_E_ARG, "neo_tbe_backward: gradient dtype must be F32, BF16 or F16");
    }
    if (rc) return rc;
    launch_error_finalize(err, indices, index_dtype, p.offsets, p.B, p.T, s);
    return check_launch("neo_tbe_backward(finalize)");
  }
  if (fast) {
    const bool h = weight_dtype == NEO_F16;
    switch (grad_dtype) {
      case NEO_F32:
        rc = h ? launch_stream<__half, float, Key>(p, s) : launch_stream<float, float, Key>(p, s);
        break;
      case NEO_BF16:
        rc = h ? launch_stream<__half, __nv_bfloat16, Key>(p, s)
               : launch_stream<float, __nv_bfloat16, Key>(p, s);
        break;
      case NEO_F16:
        rc = h ? launch_stream<__half, __half, Key>(p, s) : launch_stream<float, __half, Key>(p, s);
        break;
      default:
        return fail(NEO_E_ARG, "neo_tbe_backward: gradient dtype must be F32, BF16 or F16");
    }
    if (rc) return rc;
    if (!apply_only) launch_error_finalize(err, indices, index_dtype, p.offsets, p.B, p.T, s);
    return check_launch("neo_tbe_backward(finalize)");
  }
  cub::CountingInputIterator<int32_t> it(0);
  temp_bytes = cub_temp_bytes<Key>(N);
  if (cub::DeviceSelect::If(temp, temp_bytes, it, starts, nseg, (int)N, HeadFlag<Key>{keys}, s) !=
      cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: segment select failed");
  p.seg_starts = starts;
  p.num_segs = nseg;

  switch (weight_dtype) {
    case NEO_F64:
      if (grad_dtype != NEO_F64) return fail(NEO_E_ARG, "F64 tables take F64 gradients");
      rc = launch_segments<double, double, Key>(p, s);
      break;
    case NEO_F32:
    case NEO_F16: {
      const bool h = weight_dtype == NEO_F16;
      switch (grad_dtype) {
        case NEO_F32:
          rc = h ? launch_segments<__half, float, Key>(p, s) : launch_segments<float, float, Key>(p, s);
          break;
        case NEO_BF16:
          rc = h ? launch_segments<__half, __nv_bfloat16, Key>(p, s)
                 : launch_segments<float, __nv_bfloat16, Key>(p, s);
          break;
        case NEO_F16:
          rc = h ? launch_segments<__half, __half, Key>(p, s) : launch_segments<float, __half, Key>(p, s);
          break;
        default:
          return fail(NEO_E_ARG, "neo_tbe_backward: gradient dtype must be F32, BF16 or F16");
      }
      break;
    }
    default:
      return fail(NEO_E_ARG, "neo_tbe_backward: weight dtype must be F32, F16 or F64");
  }
  if (rc) return rc;
  if (out_count) {
    count_valid_kernel<Key><<<1, 1, 0, s>>>(keys, starts, nseg, p.total_rows, out_count);
    rc = check_launch("neo_tbe_backward(count)");
    if (rc) return rc;
  }
  launch_error_finalize(err, indices, index_dtype, p.offsets, p.B, p.T, s);
  return check_launch("neo_tbe_backward(finalize)");
}

}  // namespace neo

extern "C" size_t neo_tbe_backward_workspace_bytes(int64_t num_indices, int64_t total_rows, int32_t max_dim) {
  if (num_indices < 1) num_indices = 1;
  return neo::use_wide_keys(total_rows) ? neo::workspace_for<uint64_t>(num_indices, max_dim)
                                        : neo::workspace_for<uint32_t>(num_indices, max_dim);
}

extern "C" int neo_tbe_backward(int32_t num_tables, int64_t batch, const int64_t* row_offsets,
                                int64_t total_rows, const int32_t* dim_offsets, int32_t max_dim,
                                const uint64_t* weights, int32_t weight_dtype,
                                const uint64_t* moments, const void* indices,
                                int32_t index_dtype, const int64_t* offsets, int64_t num_indices,
                                int32_t pooling, const void* grad, int32_t grad_dtype,
                                int64_t grad_stride, int32_t mode, int32_t optim, double lr,
                                double eps, int64_t* out_ids, void* out_grads,
                                int64_t* out_count, const uint64_t* dense_grads, void* workspace,
                                size_t workspace_bytes, neo_error* err, void* stream) {
  using namespace neo;
  cudaStream_t s = as_stream(stream);
  if (num_tables < 0 || batch < 0 || num_indices < 0 || max_dim < 0 || total_rows < 0)
    return fail(NEO_E_ARG, "neo_tbe_backward: negative size");
  if ((int64_t)num_tables * batch >= INT_MAX || num_indices >= INT_MAX)
    return fail(NEO_E_ARG, "neo_tbe_backward: more than 2^31 bags or indices in one call");
  const int32_t base_mode = mode & 0xff;
  if (base_mode != NEO_BWD_UPDATE && base_mode != NEO_BWD_AGGREGATE && base_mode != NEO_BWD_DENSE)
    return fail(NEO_E_ARG, "neo_tbe_backward: bad mode");
  if (base_mode == NEO_BWD_UPDATE) {
    if (optim != NEO_OPT_SGD && optim != NEO_OPT_ROWWISE_ADAGRAD && optim != NEO_OPT_ADAGRAD)
      return fail(NEO_E_ARG, "cfg.kind: unknown optimizer");
    if (!(lr > 0)) return fail(NEO_E_ARG, "lr: must be > 0");
    if (eps < 0) return fail(NEO_E_ARG, "eps: must be >= 0");
    if (optim != NEO_OPT_SGD && !moments) return fail(NEO_E_ARG, "moment: state required");
  }
  if (base_mode == NEO_BWD_AGGREGATE && (!out_ids || !out_grads))
    return fail(NEO_E_ARG, "neo_tbe_backward: AGGREGATE needs out_ids/out_grads");
  if (base_mode == NEO_BWD_DENSE && !dense_grads)
    return fail(NEO_E_ARG, "neo_tbe_backward: DENSE needs dense_grads");
  if (pooling != NEO_POOL_SUM && pooling != NEO_POOL_MEAN)
    return fail(NEO_E_ARG, "neo_tbe_backward: pooling must be SUM or MEAN");
  if (num_tables == 0 || batch == 0 || num_indices == 0) {
    if (out_count) {
      if (cudaMemsetAsync(out_count, 0, sizeof(int64_t), s) != cudaSuccess)
        return fail(NEO_E_CUDA, "neo_tbe_backward: memset failed");
    }
    return NEO_OK;
  }
  SegParams p{};
  p.T = num_tables;
  p.B = batch;
  p.row_offsets = row_offsets;
  p.total_rows = total_rows;
  p.dim_offsets = dim_offsets;
  p.max_dim = max_dim;
  p.weights = weights;
  p.moments = moments;
  p.grad = grad;
  p.grad_stride = grad_stride;
  p.pooling = pooling;
  p.offsets = offsets;
  p.mode = mode & 0xff;
  p.flags = mode & ~0xff;
  p.optim = optim;
  p.lr = lr;
  p.eps = eps;
  p.out_ids = out_ids;
  p.out_grads = out_grads;
  p.dense_grads = dense_grads;
  p.N = num_indices;
  if (bkt_eligible(p, weight_dtype, grad_dtype, out_count != nullptr))
    return run_bucket_backward(p, weight_dtype, grad_dtype, indices, index_dtype, workspace, workspace_bytes, err, s);
  if (use_wide_keys(total_rows))
    return run_backward<uint64_t>(p, weight_dtype, grad_dtype, indices, index_dtype, workspace,
                                  workspace_bytes, out_count, err, s);
  return run_backward<uint32_t>(p, weight_dtype, grad_dtype, indices, index_dtype, workspace,
                                workspace_bytes, out_count, err, s);
}
