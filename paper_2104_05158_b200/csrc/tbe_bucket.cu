// Bucketed fused backward + optimizer: the default UPDATE / DENSE fast path.
//
// Reference semantics (unchanged): embedding.py:175-192 backward_sort_aggregate
// (touched rows ascending, each row's gradient = the sum of its occurrences'
// upstream rows in buffer order) followed by exactly one optimizer step per
// touched row (embedding.py:212-254, fused as embedding.py:270-281).  The
// stable order that np.unique + np.add.at imply is produced here by a
// hand-written two-level counting sort — no library sort:
//
//   1. bkt_setup      per table: bucket size 2^s rows (s chosen so a bucket
//                     holds ~`target` occurrences and a table has <= kMaxB
//                     buckets), bucket bases (block scan over tables).
//   2. bkt_count      CTA per (table, chunk of kCHB bags): shared-memory
//                     histogram of the chunk's ids by bucket -> count matrix
//                     [bucket][chunk] (range-checks ids, first bad position
//                     into neo_error).
//   3. bkt_scan_*     exclusive scan of the count matrix (bucket-major, chunk-
//                     minor): every (bucket, chunk) gets its output offset.
//   4. bkt_classify   bucket starts; buckets larger than kCap are queued.
//   5. bkt_scatter    CTA per chunk again: per-warp histograms, per-warp
//                     cursors, then each warp walks its contiguous bag range
//                     in buffer order and places (row_low, bag) entries with
//                     __match_any_sync ranking: a STABLE scatter, so every
//                     bucket's entries are in buffer order.
//   6. bkt_update     persistent CTAs claim buckets (queued big ones first,
//                     then table-major order so each table's upstream slice
//                     stays L2-resident).  Per bucket: stable counting sort by
//                     row within the bucket (shared memory; <= 9-bit digits,
//                     one pass for the usual bucket), row heads compacted by a
//                     block scan, then a sub-warp of S lanes (8 row elements
//                     per lane) per touched row: weight row + optimizer state
//                     are prefetched, the row's upstream rows are gathered and
//                     summed in order (two in flight), and one optimizer step
//                     is applied and stored.  Rows with more than kLong
//                     occurrences are split across every sub-warp of the CTA
//                     (contiguous pieces, partials combined in piece order).
//                     Buckets larger than kCap are sorted through global
//                     scratch in kCap chunks by the same stable passes.
//
// Everything is deterministic: the order of every floating-point sum depends
// only on the input.
#include <cstdio>
#include <string>

#include "bwd_common.cuh"

namespace neo {
namespace bkt {

constexpr int kMaxB = 2048;    // row buckets per table (count / scatter shared-memory histograms)
constexpr int kSMin = 4;       // smallest bucket: 16 rows
constexpr int kCHB = 2048;     // bags per count / scatter chunk
constexpr int kScW = 8;        // warps per count / scatter CTA
constexpr int kCap = 4096;     // entries per bucket sorted in shared memory
constexpr int kUW = 16;        // warps per update CTA
constexpr int kUT = kUW * kWarp;
constexpr int kDigit = 9;      // bits per stable counting pass
constexpr int kBins = 1 << kDigit;
constexpr int kLong = 64;      // rows with more occurrences are split across the CTA
constexpr int kEPL = 8;        // row elements per lane
constexpr int kMaxDim = kWarp * kEPL;
constexpr int kScanTile = 4096;  // 256 threads x 16
constexpr int kTarget = 1024;    // default occurrences per bucket
static_assert(kUT == kBins, "one digit bin per update thread");

struct Params {
  int32_t T;
  int64_t B;
  int32_t cpt;       // chunks per table = ceil(B / kCHB)
  int32_t bag_bits;  // bits of a table-local bag index
  int32_t target;
  const int64_t* row_offsets;
  const int64_t* offsets;
  int32_t* sbits;    // [T]
  int64_t* bbase;    // [T+1], bbase[T] = total buckets
  int32_t* mat;      // [nb*cpt + 1] counts, then exclusive offsets (+ total)
  int32_t* tiles;    // scan tile sums
  int32_t* bstart;   // [nb+1]
  int32_t* big;      // queued big buckets
  int32_t* ctr;      // [0] claim counter, [1] big-bucket count
  uint32_t* ent;     // bucketed entries (row_low << bag_bits | bag)
  uint32_t* ent2;    // scratch for big buckets
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int bits_for(int64_t v) {  // ceil(log2(v)), v >= 1
  int b = 0;
  while (b < 62 && (int64_t(1) << b) < v) ++b;
  return b;
}

// Block-wide exclusive scan of one int per thread (NT threads); wsum must hold
// NT/32 + 1 ints.  Returns the exclusive prefix; *total gets the sum.
template <int NT>
__device__ __forceinline__ int block_scan_excl(int v, int* wsum, int* total) {
  constexpr int NW = NT / kWarp;
  const int lane = threadIdx.x % kWarp, warp = threadIdx.x / kWarp;
  int incl = v;
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == kWarp - 1) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int x = lane < NW ? wsum[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < NW) wsum[lane] = xi - x;
    if (lane == NW - 1) wsum[NW] = xi;
  }
  __syncthreads();
  const int r = wsum[warp] + incl - v;
  *total = wsum[NW];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// 1. per-table bucket geometry

__global__ void __launch_bounds__(1024) bkt_setup_kernel(Params q) {
  __shared__ int wsum[33];
  __shared__ long long s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  if (threadIdx.x < 4) q.ctr[threadIdx.x] = 0;
  __syncthreads();
  for (int t0 = 0; t0 < q.T; t0 += 1024) {
    const int t = t0 + threadIdx.x;
    int nb = 0;
    if (t < q.T) {
      const int64_t H = q.row_offsets[t + 1] - q.row_offsets[t];
      const int64_t Nt = q.offsets[(int64_t)(t + 1) * q.B] - q.offsets[(int64_t)t * q.B];
      const int hb = H > 1 ? bits_for(H) : 0;
      int s = kSMin;
      while (((H + (int64_t(1) << s) - 1) >> s) > kMaxB) ++s;
      // occurrences per bucket ~ Nt * 2^s / H >= target (a bucket of the whole table at most)
      while (s < hb && (double)Nt * (double)(int64_t(1) << s) < (double)q.target * (double)H) ++s;
      if (s > 32 - q.bag_bits) s = 32 - q.bag_bits;  // the host checked the kMaxB bound still holds
      q.sbits[t] = s;
      nb = (int)((H + (int64_t(1) << s) - 1) >> s);
    }
    int total;
    const int ex = block_scan_excl<1024>(nb, wsum, &total);
    if (t < q.T) q.bbase[t] = s_carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) q.bbase[q.T] = s_carry;
}

__device__ __forceinline__ int table_of_bucket(const int64_t* bbase, int T, int64_t b) {
  int lo = 0, hi = T - 1;  // last t with bbase[t] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bbase[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// 2. count matrix

template <typename Idx>
__global__ void __launch_bounds__(kScW* kWarp) bkt_count_kernel(Params q, const Idx* __restrict__ indices,
                                                                  neo_error* err) {
  __shared__ int hist[kMaxB];
  const int t = blockIdx.x / q.cpt, cc = blockIdx.x % q.cpt;
  if (t >= q.T) return;
  const int s = q.sbits[t];
  const int64_t bb0 = q.bbase[t];
  const int nb = (int)(q.bbase[t + 1] - bb0);
  const int64_t H = q.row_offsets[t + 1] - q.row_offsets[t];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t g0 = (int64_t)t * q.B + (int64_t)cc * kCHB;
  const int64_t g1 = (int64_t)t * q.B + min64(q.B, (int64_t)(cc + 1) * kCHB);
  const int64_t p0 = q.offsets[g0], p1 = q.offsets[g1];
  for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const int64_t id = (int64_t)indices[p];
    if (id < 0 || id >= H) record_bad_index(err, p);
    else atomicAdd(&hist[(int)(id >> s)], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) q.mat[(bb0 + i) * q.cpt + cc] = hist[i];
}

// ---------------------------------------------------------------------------
// 3. exclusive scan of the count matrix (M = total buckets * cpt entries)

__global__ void __launch_bounds__(256) bkt_scan_reduce_kernel(Params q) {
  __shared__ int ws[8];
  const int64_t M = q.bbase[q.T] * q.cpt;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  if (t0 >= M) return;
  int s = 0;
  for (int64_t i = t0 + threadIdx.x; i < t0 + kScanTile && i < M; i += 256) s += q.mat[i];
  s = warp_sum(s);
  if (threadIdx.x % kWarp == 0) ws[threadIdx.x / kWarp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int w = 0; w < 8; ++w) a += ws[w];
    q.tiles[blockIdx.x] = a;
  }
}

__global__ void __launch_bounds__(1024) bkt_scan_tiles_kernel(Params q) {
  __shared__ int wsum[33];
  __shared__ int s_carry;
  const int64_t M = q.bbase[q.T] * q.cpt;
  const int ntiles = (int)((M + kScanTile - 1) / kScanTile);
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int i0 = 0; i0 < ntiles; i0 += 1024) {
    const int i = i0 + threadIdx.x;
    const int v = i < ntiles ? q.tiles[i] : 0;
    int total;
    const int ex = block_scan_excl<1024>(v, wsum, &total);
    if (i < ntiles) q.tiles[i] = s_carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) q.mat[M] = s_carry;  // total valid entries
}

__global__ void __launch_bounds__(256) bkt_scan_down_kernel(Params q) {
  __shared__ int wsum[9];
  const int64_t M = q.bbase[q.T] * q.cpt;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  if (t0 >= M) return;
  constexpr int kPer = kScanTile / 256;
  int v[kPer];
  int s = 0;
  const int64_t base = t0 + (int64_t)threadIdx.x * kPer;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    v[k] = base + k < M ? q.mat[base + k] : 0;
    s += v[k];
  }
  int total;
  int ex = block_scan_excl<256>(s, wsum, &total) + q.tiles[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (base + k < M) q.mat[base + k] = ex;
    ex += v[k];
  }
}

// ---------------------------------------------------------------------------
// 4. bucket starts, big-bucket queue

__global__ void __launch_bounds__(256) bkt_classify_kernel(Params q) {
  const int64_t nbt = q.bbase[q.T];
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbt) return;
  const int32_t st = q.mat[b * q.cpt];
  const int32_t en = q.mat[(b + 1) * q.cpt];  // b + 1 == nbt: the total at mat[M]
  q.bstart[b] = st;
  if (b + 1 == nbt) q.bstart[nbt] = en;
  if (en - st > kCap) q.big[atomicAdd(&q.ctr[1], 1)] = (int32_t)b;
}

// ---------------------------------------------------------------------------
// 5. stable scatter into buckets

template <typename Idx>
__global__ void __launch_bounds__(kScW* kWarp) bkt_scatter_kernel(Params q, const Idx* __restrict__ indices) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = blockIdx.x / q.cpt, cc = blockIdx.x % q.cpt;
  if (t >= q.T) return;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const unsigned full = 0xffffffffu;
  const int s = q.sbits[t];
  const int64_t bb0 = q.bbase[t];
  const int nb = (int)(q.bbase[t + 1] - bb0);
  const int64_t H = q.row_offsets[t + 1] - q.row_offsets[t];
  const uint32_t rmask = (uint32_t)((int64_t(1) << s) - 1);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw);  // [kScW][nb]
  int32_t* base = reinterpret_cast<int32_t*>(hist + kScW * nb);
  for (int i = threadIdx.x; i < kScW * nb; i += blockDim.x) hist[i] = 0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) base[i] = q.mat[(bb0 + i) * q.cpt + cc];
  __syncthreads();
  // this warp's contiguous bag range (buffer order)
  const int64_t cb0 = (int64_t)cc * kCHB, cb1 = min64(q.B, cb0 + kCHB);
  const int64_t per = (cb1 - cb0 + kScW - 1) / kScW;
  const int64_t wb0 = min64(cb1, cb0 + warp * per), wb1 = min64(cb1, wb0 + per);
  const int64_t* off = q.offsets + (int64_t)t * q.B;
  const int64_t p0 = off[wb0], p1 = off[wb1];
  uint32_t* wh = hist + warp * nb;
  for (int64_t p = p0 + lane; p < p1; p += kWarp) {
    const int64_t id = (int64_t)indices[p];
    if (id >= 0 && id < H) atomicAdd(&wh[(int)(id >> s)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    uint32_t run = (uint32_t)base[i];
    for (int w = 0; w < kScW; ++w) {
      const uint32_t c = hist[w * nb + i];
      hist[w * nb + i] = run;
      run += c;
    }
  }
  __syncthreads();
  // place: 32 bags per window; each lane finds its entry's bag by a shuffle search
  for (int64_t bw = wb0; bw < wb1; bw += kWarp) {
    const int nbg = (int)min64(kWarp, wb1 - bw);
    const int64_t oend = off[bw + nbg];
    const int64_t o = lane < nbg ? off[bw + lane] : oend;
    const int64_t ostart = __shfl_sync(full, o, 0);
    for (int64_t pb = ostart; pb < oend; pb += kWarp) {
      const int64_t p = pb + lane;
      const bool in = p < oend;
      int k = 0;  // last bag of the window starting at or before p
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int64_t ok = __shfl_sync(full, o, k + step);
        if (ok <= p) k += step;
      }
      const int64_t id = in ? (int64_t)indices[p] : -1;
      const bool valid = in && id >= 0 && id < H;
      const uint32_t bk = valid ? (uint32_t)(id >> s) : 0xffffffffu;
      const unsigned peers = __match_any_sync(full, bk);
      if (valid) {
        const uint32_t pos = wh[bk] + __popc(peers & lanemask_lt());
        q.ent[pos] = (((uint32_t)id & rmask) << q.bag_bits) | (uint32_t)(bw + k);
      }
      __syncwarp();
      if (valid && (peers >> lane) == 1u) wh[bk] += __popc(peers);
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// 6. per-bucket sort + fused segment reduce + optimizer

struct alignas(16) USmem {
  uint32_t a[kCap];
  uint32_t b[kCap];
  int32_t rbeg[kCap + 1];
  float part[kUW * kWarp * kEPL];
  uint16_t hist[kBins * kUW];  // [bin][warp]
  int32_t cursor[kBins];
  int32_t tot[kBins];
  int32_t longs[kCap / kLong + 2];
  int32_t wsum[kUW + 1];
  int32_t nlong;
  int32_t bucket;
  int32_t table;
  int32_t nrows;
};

// One stable counting pass over [c0, c1) of src (c1 - c0 <= kCap) into dst by
// digit (e >> shift) & (nbins - 1) at dst[cursor[d] + ...]; cursor advances by
// the chunk's per-digit totals.  All kUT threads call it.
__device__ __forceinline__ void place_chunk(const uint32_t* src, uint32_t* dst, int64_t c0, int64_t c1, int shift,
                                            int nbins, USmem& sm) {
  const unsigned full = 0xffffffffu;
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const uint32_t dm = (uint32_t)nbins - 1;
  for (int i = tid; i < nbins * kUW; i += kUT) sm.hist[i] = 0;
  __syncthreads();
  const int len = (int)(c1 - c0);
  const int per = (len + kUW - 1) / kUW;
  const int64_t r0 = c0 + min(len, warp * per), r1 = c0 + min(len, warp * per + per);
  for (int64_t i0 = r0; i0 < r1; i0 += kWarp) {  // per-warp digit counts (leader read-modify-write)
    const int64_t i = i0 + lane;
    const bool v = i < r1;
    const uint32_t d = v ? (src[i] >> shift) & dm : 0xffffffffu;
    const unsigned peers = __match_any_sync(full, d);
    if (v && (peers >> lane) == 1u) sm.hist[d * kUW + warp] += (uint16_t)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = tid; d < nbins; d += kUT) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < kUW; ++w) {
      const int c = sm.hist[d * kUW + w];
      sm.hist[d * kUW + w] = (uint16_t)run;
      run += c;
    }
    sm.tot[d] = run;
  }
  __syncthreads();
  for (int64_t i0 = r0; i0 < r1; i0 += kWarp) {
    const int64_t i = i0 + lane;
    const bool v = i < r1;
    const uint32_t e = v ? src[i] : 0u;
    const uint32_t d = v ? (e >> shift) & dm : 0xffffffffu;
    const unsigned peers = __match_any_sync(full, d);
    if (v) dst[sm.cursor[d] + sm.hist[d * kUW + warp] + __popc(peers & lanemask_lt())] = e;
    __syncwarp();
    if (v && (peers >> lane) == 1u) sm.hist[d * kUW + warp] += (uint16_t)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = tid; d < nbins; d += kUT) sm.cursor[d] += sm.tot[d];
  __syncthreads();
}

// stable sort of n entries by bits [shift, shift + nbits) (one full pass)
__device__ __forceinline__ void sort_pass(const uint32_t* src, uint32_t* dst, int64_t n, int shift, int nbits,
                                          USmem& sm) {
  const int tid = threadIdx.x;
  const int nbins = 1 << nbits;
  const uint32_t dm = (uint32_t)nbins - 1;
  sm.tot[tid] = 0;  // kUT == kBins
  __syncthreads();
  for (int64_t i = tid; i < n; i += kUT) atomicAdd(&sm.tot[(src[i] >> shift) & dm], 1);
  __syncthreads();
  int total;
  const int ex = block_scan_excl<kUT>(tid < nbins ? sm.tot[tid] : 0, sm.wsum, &total);
  sm.cursor[tid] = ex;
  __syncthreads();
  for (int64_t c0 = 0; c0 < n; c0 += kCap) place_chunk(src, dst, c0, min64(n, c0 + kCap), shift, nbins, sm);
}

template <typename W, typename G, int OPT>
struct RowCtx {
  const G* grad;
  int64_t stride;
  int32_t doff;
  int32_t D;
  W* wt;          // table weights (the dense gradient for OPT_NONE)
  float* mom;     // optimizer state
  int64_t row0;   // first row of the bucket
  int32_t bag_bits;
  uint32_t bmask;
  float lr, eps, invD;
};

template <typename T>
__device__ __forceinline__ void ld8(const T* p, float (&x)[kEPL]) {
  const Vec<T, kEPL> v = ld_vec<T, kEPL>(p);
#pragma unroll
  for (int e = 0; e < kEPL; ++e) x[e] = Elem<T>::to_f(v.v[e]);
}

template <typename T>
__device__ __forceinline__ void ld8_plain(const T* p, float (&x)[kEPL]) {
  Vec<T, kEPL> v;
  constexpr int kB = (int)sizeof(T) * kEPL;
  if constexpr (kB == 32) {
    reinterpret_cast<uint4*>(&v)[0] = reinterpret_cast<const uint4*>(p)[0];
    reinterpret_cast<uint4*>(&v)[1] = reinterpret_cast<const uint4*>(p)[1];
  } else {
    *reinterpret_cast<uint4*>(&v) = *reinterpret_cast<const uint4*>(p);
  }
#pragma unroll
  for (int e = 0; e < kEPL; ++e) x[e] = Elem<T>::to_f(v.v[e]);
}

template <typename T>
__device__ __forceinline__ void st8(T* p, const float (&x)[kEPL]) {
  Vec<T, kEPL> v;
#pragma unroll
  for (int e = 0; e < kEPL; ++e) v.v[e] = Elem<T>::from_f(x[e]);
  st_vec<T, kEPL>(p, v);
}

// acc += upstream rows of entries [j0, j1) of list, in order; the trip count
// (jmax - j0) is warp-uniform
template <typename W, typename G, int OPT>
__device__ __forceinline__ void gather_sum(const RowCtx<W, G, OPT>& c, const uint32_t* list, int64_t j0, int64_t j1,
                                           int64_t jmax, bool col, int sl, float (&acc)[kEPL]) {
  for (int64_t j = j0; j < jmax; j += 2) {
    const bool h0 = col && j < j1, h1 = col && j + 1 < j1;
    const uint32_t e0 = h0 ? list[j] : 0u;
    const uint32_t e1 = h1 ? list[j + 1] : 0u;
    float x0[kEPL], x1[kEPL];
    if (h0) ld8<G>(c.grad + (int64_t)(e0 & c.bmask) * c.stride + c.doff + sl * kEPL, x0);
    if (h1) ld8<G>(c.grad + (int64_t)(e1 & c.bmask) * c.stride + c.doff + sl * kEPL, x1);
    if (h0) {
#pragma unroll
      for (int e = 0; e < kEPL; ++e) acc[e] += x0[e];
    }
    if (h1) {
#pragma unroll
      for (int e = 0; e < kEPL; ++e) acc[e] += x1[e];
    }
  }
}

template <typename W, typename G, int OPT>
__device__ __forceinline__ void prefetch_row(const RowCtx<W, G, OPT>& c, int64_t row, bool valid, bool col, int sl,
                                             float (&wv)[kEPL], float (&mv)[kEPL], float& mrow) {
#pragma unroll
  for (int e = 0; e < kEPL; ++e) wv[e] = mv[e] = 0.f;
  mrow = 0.f;
  if (OPT == NEO_OPT_NONE || !valid) return;
  if (col) ld8_plain<W>(c.wt + row * c.D + sl * kEPL, wv);
  if (OPT == NEO_OPT_ROWWISE_ADAGRAD) mrow = c.mom[row];
  if (OPT == NEO_OPT_ADAGRAD && col) ld8_plain<float>(c.mom + row * c.D + sl * kEPL, mv);
}

// exactly one optimizer step (or the DENSE store) for one row; every lane of
// the warp calls it (sub-warps of S lanes, one row each)
template <typename W, typename G, int OPT>
__device__ __forceinline__ void finish_row(const RowCtx<W, G, OPT>& c, int64_t row, bool valid, bool col, int S,
                                           int sub, int sl, const float (&wv)[kEPL], const float (&mv)[kEPL],
                                           float mrow, const float (&acc)[kEPL]) {
  const unsigned full = 0xffffffffu;
  const unsigned submask = S == kWarp ? full : (((1u << S) - 1u) << (sub * S));
  if (OPT == NEO_OPT_NONE) {
    if (valid && col) st8<float>(reinterpret_cast<float*>(c.wt) + row * c.D + sl * kEPL, acc);
    return;
  }
  float ss = 0.f;
  if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
#pragma unroll
    for (int e = 0; e < kEPL; ++e) ss += acc[e] * acc[e];
    for (int o = S >> 1; o > 0; o >>= 1) ss += __shfl_xor_sync(full, ss, o);
  }
  bool live = valid;
  if (OPT == NEO_OPT_ADAGRAD || OPT == NEO_OPT_ROWWISE_ADAGRAD) {
    // an identically zero gradient leaves the row untouched (embedding.py:223-228);
    // ss can underflow to 0 for tiny nonzero gradients, so vote
    bool nz = false;
#pragma unroll
    for (int e = 0; e < kEPL; ++e) nz |= acc[e] != 0.f;
    const unsigned vote = __ballot_sync(full, nz);  // every lane votes (no short circuit)
    live = live && (vote & submask) != 0u;
  }
  if (!live) return;
  float out[kEPL];
  if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
    const float m = mrow + ss * c.invD;
    if (sl == 0) c.mom[row] = m;
    const float scale = __fdividef(c.lr, __fsqrt_rn(m) + c.eps);
#pragma unroll
    for (int e = 0; e < kEPL; ++e) out[e] = wv[e] - acc[e] * scale;
  } else if (OPT == NEO_OPT_ADAGRAD) {
    float mo[kEPL];
#pragma unroll
    for (int e = 0; e < kEPL; ++e) {
      mo[e] = mv[e] + acc[e] * acc[e];
      out[e] = wv[e] - __fdividef(c.lr * acc[e], __fsqrt_rn(mo[e]) + c.eps);
    }
    if (col) st8<float>(c.mom + row * c.D + sl * kEPL, mo);
  } else {
#pragma unroll
    for (int e = 0; e < kEPL; ++e) out[e] = wv[e] - c.lr * acc[e];
  }
  if (col) st8<W>(c.wt + row * c.D + sl * kEPL, out);
}

// rows [0, nr) of the current window (starts in sm.rbeg): short rows one per
// sub-warp, long rows split across the CTA
template <typename W, typename G, int OPT>
__device__ __forceinline__ void process_rows(const RowCtx<W, G, OPT>& c, const uint32_t* list, int nr, USmem& sm) {
  const unsigned full = 0xffffffffu;
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  int S = 1;
  while (S * kEPL < c.D) S <<= 1;
  const int R = kWarp / S, sub = lane / S, sl = lane % S;
  const bool col = sl * kEPL < c.D;
  if (tid == 0) sm.nlong = 0;
  __syncthreads();
  for (int g = warp; g * R < nr; g += kUW) {
    const int r = g * R + sub;
    bool valid = r < nr;
    int64_t rb = 0, re = 0;
    if (valid) {
      rb = sm.rbeg[r];
      re = sm.rbeg[r + 1];
      if (re - rb > kLong) {
        if (sl == 0) sm.longs[atomicAdd(&sm.nlong, 1)] = r;
        valid = false;
      }
    }
    const int64_t row = valid ? c.row0 + (int64_t)(list[rb] >> c.bag_bits) : 0;
    float wv[kEPL], mv[kEPL], mrow;
    prefetch_row<W, G, OPT>(c, row, valid, col, sl, wv, mv, mrow);
    float acc[kEPL];
#pragma unroll
    for (int e = 0; e < kEPL; ++e) acc[e] = 0.f;
    const int len = valid ? (int)(re - rb) : 0;
    const int maxlen = (int)__reduce_max_sync(full, (unsigned)len);
    gather_sum<W, G, OPT>(c, list, rb, rb + len, rb + maxlen, col && valid, sl, acc);
    finish_row<W, G, OPT>(c, row, valid, col, S, sub, sl, wv, mv, mrow, acc);
  }
  __syncthreads();
  const int nl = sm.nlong;
  const int nsub = kUW * R;
  const int k = warp * R + sub;
  for (int l = 0; l < nl; ++l) {
    const int r = sm.longs[l];
    const int64_t rb = sm.rbeg[r], re = sm.rbeg[r + 1], len = re - rb;
    const int64_t row = c.row0 + (int64_t)(list[rb] >> c.bag_bits);
    float acc[kEPL];
#pragma unroll
    for (int e = 0; e < kEPL; ++e) acc[e] = 0.f;
    const int64_t a0 = rb + len * k / nsub, a1 = rb + len * (k + 1) / nsub;
    const int64_t span = (int64_t)__reduce_max_sync(full, (unsigned)(a1 - a0));
    gather_sum<W, G, OPT>(c, list, a0, a1, a0 + span, col, sl, acc);
    if (col) {
#pragma unroll
      for (int e = 0; e < kEPL; ++e) sm.part[(k * S + sl) * kEPL + e] = acc[e];
    }
    __syncthreads();
    if (warp == 0) {  // sub-warp 0 combines the partials in piece order, then one step
      const bool own = sub == 0;
      float wv[kEPL], mv[kEPL], mrow;
      prefetch_row<W, G, OPT>(c, row, own, col, sl, wv, mv, mrow);
#pragma unroll
      for (int e = 0; e < kEPL; ++e) acc[e] = 0.f;
      if (own && col) {
        for (int qq = 0; qq < nsub; ++qq)
#pragma unroll
          for (int e = 0; e < kEPL; ++e) acc[e] += sm.part[(qq * S + sl) * kEPL + e];
      }
      finish_row<W, G, OPT>(c, row, own, col, S, sub, sl, wv, mv, mrow, acc);
    }
    __syncthreads();
  }
}

template <typename W, typename G, int OPT>
__global__ void __launch_bounds__(kUT, 2) bkt_update_kernel(Params q, SegParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  USmem& sm = *reinterpret_cast<USmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t nbt = q.bbase[q.T];
  const int nbig = q.ctr[1];
  for (;;) {
    if (tid == 0) {
      int b = -1;
      for (;;) {
        const int idx = atomicAdd(&q.ctr[0], 1);
        if (idx < nbig) {
          b = q.big[idx];
          break;
        }
        const int64_t j = (int64_t)idx - nbig;
        if (j >= nbt) break;
        const int n = q.bstart[j + 1] - q.bstart[j];
        if (n > 0 && n <= kCap) {
          b = (int)j;
          break;
        }
      }
      sm.bucket = b;
      if (b >= 0) sm.table = table_of_bucket(q.bbase, q.T, b);
    }
    __syncthreads();
    const int b = sm.bucket;
    if (b < 0) break;
    const int t = sm.table;
    const int s = q.sbits[t];
    const int64_t bs = q.bstart[b];
    const int64_t n = q.bstart[b + 1] - bs;
    RowCtx<W, G, OPT> c;
    c.grad = reinterpret_cast<const G*>(p.grad);
    c.stride = p.grad_stride;
    c.doff = p.dim_offsets[t];
    c.D = p.dim_offsets[t + 1] - c.doff;
    c.wt = reinterpret_cast<W*>(OPT == NEO_OPT_NONE ? p.dense_grads[t] : p.weights[t]);
    c.mom = (OPT == NEO_OPT_ROWWISE_ADAGRAD || OPT == NEO_OPT_ADAGRAD) ? reinterpret_cast<float*>(p.moments[t])
                                                                       : nullptr;
    c.row0 = (int64_t)(b - q.bbase[t]) << s;
    c.bag_bits = q.bag_bits;
    c.bmask = (uint32_t)((1u << q.bag_bits) - 1u);
    c.lr = (float)p.lr;
    c.eps = (float)p.eps;
    c.invD = 1.0f / (float)c.D;
    // stable LSD passes over the s row bits (entries arrive in buffer order)
    const int passes = (s + kDigit - 1) / kDigit;
    const int wbits = (s + passes - 1) / passes;
    const bool small = n <= kCap;
    const uint32_t* list = q.ent + bs;
    for (int k = 0; k < passes; ++k) {
      const int nbits = min(wbits, s - k * wbits);
      uint32_t* dst = small ? ((k & 1) ? sm.b : sm.a) : ((k & 1) ? q.ent + bs : q.ent2 + bs);
      sort_pass(list, dst, n, q.bag_bits + k * wbits, nbits, sm);
      list = dst;
    }
    // row windows of <= kCap entries: heads compacted by a block scan
    int64_t pos = 0;
    while (pos < n) {
      const int64_t w1 = min64(n, pos + kCap);
      constexpr int kPer = kCap / kUT;
      const int64_t i0 = pos + (int64_t)tid * kPer;
      unsigned hm = 0;
      {
        uint32_t prev = (i0 > pos && i0 < w1) ? (list[i0 - 1] >> q.bag_bits) : 0xffffffffu;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int64_t i = i0 + j;
          if (i < w1) {
            const uint32_t r = list[i] >> q.bag_bits;
            if (r != prev) hm |= 1u << j;
            prev = r;
          }
        }
      }
      int nr;
      int ex = block_scan_excl<kUT>(__popc(hm), sm.wsum, &nr);
#pragma unroll
      for (int j = 0; j < kPer; ++j)
        if ((hm >> j) & 1u) sm.rbeg[ex++] = (int32_t)(i0 + j);
      if (tid == 0) {
        // end of the window's last row (it may run past the window)
        int64_t end = w1;
        if (w1 < n) {
          const uint32_t last = list[w1 - 1] >> q.bag_bits;
          int64_t lo = w1, hi = n;  // first index with a different (larger) row
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((list[mid] >> q.bag_bits) == last) lo = mid + 1;
            else hi = mid;
          }
          end = lo;
        }
        sm.rbeg[nr] = (int32_t)end;
        sm.nrows = nr;
      }
      __syncthreads();
      process_rows<W, G, OPT>(c, list, sm.nrows, sm);
      pos = sm.rbeg[sm.nrows];
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// host driver

static int64_t bucket_bound(int32_t T, int64_t total_rows) {
  int64_t nb = (int64_t)kMaxB * T;
  const int64_t nb2 = total_rows / (1 << kSMin) + T;
  return nb2 < nb ? nb2 : nb;
}

static int bag_bits_for(int64_t B) {
  int b = 1;
  while ((int64_t(1) << b) < B) ++b;
  return b;
}

// NEO_BKT_DEBUG=1: synchronise and report after every launch (diagnostics)
static int dbg(cudaStream_t s, const char* what) {
  static const bool on = std::getenv("NEO_BKT_DEBUG") != nullptr;
  if (!on) return check_launch(what);
  const cudaError_t e = cudaStreamSynchronize(s);
  std::fprintf(stderr, "[bkt] %s: %s\n", what, cudaGetErrorString(e));
  return e == cudaSuccess ? NEO_OK : fail(NEO_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename W, typename G, int OPT>
static int launch_update(const Params& q, const SegParams& p, int sms, cudaStream_t s) {
  auto kern = bkt_update_kernel<W, G, OPT>;
  const int smem = (int)sizeof(USmem);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve bucket shared memory");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kUT, smem);
  if (per_sm < 1) per_sm = 1;
  kern<<<(unsigned)(sms * per_sm), kUT, smem, s>>>(q, p);
  return dbg(s, "neo_tbe_backward(bucket update)");
}

template <typename W, typename G>
static int launch_update_opt(const Params& q, const SegParams& p, int sms, cudaStream_t s) {
  if (p.mode == NEO_BWD_DENSE) {
    if constexpr (std::is_same<W, float>::value) return launch_update<W, G, NEO_OPT_NONE>(q, p, sms, s);
    return fail(NEO_E_ARG, "neo_tbe_backward: DENSE needs f32");
  }
  switch (p.optim) {
    case NEO_OPT_SGD: return launch_update<W, G, NEO_OPT_SGD>(q, p, sms, s);
    case NEO_OPT_ROWWISE_ADAGRAD: return launch_update<W, G, NEO_OPT_ROWWISE_ADAGRAD>(q, p, sms, s);
    default: return launch_update<W, G, NEO_OPT_ADAGRAD>(q, p, sms, s);
  }
}

static int target_entries() {
  const char* v = std::getenv("NEO_BKT_TARGET");
  const int t = v ? std::atoi(v) : 0;
  return t > 0 ? t : kTarget;
}

}  // namespace bkt

size_t bkt_workspace(int32_t T, int64_t B, int64_t N, int64_t total_rows) {
  using namespace bkt;
  const int64_t cpt = (B + kCHB - 1) / kCHB;
  const int64_t nb = bucket_bound(T, total_rows);
  const int64_t M = nb * cpt;
  size_t b = 0;
  b += align256(sizeof(int32_t) * T);                    // sbits
  b += align256(sizeof(int64_t) * (T + 1));              // bbase
  b += align256(sizeof(int32_t) * (M + 1));              // count matrix
  b += align256(sizeof(int32_t) * (M / kScanTile + 2));  // scan tiles
  b += align256(sizeof(int32_t) * (nb + 1));             // bucket starts
  b += align256(sizeof(int32_t) * (nb + 1));             // big-bucket queue
  b += align256(sizeof(int32_t) * 4);                    // counters
  b += 2 * align256(sizeof(uint32_t) * (N > 0 ? N : 1));  // entries + scratch
  return b;
}

// can the bucketed path take this call? (host side; layout promises from the caller)
bool bkt_eligible(const SegParams& p, int32_t weight_dtype, int32_t grad_dtype, bool out_count) {
  using namespace bkt;
  const char* v = std::getenv("NEO_BWD_VARIANT");
  if (v && (std::strcmp(v, "pipe") == 0 || std::strcmp(v, "stream") == 0)) return false;
  if (!(p.flags & NEO_BWD_FLAG_DIM8) || out_count) return false;
  if (p.flags & (NEO_BWD_FLAG_PREPARE | NEO_BWD_FLAG_APPLY)) return false;
  if (p.pooling != NEO_POOL_SUM || p.max_dim > kMaxDim) return false;
  if (grad_dtype != NEO_F32 && grad_dtype != NEO_BF16 && grad_dtype != NEO_F16) return false;
  if (p.mode == NEO_BWD_UPDATE) {
    if (weight_dtype != NEO_F32 && weight_dtype != NEO_F16) return false;
  } else if (p.mode == NEO_BWD_DENSE) {
    if (weight_dtype != NEO_F32) return false;
  } else {
    return false;
  }
  // the bucket bits of the largest possible table (kMaxB buckets) + bag bits must fit 32
  int s = kSMin;
  while (((p.total_rows + (int64_t(1) << s) - 1) >> s) > kMaxB) ++s;
  return s + bag_bits_for(p.B) <= 32;
}

int run_bucket_backward(SegParams p, int32_t weight_dtype, int32_t grad_dtype, const void* indices,
                        int32_t index_dtype, void* workspace, size_t ws_bytes, neo_error* err, cudaStream_t s) {
  using namespace bkt;
  const int64_t N = p.N;
  if (ws_bytes < bkt_workspace(p.T, p.B, N, p.total_rows))
    return fail(NEO_E_ARG, "neo_tbe_backward: workspace too small (bucketed path: neo_tbe_bucket_workspace_bytes)");
  Params q{};
  q.T = p.T;
  q.B = p.B;
  q.cpt = (int32_t)((p.B + kCHB - 1) / kCHB);
  q.bag_bits = bag_bits_for(p.B);
  q.target = target_entries();
  q.row_offsets = p.row_offsets;
  q.offsets = p.offsets;
  const int64_t nb = bucket_bound(p.T, p.total_rows);
  const int64_t M = nb * q.cpt;
  unsigned char* w = static_cast<unsigned char*>(workspace);
  q.sbits = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * p.T);
  q.bbase = reinterpret_cast<int64_t*>(w);
  w += align256(sizeof(int64_t) * (p.T + 1));
  q.mat = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (M + 1));
  q.tiles = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (M / kScanTile + 2));
  q.bstart = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (nb + 1));
  q.big = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (nb + 1));
  q.ctr = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * 4);
  q.ent = reinterpret_cast<uint32_t*>(w);
  w += align256(sizeof(uint32_t) * (N > 0 ? N : 1));
  q.ent2 = reinterpret_cast<uint32_t*>(w);

  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  bkt_setup_kernel<<<1, 1024, 0, s>>>(q);
  int rc = dbg(s, "neo_tbe_backward(bucket setup)");
  if (rc) return rc;
  const unsigned chunks = (unsigned)(p.T * (int64_t)q.cpt);
  if (index_dtype == NEO_I32)
    bkt_count_kernel<int32_t><<<chunks, kScW * kWarp, 0, s>>>(q, (const int32_t*)indices, err);
  else
    bkt_count_kernel<int64_t><<<chunks, kScW * kWarp, 0, s>>>(q, (const int64_t*)indices, err);
  if ((rc = dbg(s, "neo_tbe_backward(bucket count)"))) return rc;
  const unsigned tiles = (unsigned)((M + kScanTile - 1) / kScanTile);
  bkt_scan_reduce_kernel<<<tiles > 0 ? tiles : 1, 256, 0, s>>>(q);
  bkt_scan_tiles_kernel<<<1, 1024, 0, s>>>(q);
  bkt_scan_down_kernel<<<tiles > 0 ? tiles : 1, 256, 0, s>>>(q);
  if ((rc = dbg(s, "neo_tbe_backward(bucket scan)"))) return rc;
  bkt_classify_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(q);
  if ((rc = dbg(s, "neo_tbe_backward(bucket classify)"))) return rc;
  {
    const int smem = (int)((kScW + 1) * kMaxB * sizeof(uint32_t));
    auto k32 = bkt_scatter_kernel<int32_t>;
    auto k64 = bkt_scatter_kernel<int64_t>;
    if (cudaFuncSetAttribute(k32, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(k64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve scatter shared memory");
    if (index_dtype == NEO_I32) k32<<<chunks, kScW * kWarp, smem, s>>>(q, (const int32_t*)indices);
    else k64<<<chunks, kScW * kWarp, smem, s>>>(q, (const int64_t*)indices);
    if ((rc = dbg(s, "neo_tbe_backward(bucket scatter)"))) return rc;
  }
  const bool h = weight_dtype == NEO_F16;
  switch (grad_dtype) {
    case NEO_F32:
      rc = h ? launch_update_opt<__half, float>(q, p, sms, s) : launch_update_opt<float, float>(q, p, sms, s);
      break;
    case NEO_BF16:
      rc = h ? launch_update_opt<__half, __nv_bfloat16>(q, p, sms, s)
             : launch_update_opt<float, __nv_bfloat16>(q, p, sms, s);
      break;
    default:
      rc = h ? launch_update_opt<__half, __half>(q, p, sms, s) : launch_update_opt<float, __half>(q, p, sms, s);
      break;
  }
  if (rc) return rc;
  launch_error_finalize(err, indices, index_dtype, p.offsets, p.B, p.T, s);
  return check_launch("neo_tbe_backward(finalize)");
}

}  // namespace neo

extern "C" size_t neo_tbe_bucket_workspace_bytes(int32_t num_tables, int64_t batch, int64_t num_indices,
                                                 int64_t total_rows) {
  if (num_tables < 0 || batch < 0 || num_indices < 0 || total_rows < 0) return 0;
  return neo::bkt_workspace(num_tables, batch, num_indices, total_rows);
}
