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
//   6. bkt_sort       persistent CTAs claim buckets (queued big ones first,
//                     then table-major order).  Per bucket: stable counting
//                     sort by row within the bucket (shared memory; <= 9-bit
//                     digits, one pass for the usual bucket; buckets larger
//                     than kCap go through global scratch in kCap chunks by
//                     the same stable passes), row heads compacted by a block
//                     scan.  Rows with more occurrences than a stage holds are
//                     split across every sub-warp of the CTA (contiguous
//                     pieces, partials combined in piece order) and updated
//                     here; the others are cut into row batches (consecutive
//                     rows that fit one stage) appended to a batch stream.
//   7. bkt_rows       persistent warp-specialised groups: a producer warp
//                     stages each batch's weight rows, optimizer state and
//                     upstream rows into shared memory with TMA bulk copies
//                     (cp.async.bulk, byte-counted mbarrier), consumer warps
//                     sum every row's upstream rows in order (sub-warp per
//                     row) and apply one optimizer step, storing to HBM.
//
// Everything is deterministic: the order of every floating-point sum depends
// only on the input.
#include <cuda.h>

#include <cstdio>
#include <string>

#include "bwd_common.cuh"

namespace neo {
namespace bkt {

constexpr int kMaxB = 2048;    // row buckets per table (count / scatter shared-memory histograms)
constexpr int kSMin = 4;       // smallest bucket: 16 rows
#ifndef NEO_BKT_CHB
#define NEO_BKT_CHB 1024
#endif
constexpr int kCHB = NEO_BKT_CHB;  // bags per count / scatter chunk
#ifndef NEO_BKT_SCW
#define NEO_BKT_SCW 8
#endif
constexpr int kScW = NEO_BKT_SCW;  // warps per count / scatter CTA
#ifndef NEO_BKT_CAP
#define NEO_BKT_CAP 2048
#endif
#ifndef NEO_BKT_UW
#define NEO_BKT_UW 8
#endif
constexpr int kCap = NEO_BKT_CAP;  // entries per bucket sorted in shared memory
constexpr int kUW = NEO_BKT_UW;    // warps per sort CTA
constexpr int kUT = kUW * kWarp;
constexpr int kDigit = 9;      // bits per stable counting pass
constexpr int kBins = 1 << kDigit;
constexpr int kLong = 64;      // rows with more occurrences are split across the CTA
constexpr int kEPL = 8;        // row elements per lane
constexpr int kMaxDim = kWarp * kEPL;
constexpr int kScanTile = 4096;  // 256 threads x 16
constexpr int kTarget = 1024;    // default occurrences per bucket
constexpr int kWCap = 1280;      // entries of a bucket one warp sorts (bkt_wsort_kernel)
constexpr int kBPT = kBins / kUT;  // digit bins per sort thread
static_assert(kBins % kUT == 0 && kCap % kUT == 0, "sort CTA geometry");
static_assert(kBins * kUW * 2 >= kCap * 4, "batch list aliases the histograms");
static_assert(kUW * kWarp * kEPL <= kCap, "long-row partials alias a sort buffer");

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
  int32_t* btab;     // [nb] table of each bucket
  uint8_t* bkind;    // [nb] 0 empty, 1 / 5 warp-sorted (9- / 10-bit rows), 2 CTA (shared memory), 3 CTA (global)
  int32_t* ctal;     // kind-2 buckets
  int32_t* big;      // queued big buckets
  int32_t* ctr;      // [0] CTA claim counter, [1] big-bucket count, [2] kind-2 count, [3] warp claim
                     // (9-bit buckets), [8] warp claim (10-bit buckets)
                     // counter, [4] capacity overflow, [5] hot rows,
                     // [6..7] one 64-bit counter: batches (low word), record units (high word)
  uint32_t* ent;     // bucketed entries (row_low << bag_bits | bag)
  uint32_t* ent2;    // bucket entries sorted by row (read by the row kernel)
  uint32_t* rec;     // row-batch records (16-byte units): {rows | entries << 8, table, -, -}, rows,
                     // row lengths (bytes), bags (entries padded to 4)
  uint2* hdr;        // per batch: {record offset, record size} in 16-byte units
  int64_t rec_cap;   // capacity of rec in 16-byte units
  int64_t hdr_cap;   // capacity of hdr
  uint4* longs;      // hot rows: {table | sorted list in ent2 << 31, row, first entry, entries}
  int64_t long_cap;
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
  if (threadIdx.x < 10) q.ctr[threadIdx.x] = 0;
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
  const int t = table_of_bucket(q.bbase, q.T, b);
  q.btab[b] = t;
  if (b + 1 == nbt) q.bstart[nbt] = en;
  const int n = en - st;
  // 1 / 5: one warp sorts it (bkt_wsort_kernel, 2^9 / 2^10 row bins); 2: a CTA, in shared memory;
  // 3: a CTA, through global scratch
  const int sb = q.sbits[t];
  const uint8_t kind = n == 0                            ? 0
                       : (n <= kWCap && sb <= kDigit)     ? 1
                       : (n <= kWCap && sb == kDigit + 1) ? 5
                       : (n <= kCap ? 2 : 3);
  q.bkind[b] = kind;
  if (kind == 3) q.big[atomicAdd(&q.ctr[1], 1)] = (int32_t)b;
  if (kind == 2) q.ctal[atomicAdd(&q.ctr[2], 1)] = (int32_t)b;
  if (kind == 5) atomicAdd(&q.ctr[9], 1);  // (the 10-bit warp sort exits at once without them)
}

// ---------------------------------------------------------------------------
// 5. stable scatter into buckets

__device__ __forceinline__ void st_u32_keep(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;\n" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

template <typename Idx>
__global__ void __launch_bounds__(kScW* kWarp) bkt_scatter_kernel(Params q, const Idx* __restrict__ indices) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t pol_keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
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
  // count pass: the next group's ids are in flight while this group's are counted
#ifndef NEO_BKT_CU
#define NEO_BKT_CU 8
#endif
  constexpr int kCU = NEO_BKT_CU;
  auto ld_id = [&](int64_t p) -> int64_t { return p < p1 ? (int64_t)indices[p] : -1; };
  {
    int64_t cur[kCU];
#pragma unroll
    for (int u = 0; u < kCU; ++u) cur[u] = ld_id(p0 + u * kWarp + lane);
    for (int64_t pb = p0; pb < p1; pb += kCU * kWarp) {
      int64_t nxt[kCU];
#pragma unroll
      for (int u = 0; u < kCU; ++u) nxt[u] = ld_id(pb + (kCU + u) * kWarp + lane);
#pragma unroll
      for (int u = 0; u < kCU; ++u)
        if (cur[u] >= 0 && cur[u] < H) atomicAdd(&wh[(int)(cur[u] >> s)], 1u);
#pragma unroll
      for (int u = 0; u < kCU; ++u) cur[u] = nxt[u];
    }
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
  // place pass, in buffer order.  Rounds of 32 consecutive entries; a window
  // of 32 bags (offsets relative to the window start, one per lane) resolves
  // each entry's bag; the next window's offsets and the next group's ids are
  // loaded ahead.  Within a round, equal buckets are ranked by lane
  // (match_any) and the group's leader reserves the slots with one shared
  // atomic, so rounds chain only through the atomics.
  const unsigned lt = lanemask_lt();
  auto win_off = [&](int64_t bw) -> int64_t { return bw + lane < wb1 ? off[bw + lane] : p1; };
  int64_t bw = wb0;
  int64_t obase = off[wb0];
  int64_t o64 = win_off(bw);
  int64_t onext = win_off(bw + kWarp);
  uint32_t orel = (uint32_t)(o64 - obase);
  int64_t wend = bw + kWarp < wb1 ? __shfl_sync(full, onext, 0) : p1;
#ifndef NEO_BKT_PU
#define NEO_BKT_PU 4
#endif
  constexpr int kPU = NEO_BKT_PU;
  int64_t cur[kPU];
#pragma unroll
  for (int u = 0; u < kPU; ++u) cur[u] = ld_id(p0 + u * kWarp + lane);
  for (int64_t pq = p0; pq < p1; pq += kPU * kWarp) {
    int64_t nxt[kPU];
#pragma unroll
    for (int u = 0; u < kPU; ++u) nxt[u] = ld_id(pq + (kPU + u) * kWarp + lane);
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
      const int64_t pb = pq + u * kWarp;
      if (pb >= p1) break;  // warp-uniform
      const int64_t p = pb + lane;
      const int64_t id = cur[u];
      int64_t lo = pb;  // first position of the round not yet placed
      for (;;) {
        const int64_t lim = min64(min64(pb + kWarp, p1), wend);
        const bool in = p >= lo && p < lim;
        // bag: the last window lane whose start is <= p
        const uint32_t prel = (uint32_t)(min64(max64(p, lo), lim - 1) - obase);
        const uint32_t ja = 31 - __clz(__ballot_sync(full, orel <= (uint32_t)(lo - obase)));
        const uint32_t jb = 31 - __clz(__ballot_sync(full, orel <= (uint32_t)(lim - 1 - obase)));
        uint32_t k = ja;
        if (ja != jb) {  // a bag starts inside the round: per-lane search
          k = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t ok = __shfl_sync(full, orel, k + step);
            if (ok <= prel) k += step;
          }
        }
        const bool valid = in && id >= 0 && id < H;
        const uint32_t bk = valid ? (uint32_t)(id >> s) : 0xffffffffu;
        const unsigned peers = __match_any_sync(full, bk);
        const int leader = __ffs(peers) - 1;
        uint32_t at = 0;
        if (valid && lane == leader) at = atomicAdd(&wh[bk], (uint32_t)__popc(peers));
        at = __shfl_sync(full, at, leader);
        // a bucket's entries land over the warp's lifetime: keep partially
        // written sectors in L2 (a partial-sector eviction costs a DRAM
        // read-modify-write)
        if (valid)
          st_u32_keep(q.ent + at + __popc(peers & lt), (((uint32_t)id & rmask) << q.bag_bits) | (uint32_t)(bw + k),
                      pol_keep);
        if (lim == min64(pb + kWarp, p1)) break;
        // the round continues past the window: the next window
        lo = lim;
        bw += kWarp;
        obase = wend;
        o64 = onext;
        onext = win_off(bw + kWarp);
        orel = (uint32_t)(o64 - obase);
        wend = bw + kWarp < wb1 ? __shfl_sync(full, onext, 0) : p1;
      }
    }
#pragma unroll
    for (int u = 0; u < kPU; ++u) cur[u] = nxt[u];
  }
}

// ---------------------------------------------------------------------------
// 6. per-bucket row sort; hot rows updated here; short rows -> row batches

struct alignas(16) USmem {
  uint32_t a[kCap];
  uint32_t b[kCap];
  int32_t rbeg[kCap + 1];
  uint16_t hist[kBins * kUW];  // [bin][warp]; after the sort: the window's batches
  int32_t cursor[kBins];
  int32_t tot[kBins];
  int32_t longs[kCap / 2 + 2];
  int32_t wsum[kUW + 1];
  int32_t nlong;
  int32_t nbat;
  int32_t hbase;
  int32_t rbase16;  // record base of the window
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
  for (int d = tid; d < kBins; d += kUT) sm.tot[d] = 0;
  __syncthreads();
  for (int64_t i = tid; i < n; i += kUT) atomicAdd(&sm.tot[(src[i] >> shift) & dm], 1);
  __syncthreads();
  int v[kBPT], loc = 0;  // bins kBPT*tid .. : a local prefix, then one block scan
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    const int d = kBPT * tid + k;
    v[k] = d < nbins ? sm.tot[d] : 0;
    loc += v[k];
  }
  int total;
  int ex = block_scan_excl<kUT>(loc, sm.wsum, &total);
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    sm.cursor[kBPT * tid + k] = ex;
    ex += v[k];
  }
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
// (jmax - j0) is warp-uniform.  KAHAN: compensated summation (hot rows, whose
// thousands of terms would otherwise lose f32 accuracy to cancellation)
template <typename W, typename G, int OPT, bool KAHAN = false>
__device__ __forceinline__ void gather_sum(const RowCtx<W, G, OPT>& c, const uint32_t* list, int64_t j0, int64_t j1,
                                           int64_t jmax, bool col, int sl, float (&acc)[kEPL]) {
  float comp[kEPL];
#pragma unroll
  for (int e = 0; e < kEPL; ++e) comp[e] = 0.f;
  auto add = [&](const float (&x)[kEPL]) {
#pragma unroll
    for (int e = 0; e < kEPL; ++e) {
      if (KAHAN) {
        const float y = x[e] - comp[e];
        const float t = acc[e] + y;
        comp[e] = (t - acc[e]) - y;
        acc[e] = t;
      } else {
        acc[e] += x[e];
      }
    }
  };
  for (int64_t j = j0; j < jmax; j += 2) {
    const bool h0 = col && j < j1, h1 = col && j + 1 < j1;
    const uint32_t e0 = h0 ? list[j] : 0u;
    const uint32_t e1 = h1 ? list[j + 1] : 0u;
    float x0[kEPL], x1[kEPL];
    if (h0) ld8<G>(c.grad + (int64_t)(e0 & c.bmask) * c.stride + c.doff + sl * kEPL, x0);
    if (h1) ld8<G>(c.grad + (int64_t)(e1 & c.bmask) * c.stride + c.doff + sl * kEPL, x1);
    if (h0) add(x0);
    if (h1) add(x1);
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

// bytes one row batch occupies in a row-kernel stage: per row the weight row
// (+ its element-wise state); per stage 128 bytes of alignment and, for the
// row-wise state, a moment span of up to kMomSpan bytes
constexpr int kMomSpan = 1024;
template <typename W, typename G, int OPT>
__host__ __device__ __forceinline__ int stage_row_bytes(int D) {
  const int wb = OPT == NEO_OPT_NONE ? 0 : D * (int)sizeof(W);
  return wb + (OPT == NEO_OPT_ADAGRAD ? D * 4 : 0);
}
template <int OPT>
__host__ __device__ __forceinline__ int stage_fixed_bytes() {
  return 128 + (OPT == NEO_OPT_ROWWISE_ADAGRAD ? kMomSpan : 0);
}

#ifndef NEO_BKT_STAGE_KB
#define NEO_BKT_STAGE_KB 24
#endif
constexpr int kStageBytes = NEO_BKT_STAGE_KB * 1024;  // one row-kernel stage
constexpr int kMaxRows = 32;            // rows per batch (one producer lane each)
constexpr int kMaxEnt = 96;             // entries per batch (gather4 groups: <= 24)
constexpr int kRecMax16 = 1 + kMaxRows / 4 + kMaxRows / 16 + kMaxEnt / 4;  // record size bound (16-byte units)

__host__ __device__ __forceinline__ int rec_units(int m, int nent) {
  const unsigned um = (unsigned)m, un = (unsigned)nent;
  return (int)(1u + ((um + 3u) >> 2) + ((um + 15u) >> 4) + ((un + 3u) >> 2));
}

// longest row staged by the row kernel; longer rows are updated by the sort kernel
template <typename W, typename G, int OPT>
__device__ __forceinline__ int long_threshold(int D) {
  const int gb = D * (int)sizeof(G);
  int lim = (kStageBytes - stage_fixed_bytes<OPT>() - stage_row_bytes<W, G, OPT>(D)) / gb - 3;  // padded to 4
  if (lim > kLong) lim = kLong;
  return lim;
}

// window rows [0, nr) of list (starts in sm.rbeg): rows longer than the
// threshold are split across the CTA and updated here; the others are cut
// into batches (consecutive rows, <= kMaxRows rows, <= kMaxEnt entries,
// <= kStageBytes staged bytes, never across a long row) appended to the
// global batch stream for the row kernel
template <typename W, typename G, int OPT>
__device__ __forceinline__ void emit_rows(const RowCtx<W, G, OPT>& c, const Params& q, int t, int64_t bs,
                                          int32_t rowidx0, const uint32_t* list, int nr, USmem& sm) {
  const unsigned full = 0xffffffffu;
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const int lth = long_threshold<W, G, OPT>(c.D);
  const int rowb = stage_row_bytes<W, G, OPT>(c.D);
  const int gb = c.D * (int)sizeof(G);
  if (tid == 0) {
    sm.nbat = 0;
    sm.nlong = 0;
  }
  __syncthreads();
  // greedy batching inside 32-row chunks, one warp per chunk; batches and
  // long rows are appended in any order (each row is updated exactly once,
  // so the order of batches does not change any result)
  uint32_t* bat = reinterpret_cast<uint32_t*>(sm.hist);  // the sort's histograms are free now
  const int nchunks = (nr + kWarp - 1) / kWarp;
  for (int ck = warp; ck < nchunks; ck += kUW) {
    const int cend = min(nr, ck * kWarp + kWarp);
    int base = ck * kWarp;
    while (base < cend) {
      const int r = base + lane;
      const bool v = r < cend;
      const int len = v ? sm.rbeg[r + 1] - sm.rbeg[r] : 0;
      const bool lg = v && len > lth;
      const unsigned lgm = __ballot_sync(full, lg);
      const int firstlong = lgm ? __ffs(lgm) - 1 : kWarp;
      if (firstlong == 0) {
        if (lane == 0) sm.longs[atomicAdd(&sm.nlong, 1)] = base;
        ++base;
        continue;
      }
      int cost = v && !lg ? rowb + len * gb : 0;  // + 128 bytes of region alignment below
      int ent = v && !lg ? len : 0;
#pragma unroll
      for (int o = 1; o < kWarp; o <<= 1) {
        const int x = __shfl_up_sync(full, cost, o), y = __shfl_up_sync(full, ent, o);
        if (lane >= o) {
          cost += x;
          ent += y;
        }
      }
      const bool fits =
          v && lane < firstlong && cost + stage_fixed_bytes<OPT>() + 3 * gb <= kStageBytes && ent <= kMaxEnt;
      const int m = __popc(__ballot_sync(full, fits));  // >= 1: one short row always fits
      if (lane == 0) bat[atomicAdd(&sm.nbat, 1)] = ((uint32_t)base << 8) | (uint32_t)m;
      base += m;
    }
  }
  __syncthreads();
  // records: offsets by a block scan over the window's batches, one
  // reservation per window, then one warp writes each record
  const int nbat = sm.nbat;
  uint32_t* roff = reinterpret_cast<uint32_t*>(list == sm.a ? sm.b : sm.a);  // free sort buffer
  {
    int carry = 0;
    for (int i0 = 0; i0 < nbat; i0 += kUT) {
      const int i = i0 + tid;
      int sz = 0;
      if (i < nbat) {
        const uint32_t bw = bat[i];
        const int r0 = (int)(bw >> 8), m = (int)(bw & 0xff);
        sz = rec_units(m, sm.rbeg[r0 + m] - sm.rbeg[r0]);
      }
      int tot;
      const int ex = block_scan_excl<kUT>(sz, sm.wsum, &tot);
      if (i < nbat) roff[i] = (uint32_t)(carry + ex);
      carry += tot;
    }
    if (tid == 0) {
      // one 64-bit reservation: batches (low word) and record units (high word)
      const unsigned long long old =
          nbat ? atomicAdd(reinterpret_cast<unsigned long long*>(q.ctr + 6),
                           ((unsigned long long)carry << 32) | (unsigned long long)nbat)
               : 0ull;
      sm.hbase = (int)(old & 0xffffffffull);
      const int rb = (int)(old >> 32);
      sm.rbase16 = rb;
      if ((int64_t)sm.hbase + nbat > q.hdr_cap || (int64_t)rb + carry > q.rec_cap) {
        atomicExch(&q.ctr[4], 1);  // capacity bound violated: the row kernel traps
        sm.nbat = 0;
      }
    }
  }
  __syncthreads();
  const uint32_t rbase = (uint32_t)sm.rbase16;
  for (int i = warp; i < sm.nbat; i += kUW) {
    const uint32_t bw = bat[i];
    const int r0 = (int)(bw >> 8), m = (int)(bw & 0xff);
    const int e0 = sm.rbeg[r0], nent = sm.rbeg[r0 + m] - e0;
    const uint32_t o16 = rbase + roff[i];
    uint32_t* rec = q.rec + (int64_t)o16 * 4;
    if (lane == 0) {
      rec[0] = (uint32_t)m | ((uint32_t)nent << 8);
      rec[1] = (uint32_t)t;
      q.hdr[sm.hbase + i] = make_uint2(o16, (uint32_t)rec_units(m, nent));
    }
    const int rw = 4 + 4 * ((m + 3) / 4);  // first length byte at word rw
    if (lane < m) {
      const int rs = sm.rbeg[r0 + lane];
      rec[4 + lane] = (uint32_t)(c.row0 + (int64_t)(list[rs] >> c.bag_bits));
      reinterpret_cast<uint8_t*>(rec + rw)[lane] = (uint8_t)(sm.rbeg[r0 + lane + 1] - rs);
    }
    uint32_t* bags = rec + rw + 4 * ((m + 15) / 16);
    const int n4 = (nent + 3) & ~3;
    for (int j = lane; j < n4; j += kWarp) bags[j] = list[e0 + min(j, nent - 1)] & c.bmask;
  }
  __syncthreads();  // roff's buffer is reused for the long-row partials
  // long rows are left to bkt_long_kernel (APPLY phase), so this kernel never
  // touches the tables and may run under the forward: their sorted entries
  // must be in global memory (ent2 for shared-memory lists)
  const int nl = sm.nlong;
  if (nl > 0) {
    uint32_t buf = 1;
    if (__isShared(list)) {
      for (int i = tid; i < sm.rbeg[nr]; i += kUT) q.ent2[bs + i] = list[i];
    } else {
      buf = list == q.ent + bs ? 0u : 1u;
    }
    if (tid == 0) sm.hbase = atomicAdd(&q.ctr[5], nl);
    __syncthreads();
    const int lb = sm.hbase;
    if ((int64_t)lb + nl > q.long_cap) {
      if (tid == 0) atomicExch(&q.ctr[4], 1);
    } else {
      for (int l = tid; l < nl; l += kUT) {
        const int r = sm.longs[l];
        const int rb = sm.rbeg[r];
        q.longs[lb + l] = make_uint4((uint32_t)t | (buf << 31), (uint32_t)(c.row0 + (int64_t)(list[rb] >> c.bag_bits)),
                                     (uint32_t)(bs + rb), (uint32_t)(sm.rbeg[r + 1] - rb));
      }
    }
  }
  __syncthreads();
}

// APPLY phase: one CTA per hot row (more occurrences than a row-kernel stage
// holds).  Every sub-warp sums a contiguous piece of the row's sorted
// occurrences with compensated summation; sub-warp 0 of warp 0 combines the
// pieces in order and applies the row's single optimizer step.
constexpr int kLW = 8;  // warps per long-row CTA

template <typename W, typename G, int OPT>
__global__ void __launch_bounds__(kLW* kWarp) bkt_long_kernel(Params q, SegParams p) {
  __shared__ float part[kLW * kWarp * kEPL];
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int nl = q.ctr[5];
  for (int l = blockIdx.x; l < nl; l += gridDim.x) {
    const uint4 rec = q.longs[l];
    const int t = (int)(rec.x & 0x7fffffffu);
    const uint32_t* list = ((rec.x >> 31) ? q.ent2 : q.ent) + rec.z;
    const int64_t row = rec.y, len = rec.w;
    RowCtx<W, G, OPT> c;
    c.grad = reinterpret_cast<const G*>(p.grad);
    c.stride = p.grad_stride;
    c.doff = p.dim_offsets[t];
    c.D = p.dim_offsets[t + 1] - c.doff;
    c.wt = reinterpret_cast<W*>(OPT == NEO_OPT_NONE ? p.dense_grads[t] : p.weights[t]);
    c.mom = (OPT == NEO_OPT_ROWWISE_ADAGRAD || OPT == NEO_OPT_ADAGRAD) ? reinterpret_cast<float*>(p.moments[t])
                                                                       : nullptr;
    c.row0 = 0;
    c.bag_bits = q.bag_bits;
    c.bmask = (uint32_t)((1u << q.bag_bits) - 1u);
    c.lr = (float)p.lr;
    c.eps = (float)p.eps;
    c.invD = 1.0f / (float)c.D;
    int S = 1;
    while (S * kEPL < c.D) S <<= 1;
    const int R = kWarp / S, sub = lane / S, sl = lane % S;
    const bool col = sl * kEPL < c.D;
    const int nsub = kLW * R;
    const int k = warp * R + sub;
    float acc[kEPL];
#pragma unroll
    for (int e = 0; e < kEPL; ++e) acc[e] = 0.f;
    const int64_t a0 = len * k / nsub, a1 = len * (k + 1) / nsub;
    const int64_t span = (int64_t)__reduce_max_sync(full, (unsigned)(a1 - a0));
    gather_sum<W, G, OPT, true>(c, list, a0, a1, a0 + span, col, sl, acc);
    if (col) {
#pragma unroll
      for (int e = 0; e < kEPL; ++e) part[(k * S + sl) * kEPL + e] = acc[e];
    }
    __syncthreads();
    if (warp == 0) {
      const bool own = sub == 0;
      float wv[kEPL], mv[kEPL], mrow;
      prefetch_row<W, G, OPT>(c, row, own, col, sl, wv, mv, mrow);
#pragma unroll
      for (int e = 0; e < kEPL; ++e) acc[e] = 0.f;
      if (own && col) {
        for (int qq = 0; qq < nsub; ++qq)
#pragma unroll
          for (int e = 0; e < kEPL; ++e) acc[e] += part[(qq * S + sl) * kEPL + e];
      }
      finish_row<W, G, OPT>(c, row, own, col, S, sub, sl, wv, mv, mrow, acc);
    }
    __syncthreads();
  }
}

// sort one bucket (entries in sm.a when it fits shared memory, else in
// ent + bs) by row, then emit its row batches / hot rows window by window
template <typename W, typename G, int OPT>
__device__ __forceinline__ void sort_bucket(const Params& q, const SegParams& p, int b, int t, int64_t bs, int64_t n,
                                            USmem& sm) {
  const int tid = threadIdx.x;
  const int s = q.sbits[t];
  RowCtx<W, G, OPT> c;
  c.doff = p.dim_offsets[t];
  c.D = p.dim_offsets[t + 1] - c.doff;
  c.row0 = (int64_t)(b - q.bbase[t]) << s;
  c.bag_bits = q.bag_bits;
  c.bmask = (uint32_t)((1u << q.bag_bits) - 1u);
  // stable LSD passes over the s row bits (entries arrive in buffer order)
  const int passes = (s + kDigit - 1) / kDigit;
  const int wbits = (s + passes - 1) / passes;
  const bool small = n <= kCap;
  const uint32_t* list = small ? sm.a : q.ent + bs;
  for (int k = 0; k < passes; ++k) {
    const int nbits = min(wbits, s - k * wbits);
    uint32_t* dst = small ? ((k & 1) ? sm.a : sm.b) : ((k & 1) ? q.ent + bs : q.ent2 + bs);
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
      if ((hm >> j) & 1u) sm.rbeg[ex++] = (int32_t)(i0 + j - pos);
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
      sm.rbeg[nr] = (int32_t)(end - pos);
      sm.nrows = nr;
    }
    __syncthreads();
    const int nrw = sm.nrows;
    emit_rows<W, G, OPT>(c, q, t, bs + pos, 0, list + pos, nrw, sm);
    pos += sm.rbeg[nrw];
    __syncthreads();
  }
}

template <typename W, typename G, int OPT>
__global__ void __launch_bounds__(kUT, 1024 / kUT) bkt_sort_kernel(Params q, SegParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  USmem& sm = *reinterpret_cast<USmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int nbig = q.ctr[1];
  // 1. buckets larger than shared memory first (claimed; global passes); the
  // first claim past the queue is this CTA's first regular bucket
  int first = -1;
  for (;;) {
    if (tid == 0) {
      const int idx = atomicAdd(&q.ctr[0], 1);
      sm.bucket = idx < nbig ? q.big[idx] : -1;
      sm.table = idx - nbig;  // regular bucket index when past the queue
    }
    __syncthreads();
    const int b = sm.bucket;
    if (b < 0) {
      first = sm.table;
      break;
    }
    const int64_t bs = q.bstart[b];
    sort_bucket<W, G, OPT>(q, p, b, q.btab[b], bs, q.bstart[b + 1] - bs, sm);
  }
  // 2. the others in claim order (table-major, so the row kernel's batch
  // stream keeps each table's upstream slice L2-resident); the next bucket is
  // claimed and its entries loaded into registers while this one is sorted
  constexpr int kPer = kCap / kUT;
  const int ncta = q.ctr[2];
  auto claim = [&]() -> int64_t {  // thread 0 only: the next kind-2 bucket
    const int k = atomicAdd(&q.ctr[0], 1) - nbig;
    return k < ncta ? q.ctal[k] : -1;
  };
  __syncthreads();  // every thread has read sm.bucket / sm.table
  if (tid == 0) sm.bucket = first < ncta ? q.ctal[first] : -1;
  __syncthreads();
  int64_t jn = sm.bucket;
  int64_t bsn = 0;
  int nn = 0, tn = 0;
  uint32_t pre[kPer];
  auto prefetch = [&]() {
    if (jn >= 0) {
      bsn = q.bstart[jn];
      nn = (int)(q.bstart[jn + 1] - bsn);
      tn = q.btab[jn];
    } else {
      nn = 0;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = tid + k * kUT;
      pre[k] = i < nn ? q.ent[bsn + i] : 0u;
    }
  };
  prefetch();
  while (jn >= 0) {
    const int64_t j = jn, bs = bsn;
    const int n = nn, t = tn;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = tid + k * kUT;
      if (i < n) sm.a[i] = pre[k];
    }
    if (tid == 0) sm.bucket = (int)claim();
    __syncthreads();
    jn = sm.bucket;
    prefetch();  // in flight during the sort below
    sort_bucket<W, G, OPT>(q, p, (int)j, t, bs, n, sm);
  }
}

// ---------------------------------------------------------------------------
// 6b. warp-per-bucket sort: the common bucket (<= kWCap entries, <= 9 row
// bits) is sorted by ONE warp with no block barriers: a warp-private digit
// histogram (match_any-aggregated), one warp scan that also lists the
// touched rows, a stable match_any placement into shared memory, greedy
// batching of 32-row chunks from one prefix scan each, and the records.

template <int BINS>
struct alignas(16) WSmem {
  uint32_t out[kWCap];       // the bucket's entries sorted by row
  uint32_t hist[BINS];       // digit counts, then cursors; after the placement: the batches
  uint16_t rstart[BINS + 2];
};
constexpr int kWW = 8;              // warps per CTA
constexpr int kWR = kWCap / kWarp;  // entries per lane (held in registers)
static_assert(kWCap % kWarp == 0, "warp-sort capacity");

// BINS = 512: buckets of <= 2^9 rows (kind 1); 1024: 2^10-row buckets (kind 5)
template <typename W, typename G, int OPT, int BINS>
__global__ void __launch_bounds__(kWW* kWarp, 3) bkt_wsort_kernel(Params q, SegParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  WSmem<BINS>& sm = reinterpret_cast<WSmem<BINS>*>(smem_raw)[warp];
  constexpr uint8_t kKind = BINS == kBins ? 1 : 5;
  int32_t* const claim_ctr = q.ctr + (BINS == kBins ? 3 : 8);
  const int64_t nbt = q.bbase[q.T];
  const uint32_t bmask = (uint32_t)((1u << q.bag_bits) - 1u);
  const unsigned lt = lanemask_lt();
  const int bb = q.bag_bits;
  auto claim = [&]() -> int64_t {
    int64_t j = -1;
    // buckets are claimed in bucket (table-major) order: the row kernel's
    // batch stream then keeps each table's upstream slice L2-resident
    if (lane == 0 && (BINS == kBins || q.ctr[9] > 0)) {
      for (;;) {
        const int64_t jj = atomicAdd(claim_ctr, 1);
        if (jj >= nbt) break;
        if (q.bkind[jj] == kKind) {
          j = jj;
          break;
        }
      }
    }
    return __shfl_sync(full, j, 0);
  };
  int64_t j = claim();
  while (j >= 0) {
    const int64_t jn = claim();  // the next bucket, claimed early (its metadata loads overlap this one)
    const int t = q.btab[j];
    const int sb = q.sbits[t];
    const int64_t bs = q.bstart[j];
    const int n = (int)(q.bstart[j + 1] - bs);
    // the bucket's entries in registers (buffer order: entry k*32 + lane),
    // all loads in flight at once; no shared-memory staging buffer, so three
    // CTAs (24 warps) fit an SM
    uint32_t e[kWR];
#pragma unroll
    for (int k = 0; k < kWR; ++k) {
      const int i = k * kWarp + lane;
      e[k] = i < n ? q.ent[bs + i] : 0u;
    }
    const int nbins = 1 << sb;
    const uint32_t dm = (uint32_t)nbins - 1;
    const int32_t doff = p.dim_offsets[t];
    const int D = p.dim_offsets[t + 1] - doff;
    const int64_t row0 = (int64_t)(j - q.bbase[t]) << sb;
    for (int d = lane; d < nbins; d += kWarp) sm.hist[d] = 0;
    __syncwarp();
    // 1. digit histogram (counts only: order does not matter here)
#pragma unroll
    for (int k = 0; k < kWR; ++k) {
      if (k * kWarp >= n) break;
      if (k * kWarp + lane < n) atomicAdd(&sm.hist[(e[k] >> bb) & dm], 1u);
    }
    __syncwarp();
    // 2. one scan: cursors (exclusive starts) and the touched rows in order
    const int per = (nbins + kWarp - 1) / kWarp;
    int cnt = 0, nz = 0;
    for (int k = 0; k < per; ++k) {
      const int d = lane * per + k;
      const int c = d < nbins ? (int)sm.hist[d] : 0;
      cnt += c;
      nz += c > 0;
    }
    int ex = cnt, exn = nz;
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
      const int x = __shfl_up_sync(full, ex, o), y = __shfl_up_sync(full, exn, o);
      if (lane >= o) {
        ex += x;
        exn += y;
      }
    }
    const int nrows = __shfl_sync(full, exn, kWarp - 1);
    ex -= cnt;
    exn -= nz;
    for (int k = 0; k < per; ++k) {
      const int d = lane * per + k;
      if (d < nbins) {
        const int c = (int)sm.hist[d];
        if (c > 0) sm.rstart[exn++] = (uint16_t)ex;
        sm.hist[d] = (uint32_t)ex;
        ex += c;
      }
    }
    if (lane == 0) sm.rstart[nrows] = (uint16_t)n;
    __syncwarp();
    // 3. stable placement (entries arrive in buffer order); the group leader
    // reserves the slots with one shared atomic
#pragma unroll
    for (int k = 0; k < kWR; ++k) {
      if (k * kWarp >= n) break;
      const bool v = k * kWarp + lane < n;
      const uint32_t d = v ? (e[k] >> bb) & dm : 0xffffffffu;
      const unsigned peers = __match_any_sync(full, d);
      const int leader = __ffs(peers) - 1;
      uint32_t at = 0;
      if (v && lane == leader) at = atomicAdd(&sm.hist[d], (uint32_t)__popc(peers));
      at = __shfl_sync(full, at, leader);
      if (v) sm.out[at + __popc(peers & lt)] = e[k];
    }
    __syncwarp();
    // 4. batches of 32-row chunks (greedy cuts from one prefix scan per chunk);
    // rows longer than a stage go to the hot-row list
    uint32_t* bat = sm.hist;
    const int lth = long_threshold<W, G, OPT>(D);
    const int rowb = stage_row_bytes<W, G, OPT>(D);
    const int gb = D * (int)sizeof(G);
    const int lim = kStageBytes - stage_fixed_bytes<OPT>() - 3 * gb;
    int nbat = 0;
    for (int ck = 0; ck < nrows; ck += kWarp) {
      const int r = ck + lane;
      const bool v = r < nrows;
      const int len = v ? sm.rstart[r + 1] - sm.rstart[r] : 0;
      const bool lg = v && len > lth;
      const unsigned lgm = __ballot_sync(full, lg);
      if (lg) {  // hot row: its sorted entries to ent2, a record for bkt_long_kernel
        const int l = atomicAdd(&q.ctr[5], 1);
        if (l < q.long_cap)
          q.longs[l] = make_uint4((uint32_t)t | (1u << 31),
                                  (uint32_t)(row0 + ((sm.out[sm.rstart[r]] >> bb) & dm)),
                                  (uint32_t)(bs + sm.rstart[r]), (uint32_t)len);
        else
          atomicExch(&q.ctr[4], 1);
      }
      for (unsigned h = lgm; h;) {
        const int k = __ffs(h) - 1;
        h &= h - 1;
        const int a0 = sm.rstart[ck + k], a1 = sm.rstart[ck + k + 1];
        for (int i = a0 + lane; i < a1; i += kWarp) q.ent2[bs + i] = sm.out[i];
      }
      int cost = v && !lg ? rowb + len * gb : 0;
      int ent = v && !lg ? len : 0;
#pragma unroll
      for (int o = 1; o < kWarp; o <<= 1) {
        const int x = __shfl_up_sync(full, cost, o), y = __shfl_up_sync(full, ent, o);
        if (lane >= o) {
          cost += x;
          ent += y;
        }
      }
      const int m_chunk = min(kWarp, nrows - ck);
      int base = 0;
      while (base < m_chunk) {
        if ((lgm >> base) & 1u) {
          ++base;
          continue;
        }
        const unsigned after = lgm & ~((2u << base) - 1u);
        const int stop = after ? __ffs(after) - 1 : m_chunk;  // the batch ends before the next hot row
        const int c0 = base ? __shfl_sync(full, cost, base - 1) : 0;  // base is warp-uniform
        const int e0 = base ? __shfl_sync(full, ent, base - 1) : 0;
        const bool fits = lane >= base && lane < stop && cost - c0 <= lim && ent - e0 <= kMaxEnt;
        const int m = __popc(__ballot_sync(full, fits));  // >= 1: a short row always fits
        if (lane == 0) bat[nbat] = ((uint32_t)(ck + base) << 8) | (uint32_t)m;
        ++nbat;
        base += m;
      }
    }
    __syncwarp();
    // 5. records: sizes -> total (warp scans), one 64-bit reservation per bucket
    int tot = 0;
    for (int i0 = 0; i0 < nbat; i0 += kWarp) {
      const int i = i0 + lane;
      int sz = 0;
      if (i < nbat) {
        const uint32_t bw = bat[i];
        const int r0 = (int)(bw >> 8), m = (int)(bw & 0xff);
        sz = rec_units(m, sm.rstart[r0 + m] - sm.rstart[r0]);
      }
      tot += __reduce_add_sync(full, (unsigned)sz);
    }
    unsigned long long old = 0;
    if (lane == 0 && nbat)
      old = atomicAdd(reinterpret_cast<unsigned long long*>(q.ctr + 6),
                      ((unsigned long long)tot << 32) | (unsigned long long)nbat);
    old = __shfl_sync(full, old, 0);
    const int hbase = (int)(old & 0xffffffffull);
    uint32_t o16 = (uint32_t)(old >> 32);
    if ((int64_t)hbase + nbat > q.hdr_cap || (int64_t)o16 + tot > q.rec_cap) {
      if (lane == 0) atomicExch(&q.ctr[4], 1);
      nbat = 0;
    }
    // headers and each record's first unit, lane-parallel over the batches
    {
      uint32_t carry = o16;
      for (int i0 = 0; i0 < nbat; i0 += kWarp) {
        const int i = i0 + lane;
        uint32_t sz = 0, w0 = 0;
        if (i < nbat) {
          const uint32_t bw = bat[i];
          const int r0 = (int)(bw >> 8), m = (int)(bw & 0xff);
          const uint32_t nent = (uint32_t)(sm.rstart[r0 + m] - sm.rstart[r0]);
          sz = (uint32_t)rec_units(m, (int)nent);
          w0 = (uint32_t)m | (nent << 8);
        }
        uint32_t incl = sz;
#pragma unroll
        for (int o = 1; o < kWarp; o <<= 1) {
          const uint32_t x = __shfl_up_sync(full, incl, o);
          if (lane >= o) incl += x;
        }
        const uint32_t at = carry + incl - sz;
        if (i < nbat) {
          q.hdr[hbase + i] = make_uint2(at, sz);
          *reinterpret_cast<uint4*>(q.rec + (int64_t)at * 4) = make_uint4(w0, (uint32_t)t, 0u, 0u);
        }
        carry += __shfl_sync(full, incl, kWarp - 1);
      }
    }
    for (int i = 0; i < nbat; ++i) {
      const uint32_t bw = bat[i];
      const int r0 = (int)(bw >> 8), m = (int)(bw & 0xff);
      const int rs = lane < m ? sm.rstart[r0 + lane] : 0;
      const int rs1 = lane < m ? sm.rstart[r0 + lane + 1] : 0;
      const int e0 = __shfl_sync(full, rs, 0);
      const int nent = __shfl_sync(full, rs1, m - 1) - e0;
      uint32_t* rec = q.rec + (int64_t)o16 * 4;
      const unsigned mu = (unsigned)m;
      const int rw = 4 + 4 * (int)((mu + 3u) >> 2);
      if (lane < m) {
        rec[4 + lane] = (uint32_t)(row0 + ((sm.out[rs] >> bb) & dm));
        reinterpret_cast<uint8_t*>(rec + rw)[lane] = (uint8_t)(rs1 - rs);
      }
      uint32_t* bags = rec + rw + 4 * (int)((mu + 15u) >> 4);
      const int n4 = (nent + 3) & ~3;
      for (int jx = lane; jx < n4; jx += kWarp) bags[jx] = sm.out[e0 + min(jx, nent - 1)] & bmask;
      o16 += (uint32_t)rec_units(m, nent);
    }
    __syncwarp();
    j = jn;
  }
}

// ---------------------------------------------------------------------------
// 7. row kernel: warp-specialised groups (one producer + kRC consumers) over
// the batch stream.  The producer stages each batch's weight rows, optimizer
// state and upstream rows into a shared-memory stage with TMA bulk copies
// (cp.async.bulk, completion counted in bytes on the stage's mbarrier), the
// consumers sum each row's upstream rows in order and apply one step.

#ifndef NEO_BKT_RG
#define NEO_BKT_RG 4
#endif
#ifndef NEO_BKT_RC
#define NEO_BKT_RC 4
#endif
#ifndef NEO_BKT_RS
#define NEO_BKT_RS 2
#endif
constexpr int kRG = NEO_BKT_RG;  // groups per CTA
constexpr int kRC = NEO_BKT_RC;  // consumer warps per group
constexpr int kRS = NEO_BKT_RS;  // stages per group
constexpr int kRT = kRG * (1 + kRC) * kWarp;

constexpr int kRQ = 3;  // record ring slots per group (records two batches ahead)

struct StageMeta {
  int32_t m;       // rows (-1: end of stream)
  int32_t nent;
  int32_t t;
  uint32_t mlo;    // row-wise state: first row of the staged moment span (~0u: read from HBM)
  uint32_t row[kMaxRows];
  uint16_t eoff[kMaxRows];
  uint8_t len[kMaxRows];
};

struct RowSmem {
  uint64_t full[kRG][kRS];
  uint64_t empty[kRG][kRS];
  uint64_t recbar[kRG][kRQ];
  StageMeta meta[kRG][kRS];
  alignas(128) uint32_t rec[kRG][kRQ][kRecMax16 * 4];
  alignas(128) unsigned char data[kRG][kRS][kStageBytes];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(1000000)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
// this thread's earlier cp.async copies complete the barrier's phase too
__device__ __forceinline__ void mbar_arrive_cp(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
// four upstream rows (bags r0..r3, columns from col) -> consecutive smem rows
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int col, uint32_t r0, uint32_t r1,
                                        uint32_t r2, uint32_t r3, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(smem_addr(dst)),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st16_hint(void* gmem, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(gmem), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// NEO_BKT_PROF builds: clock64 breakdown of the row kernel's roles
// (diagnostics; read with neo_bkt_prof)
#ifdef NEO_BKT_PROF
__device__ unsigned long long g_bkt_prof[12];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(k, x) \
  if (lane == 0) atomicAdd(&g_bkt_prof[k], (unsigned long long)(x))
#else
#define PROF_T(v)
#define PROF_ADD(k, x)
#endif

template <typename W, typename G, int OPT>
__global__ void __launch_bounds__(kRT, 1) bkt_rows_kernel(Params q, SegParams p,
                                                          const __grid_constant__ CUtensorMap gmap, int32_t tma_dim) {
  extern __shared__ __align__(16) unsigned char smem_raw[];  // dynamic smem starts 1024-aligned
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int g = warp / (1 + kRC), role = warp % (1 + kRC);  // role 0 = producer
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRG; ++i)
      for (int s = 0; s < kRS; ++s) {
        mbar_init(&sm.full[i][s], 1);  // producer lane 0 (arrive + expected bytes)
        mbar_init(&sm.empty[i][s], kRC);
      }
    for (int i = 0; i < kRG; ++i)
      for (int r = 0; r < kRQ; ++r) mbar_init(&sm.recbar[i][r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  constexpr int kVW = 16 / (int)sizeof(W);  // W elements per 16-byte vector
  if (role == 0) {
    // ------------------------------------------------------------ producer
    // Everything this warp moves goes through the TMA engine: per-lane global
    // loads / cp.async stall a warp under this much memory traffic, TMA ops
    // do not.  Per batch: the record (rows, lengths, bags) was bulk-copied
    // into the record ring two batches ahead; upstream rows as tile::gather4
    // ops (four rows each) or one bulk copy per row; weight rows (and
    // element-wise state) as one bulk copy per run of consecutive rows; the
    // row-wise moments as one 16-byte-aligned span.
    if (q.ctr[4] != 0) __trap();  // the sort kernel overflowed a capacity bound
    const int64_t nhdr = q.ctr[6];
    const int64_t P = (int64_t)gridDim.x * kRG;
    const G* gbase = reinterpret_cast<const G*>(p.grad);
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_first = policy_evict_first();
    int s = 0;
    uint32_t ephase = 1;  // stages start empty
    int64_t i = (int64_t)blockIdx.x * kRG + g;
    auto hdr_at = [&](int64_t k) { return k < nhdr ? q.hdr[k] : make_uint2(0, 0); };
    auto fetch_rec = [&](int slot, const uint2& hh, bool ok) {
      if (ok && lane == 0) {
        mbar_arrive_tx(&sm.recbar[g][slot], hh.y * 16);
        bulk_g2s(sm.rec[g][slot], q.rec + (int64_t)hh.x * 4, hh.y * 16, &sm.recbar[g][slot], pol_first);
      }
    };
    uint2 hC = hdr_at(i + 2 * P);
    fetch_rec(0, hdr_at(i), i < nhdr);
    fetch_rec(1, hdr_at(i + P), i + P < nhdr);
    int rs = 0;
    uint32_t rph = 0;  // parity of the ring pass
    int tcur = -1, D = 0, wb = 0, gb = 0;
    int32_t doff = 0;
    int64_t H = 0;
    const W* wbase = nullptr;
    const float* mbase = nullptr;
    for (; i < nhdr; i += P) {
      PROF_T(p_top);
      mbar_wait(&sm.recbar[g][rs], rph);
      const uint32_t* rec = sm.rec[g][rs];
      const int m = (int)(rec[0] & 0xff), nent = (int)(rec[0] >> 8), t = (int)rec[1];
      const int rw = 4 + 4 * ((m + 3) / 4);
      const uint32_t row = lane < m ? rec[4 + lane] : 0u;
      const int len = lane < m ? (int)reinterpret_cast<const uint8_t*>(rec + rw)[lane] : 0;
      const int ng = (nent + 3) >> 2;  // gather4 groups
      const uint32_t* bg = rec + rw + 4 * ((m + 15) / 16);
      uint4 b4 = lane < ng ? reinterpret_cast<const uint4*>(bg)[lane] : make_uint4(0, 0, 0, 0);
      uint32_t bagx[3] = {0, 0, 0};  // per-entry path: entries lane, lane + 32, lane + 64
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (lane + k * kWarp < nent) bagx[k] = bg[lane + k * kWarp];
      __syncwarp();  // the slot is read: refill it with batch i + 2P
      fetch_rec(rs == 0 ? 2 : rs - 1, hC, i + 2 * P < nhdr);
      hC = hdr_at(i + 3 * P);
      if (++rs == kRQ) {
        rs = 0;
        rph ^= 1;
      }
      if (t != tcur) {  // per-table constants (consecutive batches mostly share a table)
        tcur = t;
        doff = p.dim_offsets[t];
        D = p.dim_offsets[t + 1] - doff;
        H = p.row_offsets[t + 1] - p.row_offsets[t];
        wb = OPT == NEO_OPT_NONE ? 0 : D * (int)sizeof(W);
        gb = D * (int)sizeof(G);
        if (OPT != NEO_OPT_NONE) wbase = reinterpret_cast<const W*>(p.weights[t]);
        if (OPT == NEO_OPT_ROWWISE_ADAGRAD || OPT == NEO_OPT_ADAGRAD)
          mbase = reinterpret_cast<const float*>(p.moments[t]);
      }
      const int mrb = OPT == NEO_OPT_ADAGRAD ? D * 4 : 0;  // element-wise state bytes per row
      int eoff = len;
#pragma unroll
      for (int o = 1; o < kWarp; o <<= 1) {
        const int x = __shfl_up_sync(full, eoff, o);
        if (lane >= o) eoff += x;
      }
      eoff -= len;
      // runs of consecutive rows (one bulk copy each)
      const uint32_t prev = __shfl_up_sync(full, row, 1);
      const bool start = lane < m && (lane == 0 || row != prev + 1u);
      const unsigned starts = __ballot_sync(full, start);
      int runlen = 0;
      if (start) {
        const unsigned later = starts & ~((2u << lane) - 1u);
        runlen = (later ? __ffs(later) - 1 : m) - lane;
      }
      // row-wise moments: one 16-byte-aligned span when it is short and inside the table
      uint32_t mlo = ~0u;
      int mspan = 0;
      if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
        const uint32_t r0 = __shfl_sync(full, row, 0), r1 = __shfl_sync(full, row, m - 1);
        const uint32_t lo = r0 & ~3u, hi = (r1 | 3u) + 1u;
        if ((int64_t)hi <= H && (int)(hi - lo) * 4 <= kMomSpan) {
          mlo = lo;
          mspan = (int)(hi - lo) * 4;
        }
      }
      const bool tma = D == tma_dim && (gb & 31) == 0;  // gather4 groups land 128-byte aligned
      const uint32_t gbytes = (uint32_t)((tma ? ng * 4 : nent) * gb);
      const uint32_t bytes = (uint32_t)(m * (wb + mrb) + mspan) + gbytes;
      PROF_T(p_w0);
      mbar_wait(&sm.empty[g][s], ephase);
      PROF_T(p_w1);
      PROF_ADD(1, p_w1 - p_w0);
      PROF_ADD(2, p_w0 - p_top);
      StageMeta& mt = sm.meta[g][s];
      if (lane < m) {
        mt.row[lane] = row;
        mt.eoff[lane] = (uint16_t)eoff;
        mt.len[lane] = (uint8_t)len;
      }
      if (lane == 0) {
        mt.m = m;
        mt.nent = nent;
        mt.t = t;
        mt.mlo = mlo;
      }
      __syncwarp();
      unsigned char* st = sm.data[g][s];
      uint64_t* fb = &sm.full[g][s];
      if (lane == 0) mbar_arrive_tx(fb, bytes);  // the phase completes when every byte has landed
      __syncwarp();
      unsigned char* gst = st + ((m * (wb + mrb) + mspan + 127) & ~127);
      PROF_T(p_g0);
      if (tma) {
        if (lane < ng) gather4(gst + lane * 4 * gb, &gmap, doff, b4.x, b4.y, b4.z, b4.w, fb, pol_keep);
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int j = lane + k * kWarp;
          if (j < nent) bulk_g2s(gst + j * gb, gbase + (int64_t)bagx[k] * p.grad_stride + doff, gb, fb, pol_keep);
        }
      }
      PROF_T(p_g1);
      PROF_ADD(8, p_g1 - p_g0);
      if constexpr (OPT != NEO_OPT_NONE) {
        if (start) {
          bulk_g2s(st + lane * wb, wbase + (int64_t)row * D, runlen * wb, fb, pol_first);
          if (OPT == NEO_OPT_ADAGRAD)
            bulk_g2s(st + m * wb + lane * mrb, mbase + (int64_t)row * D, runlen * mrb, fb, pol_first);
        }
        if (OPT == NEO_OPT_ROWWISE_ADAGRAD && mspan && lane == 0)
          bulk_g2s(st + m * wb, mbase + mlo, mspan, fb, pol_first);
      }
      PROF_T(p_end);
      PROF_ADD(9, p_end - p_g1);
      PROF_ADD(3, p_end - p_w1);
      PROF_ADD(4, 1);
      if (++s == kRS) {
        s = 0;
        ephase ^= 1;
      }
    }
    // end of stream
    mbar_wait(&sm.empty[g][s], ephase);
    if (lane == 0) {
      sm.meta[g][s].m = -1;
      mbar_arrive(&sm.full[g][s]);
    }
    return;
  }

  // -------------------------------------------------------------- consumer
  // a sub-warp of S lanes per row; lane sl owns the row's 16-byte W vectors
  // v*S + sl (v < kLV: kEL elements per lane, interleaved so every shared-
  // memory access of a sub-warp is contiguous), R = 32/S rows per warp
  constexpr int kEL = 16;
  constexpr int kLV = kEL / kVW;
  const int c = role - 1;
  const uint64_t pol_stream = policy_evict_first();
  const float lr = (float)p.lr, eps = (float)p.eps;
  int s = 0;
  uint32_t fphase = 0;
  int t_cur = -1, D = 0, wb = 0, mb = 0, gb = 0, nv = 0, lgS = 0, S = 1, R = kWarp, sub = 0, sl = 0;
  unsigned submask = full;
  W* wt = nullptr;
  float* mom = nullptr;
  float invD = 1.f;
  for (;;) {
    PROF_T(c_w0);
    mbar_wait(&sm.full[g][s], fphase);
    PROF_T(c_w1);
    PROF_ADD(5, c_w1 - c_w0);
    const StageMeta& mt = sm.meta[g][s];
    const int m = mt.m;
    if (m < 0) break;
    const int t = mt.t;
    if (t != t_cur) {  // batches arrive table-major: per-table values change rarely
      t_cur = t;
      D = p.dim_offsets[t + 1] - p.dim_offsets[t];
      wb = OPT == NEO_OPT_NONE ? 0 : D * (int)sizeof(W);
      mb = OPT == NEO_OPT_ADAGRAD ? D * 4 : 0;  // element-wise state bytes per row
      gb = D * (int)sizeof(G);
      nv = D / kVW;  // 16-byte W vectors per row
      // S lanes per row (the smallest power of two with S * kLV >= nv), R rows per warp round
      const int need = (nv + kLV - 1) / kLV;
      lgS = need <= 1 ? 0 : 32 - __clz(need - 1);
      S = 1 << lgS;
      R = kWarp >> lgS;
      sub = lane >> lgS;
      sl = lane & (S - 1);
      submask = S == kWarp ? full : (((1u << S) - 1u) << (sub * S));
      wt = reinterpret_cast<W*>(OPT == NEO_OPT_NONE ? p.dense_grads[t] : p.weights[t]);
      mom = (OPT == NEO_OPT_ROWWISE_ADAGRAD || OPT == NEO_OPT_ADAGRAD) ? reinterpret_cast<float*>(p.moments[t])
                                                                       : nullptr;
      invD = 1.0f / (float)D;
    }
    const uint32_t mlo = mt.mlo;
    const int mspan = (OPT == NEO_OPT_ROWWISE_ADAGRAD && mlo != ~0u)
                          ? (int)(((mt.row[m - 1] | 3u) + 1u - mlo) * 4)
                          : 0;
    const unsigned char* st = sm.data[g][s];
    const unsigned char* gst = st + ((m * (wb + mb) + mspan + 127) & ~127);
    const int rounds = (int)((unsigned)((m + kRC * R - 1) >> (5 - lgS)) / (unsigned)kRC);
    for (int rd = 0; rd < rounds; ++rd) {
      const int rr = (rd * kRC + c) * R + sub;
      const bool valid = rr < m;
      const int len = valid ? mt.len[rr] : 0;
      const int eo = valid ? mt.eoff[rr] : 0;
      const uint32_t row = valid ? mt.row[rr] : 0u;
      const int maxlen = (int)__reduce_max_sync(full, (unsigned)len);
      float acc[kLV][kVW];
#pragma unroll
      for (int v = 0; v < kLV; ++v)
#pragma unroll
        for (int e = 0; e < kVW; ++e) acc[v][e] = 0.f;
      const G* gr = reinterpret_cast<const G*>(gst + eo * gb);
      for (int j = 0; j < maxlen; ++j) {  // the row's upstream rows, in order
        if (j < len) {
#pragma unroll
          for (int v = 0; v < kLV; ++v) {
            const int vi = v * S + sl;
            if (vi < nv) {
              Vec<G, kVW> x;
              if constexpr (sizeof(G) * kVW == 32) {
                reinterpret_cast<uint4*>(&x)[0] = reinterpret_cast<const uint4*>(gr + vi * kVW)[0];
                reinterpret_cast<uint4*>(&x)[1] = reinterpret_cast<const uint4*>(gr + vi * kVW)[1];
              } else {
                x = *reinterpret_cast<const Vec<G, kVW>*>(gr + vi * kVW);
              }
#pragma unroll
              for (int e = 0; e < kVW; ++e) acc[v][e] += Elem<G>::to_f(x.v[e]);
            }
          }
        }
        gr += D;
      }
      if (OPT == NEO_OPT_NONE) {
        if (valid) {
#pragma unroll
          for (int v = 0; v < kLV; ++v) {
            const int vi = v * S + sl;
            if (vi < nv) {
              float* dst = reinterpret_cast<float*>(wt) + (int64_t)row * D + vi * kVW;
#pragma unroll
              for (int e = 0; e < kVW; e += 4)
                *reinterpret_cast<float4*>(dst + e) =
                    make_float4(acc[v][e], acc[v][e + 1], acc[v][e + 2], acc[v][e + 3]);
            }
          }
        }
        continue;
      }
      float ss = 0.f;
      if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
#pragma unroll
        for (int v = 0; v < kLV; ++v)
#pragma unroll
          for (int e = 0; e < kVW; ++e) ss += acc[v][e] * acc[v][e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
          if (o < S) ss += __shfl_xor_sync(full, ss, o);
      }
      bool live = valid;
      if (OPT == NEO_OPT_ADAGRAD || OPT == NEO_OPT_ROWWISE_ADAGRAD) {
        // an identically zero gradient leaves the row untouched (embedding.py:223-228);
        // for row-wise AdaGrad a nonzero sum of squares already decides it
        bool nz = OPT == NEO_OPT_ROWWISE_ADAGRAD && ss != 0.f;
        if (!nz) {
#pragma unroll
          for (int v = 0; v < kLV; ++v)
#pragma unroll
            for (int e = 0; e < kVW; ++e) nz |= acc[v][e] != 0.f;
        }
        const unsigned vote = __ballot_sync(full, nz);
        live = live && (vote & submask) != 0u;
      }
      if (!live) continue;
      float scale = lr;
      if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
        const float mr = mlo != ~0u ? reinterpret_cast<const float*>(st + m * wb)[row - mlo] : mom[row];
        const float mn = mr + ss * invD;
        if (sl == 0) mom[row] = mn;
        scale = __fdividef(lr, __fsqrt_rn(mn) + eps);
      }
#pragma unroll
      for (int v = 0; v < kLV; ++v) {
        const int vi = v * S + sl;
        if (vi < nv) {
          const Vec<W, kVW> w = *reinterpret_cast<const Vec<W, kVW>*>(st + rr * wb + vi * 16);
          Vec<W, kVW> o;
          if (OPT == NEO_OPT_ADAGRAD) {
            const float* mv = reinterpret_cast<const float*>(st + m * wb + rr * mb) + vi * kVW;
            float mo[kVW];
#pragma unroll
            for (int e = 0; e < kVW; ++e) {
              mo[e] = mv[e] + acc[v][e] * acc[v][e];
              o.v[e] = Elem<W>::from_f(Elem<W>::to_f(w.v[e]) -
                                       __fdividef(lr * acc[v][e], __fsqrt_rn(mo[e]) + eps));
            }
            float* md = mom + (int64_t)row * D + vi * kVW;
#pragma unroll
            for (int e = 0; e < kVW; e += 4)
              *reinterpret_cast<float4*>(md + e) = make_float4(mo[e], mo[e + 1], mo[e + 2], mo[e + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < kVW; ++e) o.v[e] = Elem<W>::from_f(Elem<W>::to_f(w.v[e]) - acc[v][e] * scale);
          }
          st16_hint(wt + (int64_t)row * D + vi * kVW, *reinterpret_cast<const uint4*>(&o), pol_stream);
        }
      }
    }
    __syncwarp();
    PROF_T(c_end);
    PROF_ADD(6, c_end - c_w1);
    PROF_ADD(7, 1);
    if (lane == 0) mbar_arrive(&sm.empty[g][s]);
    if (++s == kRS) {
      s = 0;
      fphase ^= 1;
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

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename G>
static bool encode_gather_map(const SegParams& p, CUtensorMap* map) {
  static EncodeTiledFn enc = [] {
    EncodeTiledFn f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return f;
  }();
  const char* off = std::getenv("NEO_BKT_NO_TMA");
  if (!enc || (off && *off == '1') || p.max_dim < 8 || p.max_dim > 256 || (reinterpret_cast<uintptr_t>(p.grad) & 15) ||
      ((p.grad_stride * sizeof(G)) & 15) || p.B > (int64_t(1) << 31))
    return false;
  const CUtensorMapDataType dt = sizeof(G) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : std::is_same<G, __half>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                  : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  cuuint64_t dims[2] = {(cuuint64_t)p.grad_stride, (cuuint64_t)p.B};
  cuuint64_t strides[1] = {(cuuint64_t)p.grad_stride * sizeof(G)};
  cuuint32_t box[2] = {(cuuint32_t)p.max_dim, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(map, dt, 2, const_cast<void*>(p.grad), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <typename W, typename G, int OPT, int BINS>
static int launch_wsort(const Params& q, const SegParams& p, int sms, cudaStream_t s) {
  auto wkern = bkt_wsort_kernel<W, G, OPT, BINS>;
  const int wsmem = (int)(sizeof(WSmem<BINS>) * kWW);
  if (cudaFuncSetAttribute(wkern, cudaFuncAttributeMaxDynamicSharedMemorySize, wsmem) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve warp-sort shared memory");
  int wper = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, wkern, kWW * kWarp, wsmem);
  if (wper < 1) wper = 1;
  wkern<<<(unsigned)(sms * wper), kWW * kWarp, wsmem, s>>>(q, p);
  return dbg(s, BINS == kBins ? "neo_tbe_backward(bucket warp sort)" : "neo_tbe_backward(bucket warp sort, 10-bit)");
}

template <typename W, typename G, int OPT>
static int launch_update(const Params& q, const SegParams& p, int sms, cudaStream_t s, bool prepare, bool apply) {
  if (prepare) {
    auto kern = bkt_sort_kernel<W, G, OPT>;
    const int smem = (int)sizeof(USmem);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve bucket shared memory");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kUT, smem);
    if (per_sm < 1) per_sm = 1;
    kern<<<(unsigned)(sms * per_sm), kUT, smem, s>>>(q, p);
    int rc = dbg(s, "neo_tbe_backward(bucket sort)");
    if (rc) return rc;
    rc = launch_wsort<W, G, OPT, kBins>(q, p, sms, s);
    if (rc) return rc;
    rc = launch_wsort<W, G, OPT, 2 * kBins>(q, p, sms, s);
    if (rc) return rc;
  }
  if (apply) {
    bkt_long_kernel<W, G, OPT><<<(unsigned)(sms * 4), kLW * kWarp, 0, s>>>(q, p);
    const int rc = dbg(s, "neo_tbe_backward(bucket hot rows)");
    if (rc) return rc;
    auto kern = bkt_rows_kernel<W, G, OPT>;
    const int smem = (int)sizeof(RowSmem);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve row-kernel shared memory");
    // tile::gather4 tensor map over the upstream (B rows x grad_stride), box =
    // one row of max_dim columns: tables of that width stage their upstream
    // rows four per TMA op; other widths use 16-byte cp.async pieces
    CUtensorMap gmap;
    std::memset(&gmap, 0, sizeof(gmap));
    const int32_t tma_dim = encode_gather_map<G>(p, &gmap) ? p.max_dim : 0;
    kern<<<(unsigned)sms, kRT, smem, s>>>(q, p, gmap, tma_dim);
    return dbg(s, "neo_tbe_backward(bucket rows)");
  }
  return NEO_OK;
}

template <typename W, typename G>
static int launch_update_opt(const Params& q, const SegParams& p, int sms, cudaStream_t s, bool prepare,
                             bool apply) {
  if (p.mode == NEO_BWD_DENSE) {
    if constexpr (std::is_same<W, float>::value)
      return launch_update<W, G, NEO_OPT_NONE>(q, p, sms, s, prepare, apply);
    return fail(NEO_E_ARG, "neo_tbe_backward: DENSE needs f32");
  }
  switch (p.optim) {
    case NEO_OPT_SGD: return launch_update<W, G, NEO_OPT_SGD>(q, p, sms, s, prepare, apply);
    case NEO_OPT_ROWWISE_ADAGRAD: return launch_update<W, G, NEO_OPT_ROWWISE_ADAGRAD>(q, p, sms, s, prepare, apply);
    default: return launch_update<W, G, NEO_OPT_ADAGRAD>(q, p, sms, s, prepare, apply);
  }
}

static int target_entries() {
  const char* v = std::getenv("NEO_BKT_TARGET");
  const int t = v ? std::atoi(v) : 0;
  return t > 0 ? t : kTarget;
}

}  // namespace bkt

// capacity bounds of the batch stream (worst case over element types: f32
// weights with element-wise state, f32 upstream).  In a 32-row chunk two
// consecutive batches together overflow the stage budget or kMaxEnt (or the
// first one ends at a long row), so batches <= 2 cost/budget + 2 N/kMaxEnt
// + chunks + long rows; every batch has >= 1 row and every row >= 1 entry.
static void stream_caps(int64_t N, int64_t nb, int32_t max_dim, int64_t* hdr_cap, int64_t* rec_cap) {
  using namespace bkt;
  const int64_t D = max_dim > 8 ? max_dim : 8;
  const int64_t rowb = 8 * D, gb = 4 * D;
  const int64_t budget = kStageBytes - 128 - kMomSpan - 3 * gb;
  const int64_t lth = budget / gb - 3 > 1 ? budget / gb - 3 : 1;
  const int64_t n = N > 0 ? N : 1;
  const int64_t chunks = n / kWarp + nb + n / kCap + 1;
  int64_t nbat = 2 * (n * (rowb + gb) / budget + 1) + 2 * (n / kMaxEnt + 1) + chunks + n / (lth + 1) + 64;
  if (nbat > n + 64) nbat = n + 64;
  *hdr_cap = nbat;
  *rec_cap = 3 * nbat + n / 4 + n / 16 + n / 4 + 64;
}

size_t bkt_workspace(int32_t T, int64_t B, int64_t N, int64_t total_rows, int32_t max_dim) {
  using namespace bkt;
  const int64_t cpt = (B + kCHB - 1) / kCHB;
  const int64_t nb = bucket_bound(T, total_rows);
  const int64_t M = nb * cpt;
  const int64_t n1 = N > 0 ? N : 1;
  int64_t hdr_cap, rec_cap;
  stream_caps(N, nb, max_dim, &hdr_cap, &rec_cap);
  size_t b = 0;
  b += align256(sizeof(int32_t) * T);                    // sbits
  b += align256(sizeof(int64_t) * (T + 1));              // bbase
  b += align256(sizeof(int32_t) * (M + 1));              // count matrix
  b += align256(sizeof(int32_t) * (M / kScanTile + 2));  // scan tiles
  b += align256(sizeof(int32_t) * (nb + 1));             // bucket starts
  b += align256(sizeof(int32_t) * (nb + 1));             // bucket tables
  b += align256(sizeof(uint8_t) * (nb + 1));             // bucket kinds
  b += align256(sizeof(int32_t) * (nb + 1));             // kind-2 list
  b += align256(sizeof(int32_t) * (nb + 1));             // big-bucket queue
  b += align256(sizeof(int32_t) * 16);                   // counters
  b += 2 * align256(sizeof(uint32_t) * n1);              // entries + big-bucket scratch
  b += align256(sizeof(uint2) * hdr_cap);                // batch headers
  b += align256((size_t)16 * rec_cap);                   // batch records
  b += align256(sizeof(uint4) * (n1 / 16 + 64));         // hot rows (> 16 occurrences each)
  return b;
}

// can the bucketed path take this call? (host side; layout promises from the caller)
bool bkt_eligible(const SegParams& p, int32_t weight_dtype, int32_t grad_dtype, bool out_count) {
  using namespace bkt;
  const char* v = std::getenv("NEO_BWD_VARIANT");
  if (v && (std::strcmp(v, "pipe") == 0 || std::strcmp(v, "stream") == 0)) return false;
  if (!(p.flags & NEO_BWD_FLAG_DIM8) || out_count) return false;
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
  return s + bag_bits_for(p.B) <= 32 && p.N < (int64_t(1) << 31);
}

int run_bucket_backward(SegParams p, int32_t weight_dtype, int32_t grad_dtype, const void* indices,
                        int32_t index_dtype, void* workspace, size_t ws_bytes, neo_error* err, cudaStream_t s) {
  using namespace bkt;
  const int64_t N = p.N;
  if (ws_bytes < bkt_workspace(p.T, p.B, N, p.total_rows, p.max_dim))
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
  const int64_t n1 = N > 0 ? N : 1;
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
  q.btab = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (nb + 1));
  q.bkind = reinterpret_cast<uint8_t*>(w);
  w += align256(sizeof(uint8_t) * (nb + 1));
  q.ctal = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (nb + 1));
  q.big = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * (nb + 1));
  q.ctr = reinterpret_cast<int32_t*>(w);
  w += align256(sizeof(int32_t) * 16);
  q.ent = reinterpret_cast<uint32_t*>(w);
  w += align256(sizeof(uint32_t) * n1);
  q.ent2 = reinterpret_cast<uint32_t*>(w);
  w += align256(sizeof(uint32_t) * n1);
  stream_caps(N, nb, p.max_dim, &q.hdr_cap, &q.rec_cap);
  q.hdr = reinterpret_cast<uint2*>(w);
  w += align256(sizeof(uint2) * q.hdr_cap);
  q.rec = reinterpret_cast<uint32_t*>(w);
  w += align256((size_t)16 * q.rec_cap);
  q.longs = reinterpret_cast<uint4*>(w);
  q.long_cap = n1 / 16 + 64;

  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // PREPARE = the sort phase (counting sort + batches; hot rows are updated
  // here), APPLY = the row kernel; the state between them is the workspace
  const bool prepare = !(p.flags & NEO_BWD_FLAG_APPLY);
  const bool apply = !(p.flags & NEO_BWD_FLAG_PREPARE);
  int rc = NEO_OK;
  if (prepare) {
    bkt_setup_kernel<<<1, 1024, 0, s>>>(q);
    if ((rc = dbg(s, "neo_tbe_backward(bucket setup)"))) return rc;
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
    const int smem = (int)((kScW + 1) * kMaxB * sizeof(uint32_t));
    auto k32 = bkt_scatter_kernel<int32_t>;
    auto k64 = bkt_scatter_kernel<int64_t>;
    if (cudaFuncSetAttribute(k32, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(k64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return fail(NEO_E_CUDA, "neo_tbe_backward: cannot reserve scatter shared memory");
    if (index_dtype == NEO_I32) k32<<<chunks, kScW * kWarp, smem, s>>>(q, (const int32_t*)indices);
    else k64<<<chunks, kScW * kWarp, smem, s>>>(q, (const int64_t*)indices);
    if ((rc = dbg(s, "neo_tbe_backward(bucket scatter)"))) return rc;
    launch_error_finalize(err, indices, index_dtype, p.offsets, p.B, p.T, s);
    if ((rc = check_launch("neo_tbe_backward(finalize)"))) return rc;
  }
  const bool h = weight_dtype == NEO_F16;
  switch (grad_dtype) {
    case NEO_F32:
      rc = h ? launch_update_opt<__half, float>(q, p, sms, s, prepare, apply)
             : launch_update_opt<float, float>(q, p, sms, s, prepare, apply);
      break;
    case NEO_BF16:
      rc = h ? launch_update_opt<__half, __nv_bfloat16>(q, p, sms, s, prepare, apply)
             : launch_update_opt<float, __nv_bfloat16>(q, p, sms, s, prepare, apply);
      break;
    default:
      rc = h ? launch_update_opt<__half, __half>(q, p, sms, s, prepare, apply)
             : launch_update_opt<float, __half>(q, p, sms, s, prepare, apply);
      break;
  }
  return rc;
}

}  // namespace neo

#ifdef NEO_BKT_PROF
extern "C" int neo_bkt_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, neo::bkt::g_bkt_prof, sizeof(unsigned long long) * 12);
  if (reset) {
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbol(neo::bkt::g_bkt_prof, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" size_t neo_tbe_bucket_workspace_bytes(int32_t num_tables, int64_t batch, int64_t num_indices,
                                                 int64_t total_rows, int32_t max_dim) {
  if (num_tables < 0 || batch < 0 || num_indices < 0 || total_rows < 0 || max_dim < 0) return 0;
  return neo::bkt_workspace(num_tables, batch, num_indices, total_rows, max_dim);
}
