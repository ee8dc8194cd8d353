// Set-associative software row cache (cache.py:68-133) on the GPU.
//
// Reference semantics (cache.py:68-98 access, 117-126 simulate_trace): row r
// maps to set r % num_sets; the clock advances once per access; a hit
// refreshes the line's last_used and bumps its frequency; a miss into a full
// set evicts argmin (last_used, i) [LRU] or (frequency, last_used, i) [LFU]
// and inserts the row.  last_used values are distinct (one clock tick per
// access), so the line-index tie-break never decides and the line order of
// a set does not matter.
//
// Sets are independent, and within a set only the ORDER of its accesses
// matters.  So: (1) a stable radix sort of (set, position) pairs groups each
// set's accesses in trace order; (2) one warp per set replays them, lane w
// holding way w (row, last_used = position + 1, frequency) in registers; a
// hit is one ballot, the victim one or two __reduce_min_sync; a run of
// accesses repeating the previous access's row (hot rows) is applied in one
// step.  Per-access
// results (hit, evicted row) land at the access's trace position, so the
// output equals the reference's sequential AccessResult stream.
#include <climits>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "common.cuh"

namespace neo {

static inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

__global__ void cache_keys_kernel(const int64_t* __restrict__ trace, int64_t n, int64_t num_sets,
                                  uint32_t* __restrict__ keys, int32_t* __restrict__ pos, neo_error* err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = trace[i];
    if (r < 0) record_bad_index(err, i);
    keys[i] = (uint32_t)(r < 0 ? 0 : r % num_sets);
    pos[i] = (int32_t)i;
  }
}

struct CacheHead {
  const uint32_t* keys;
  __device__ __forceinline__ bool operator()(const int32_t& i) const { return i == 0 || keys[i] != keys[i - 1]; }
};

// K ways per lane: way k*32 + lane lives in lane `lane`, slot k (ways <= 32K)
template <int K>
__global__ void __launch_bounds__(256)
cache_replay_kernel(const int64_t* __restrict__ trace, const int32_t* __restrict__ pos,
                    const int32_t* __restrict__ starts, const int64_t* __restrict__ num_segs, int64_t n,
                    int32_t ways, int32_t lfu, uint8_t* __restrict__ hit_out, int64_t* __restrict__ ev_out,
                    unsigned long long* __restrict__ stats) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x % kWarp;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / kWarp;
  const int64_t S = *num_segs;
  unsigned waymask[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int w = ways - k * kWarp;
    waymask[k] = w >= 32 ? full : (w <= 0 ? 0u : ((1u << w) - 1u));
  }
  unsigned long long h = 0, m = 0, e = 0;
  for (int64_t seg = warp; seg < S; seg += nwarps) {
    const int64_t s0 = starts[seg];
    const int64_t s1 = seg + 1 < S ? (int64_t)starts[seg + 1] : n;
    int64_t row[K];            // this lane's ways
    uint32_t last[K], freq[K];
    bool valid[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      row[k] = -1;
      last[k] = freq[k] = 0;
      valid[k] = false;
    }
    int cnt = 0;
    int64_t prev_r = -1;  // row of the set's previous access (resident after it)
    // the (slot, lane) holding row r, as slot * 32 + lane, or -1
    auto find = [&](int64_t r) -> int {
      int where = -1;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const unsigned hm = __ballot_sync(full, valid[k] && row[k] == r);
        if (where < 0 && hm) where = k * kWarp + __ffs(hm) - 1;
      }
      return where;
    };
    for (int64_t j0 = s0; j0 < s1; j0 += kWarp) {
      const int mm = (int)min64(kWarp, s1 - j0);
      const int32_t my_p = lane < mm ? pos[j0 + lane] : 0;
      const int64_t my_r = lane < mm ? trace[my_p] : -2;
      // runs of one row: an access repeating the previous access's row is a
      // hit on the way that row occupies (hot rows of skewed traces), so a
      // run of L such accesses is applied at once: frequency += L,
      // last_used = the run's last clock
      int64_t up = __shfl_up_sync(full, my_r, 1);
      if (lane == 0) up = prev_r;
      const unsigned same = __ballot_sync(full, lane < mm && my_r == up);
      prev_r = __shfl_sync(full, my_r, mm - 1);
      for (int k = 0; k < mm;) {
        if ((same >> k) & 1u) {
          const unsigned rest = ~(same >> k);  // first access after the run
          const int L = min(rest ? __ffs(rest) - 1 : kWarp - k, mm - k);
          const int64_t r = __shfl_sync(full, my_r, k);
          const uint32_t clock_end = (uint32_t)__shfl_sync(full, my_p, k + L - 1) + 1u;
          const int wh = find(r);
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (wh == q * kWarp + lane) {
              last[q] = clock_end;
              freq[q] += (uint32_t)L;
            }
          if (lane >= k && lane < k + L) {
            if (hit_out) hit_out[my_p] = 1;
            if (ev_out) ev_out[my_p] = -1;
          }
          h += (unsigned long long)L;
          k += L;
          continue;
        }
        const int32_t p = __shfl_sync(full, my_p, k);
        const int64_t r = __shfl_sync(full, my_r, k);
        const uint32_t clock = (uint32_t)p + 1u;
        ++k;
        const int wh = find(r);
        if (wh >= 0) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (wh == q * kWarp + lane) {
              last[q] = clock;
              freq[q] += 1;
            }
          ++h;
          if (lane == 0) {
            if (hit_out) hit_out[p] = 1;
            if (ev_out) ev_out[p] = -1;
          }
          continue;
        }
        ++m;
        int64_t ev = -1;
        int tgt = -1;
        if (cnt < ways) {  // a free way (which one does not change any result)
#pragma unroll
          for (int q = 0; q < K; ++q) {
            const unsigned fm = ~__ballot_sync(full, valid[q]) & waymask[q];
            if (tgt < 0 && fm) tgt = q * kWarp + __ffs(fm) - 1;
          }
          ++cnt;
        } else {  // LRU: least recently used; LFU: least frequently used, then least recently
          uint32_t fmin = UINT_MAX;
          if (lfu) {
            uint32_t f = UINT_MAX;
#pragma unroll
            for (int q = 0; q < K; ++q) f = min(f, valid[q] ? freq[q] : UINT_MAX);
            fmin = __reduce_min_sync(full, f);
          }
          uint32_t key[K], kmin = UINT_MAX;
#pragma unroll
          for (int q = 0; q < K; ++q) {
            key[q] = (valid[q] && (!lfu || freq[q] == fmin)) ? last[q] : UINT_MAX;
            kmin = min(kmin, key[q]);
          }
          const uint32_t lmin = __reduce_min_sync(full, kmin);
#pragma unroll
          for (int q = 0; q < K; ++q) {
            const unsigned bm = __ballot_sync(full, valid[q] && key[q] == lmin);
            if (tgt < 0 && bm) tgt = q * kWarp + __ffs(bm) - 1;
          }
          int64_t evr = -1;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (tgt / kWarp == q) evr = row[q];
          ev = __shfl_sync(full, evr, tgt % kWarp);
          ++e;
        }
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (tgt == q * kWarp + lane) {
            row[q] = r;
            last[q] = clock;
            freq[q] = 1;
            valid[q] = true;
          }
        if (lane == 0) {
          if (hit_out) hit_out[p] = 0;
          if (ev_out) ev_out[p] = ev;
        }
      }
    }
  }
  if (lane == 0 && (h | m | e)) {
    atomicAdd(stats + 0, h);
    atomicAdd(stats + 1, m);
    atomicAdd(stats + 2, e);
  }
}

static size_t cub_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int)n, 0, 32);
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::If(nullptr, b, it, (int32_t*)nullptr, (int64_t*)nullptr, (int)n, CacheHead{nullptr});
  return a > b ? a : b;
}

static size_t cache_ws(int64_t n) {
  return 2 * a256(4 * (size_t)n) + 2 * a256(4 * (size_t)n) + a256(4 * (size_t)n) + a256(8) + a256(cub_bytes(n));
}

}  // namespace neo

extern "C" size_t neo_cache_workspace_bytes(int64_t num_accesses) {
  return neo::cache_ws(num_accesses < 1 ? 1 : num_accesses);
}

extern "C" int neo_cache_simulate(int64_t num_sets, int32_t ways, int32_t policy, const int64_t* trace,
                                  int64_t num_accesses, uint8_t* hit, int64_t* evicted, int64_t* stats,
                                  void* workspace, size_t workspace_bytes, neo_error* err, void* stream) {
  using namespace neo;
  cudaStream_t s = as_stream(stream);
  if (num_sets < 1) return fail(NEO_E_ARG, "num_sets: must be >= 1");
  if (ways < 1) return fail(NEO_E_ARG, "ways: must be >= 1");
  if (ways > 4 * kWarp) return fail(NEO_E_ARG, "ways: this implementation holds up to 4 ways per lane (<= 128)");
  if (num_sets > (int64_t)UINT32_MAX) return fail(NEO_E_ARG, "num_sets: must be < 2^32");
  if (policy != NEO_CACHE_LRU && policy != NEO_CACHE_LFU) return fail(NEO_E_ARG, "policy: LRU or LFU");
  if (num_accesses < 0 || num_accesses >= INT_MAX) return fail(NEO_E_ARG, "trace: 0 .. 2^31-1 accesses");
  if (!stats) return fail(NEO_E_ARG, "stats: [3] device int64 required");
  if (cudaMemsetAsync(stats, 0, 3 * sizeof(int64_t), s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_cache_simulate: memset failed");
  const int64_t n = num_accesses;
  if (n == 0) return NEO_OK;
  if (workspace_bytes < cache_ws(n)) return fail(NEO_E_ARG, "neo_cache_simulate: workspace too small");
  unsigned char* w = static_cast<unsigned char*>(workspace);
  uint32_t* k0 = reinterpret_cast<uint32_t*>(w); w += a256(4 * (size_t)n);
  uint32_t* k1 = reinterpret_cast<uint32_t*>(w); w += a256(4 * (size_t)n);
  int32_t* v0 = reinterpret_cast<int32_t*>(w); w += a256(4 * (size_t)n);
  int32_t* v1 = reinterpret_cast<int32_t*>(w); w += a256(4 * (size_t)n);
  int32_t* starts = reinterpret_cast<int32_t*>(w); w += a256(4 * (size_t)n);
  int64_t* nseg = reinterpret_cast<int64_t*>(w); w += a256(8);
  size_t tb = cub_bytes(n);
  const unsigned kb_grid = (unsigned)min64((n + 255) / 256, 148 * 32);
  cache_keys_kernel<<<kb_grid, 256, 0, s>>>(trace, n, num_sets, k0, v0, err);
  int rc = check_launch("neo_cache_simulate(keys)");
  if (rc) return rc;
  int bits = 1;
  while (bits < 32 && (uint64_t(1) << bits) < (uint64_t)num_sets) ++bits;
  cub::DoubleBuffer<uint32_t> kbuf(k0, k1);
  cub::DoubleBuffer<int32_t> vbuf(v0, v1);
  if (cub::DeviceRadixSort::SortPairs(w, tb, kbuf, vbuf, (int)n, 0, bits, s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_cache_simulate: radix sort failed");
  tb = cub_bytes(n);
  cub::CountingInputIterator<int32_t> it(0);
  if (cub::DeviceSelect::If(w, tb, it, starts, nseg, (int)n, CacheHead{kbuf.Current()}, s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_cache_simulate: segment select failed");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (min64(n, (int64_t)num_sets) + 7) / 8;
  const unsigned grid = (unsigned)(want < (int64_t)sms * 8 ? (want > 0 ? want : 1) : (int64_t)sms * 8);
  const int lfu = policy == NEO_CACHE_LFU ? 1 : 0;
  unsigned long long* st = reinterpret_cast<unsigned long long*>(stats);
  if (ways <= kWarp)
    cache_replay_kernel<1><<<grid, 256, 0, s>>>(trace, vbuf.Current(), starts, nseg, n, ways, lfu, hit, evicted, st);
  else if (ways <= 2 * kWarp)
    cache_replay_kernel<2><<<grid, 256, 0, s>>>(trace, vbuf.Current(), starts, nseg, n, ways, lfu, hit, evicted, st);
  else
    cache_replay_kernel<4><<<grid, 256, 0, s>>>(trace, vbuf.Current(), starts, nseg, n, ways, lfu, hit, evicted, st);
  rc = check_launch("neo_cache_simulate(replay)");
  if (rc) return rc;
  return NEO_OK;
}

// ===========================================================================
// HBM tier over host-resident tables: the embedding rows
// live in pinned host memory (device-addressable through UVA); an HBM cache
// of num_sets x ways slots per table holds the rows a batch touches, and the
// TBE kernels run on the slots.  Per batch:
//   1. stable radix sort of (set = id % num_sets, position);
//   2. one warp per set (lane = way): pass 1 stamps every way whose row the
//      batch uses; pass 2 maps each access to its slot, filling misses into
//      ways NOT used by this batch (least recently stamped, lowest way on
//      ties) and queueing (slot, evicted row, fetched row) transfers.  Rows
//      a batch uses are never evicted by it, so no row is both written back
//      and fetched in one batch;
//   3. one warp per transfer writes the evicted slot (row + optimizer state)
//      back to host memory, then fetches the new row into the slot.
// A set that needs more than `ways` distinct rows in one batch cannot be
// served: its extra accesses map to slot -1 and counters[2] counts them.
// Training through the tier is bitwise identical to training with the whole
// table in HBM: the same rows, in the same per-row order, feed the same
// kernels.

namespace neo {

template <typename Idx>
__global__ void tier_keys_kernel(const Idx* __restrict__ ids, int64_t n, int64_t H, int64_t num_sets,
                                 uint32_t* __restrict__ keys, int32_t* __restrict__ pos, neo_error* err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)ids[i];
    const bool ok = r >= 0 && r < H;
    if (!ok) record_bad_index(err, i);
    keys[i] = (uint32_t)(ok ? r % num_sets : 0);
    pos[i] = (int32_t)i;
  }
}

template <typename Idx>
__global__ void __launch_bounds__(256)
tier_assign_kernel(const Idx* __restrict__ ids, const int32_t* __restrict__ pos, const int32_t* __restrict__ starts,
                   const int64_t* __restrict__ num_segs, int64_t n, int64_t H, int64_t num_sets, int32_t ways,
                   int64_t* __restrict__ tags, uint32_t* __restrict__ stamps, uint32_t stamp,
                   int32_t* __restrict__ slots_out, int64_t* __restrict__ xfer,
                   unsigned long long* __restrict__ counters, int64_t spill_cap, int64_t* __restrict__ spill_list) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x % kWarp;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / kWarp;
  const int64_t S = *num_segs;
  unsigned long long misses = 0, wbs = 0, over = 0;
  for (int64_t seg = warp; seg < S; seg += nwarps) {
    const int64_t s0 = starts[seg];
    const int64_t s1 = seg + 1 < S ? (int64_t)starts[seg + 1] : n;
    const int64_t r0 = (int64_t)ids[pos[s0]];
    // out-of-range ids were keyed to set 0 (and are skipped per access below)
    const int64_t set_id = (r0 >= 0 && r0 < H) ? r0 % num_sets : 0;
    const int64_t base = set_id * ways;
    int64_t tag = lane < ways ? tags[base + lane] : -2;
    uint32_t st = lane < ways ? stamps[base + lane] : 0xffffffffu;
    // rows of this set that found no free way this batch: one spill slot each
    // (lane k holds the k-th), fetched now, written back after the backward
    int64_t sp_tag = -1;
    int32_t sp_slot = -1;
    int sp_n = 0;
    // pass 1: stamp the ways this batch uses (lane-parallel: the 32 accesses
    // of a window against each way's tag)
    for (int64_t j0 = s0; j0 < s1; j0 += kWarp) {
      const int mm = (int)min64(kWarp, s1 - j0);
      const int64_t my_r = lane < mm ? (int64_t)ids[pos[j0 + lane]] : -1;
      for (int w = 0; w < ways; ++w) {
        const int64_t tw = __shfl_sync(full, tag, w);
        if (__any_sync(full, tw >= 0 && my_r == tw) && lane == w) st = stamp;
      }
    }
    // pass 2: map every access to its slot, filling misses.  A run of accesses
    // repeating the previous access's row (hot rows) shares its slot.
    int64_t prev_r = -1;
    int32_t prev_slot = -1;
    for (int64_t j0 = s0; j0 < s1; j0 += kWarp) {
      const int mm = (int)min64(kWarp, s1 - j0);
      const int32_t my_p = lane < mm ? pos[j0 + lane] : 0;
      const int64_t my_r = lane < mm ? (int64_t)ids[my_p] : -1;
      int64_t up = __shfl_up_sync(full, my_r, 1);
      if (lane == 0) up = prev_r;
      const unsigned same = __ballot_sync(full, lane < mm && my_r >= 0 && my_r < H && my_r == up);
      for (int k = 0; k < mm;) {
        if ((same >> k) & 1u) {
          const unsigned rest = ~(same >> k);
          const int L = min(rest ? __ffs(rest) - 1 : kWarp - k, mm - k);
          if (lane >= k && lane < k + L) slots_out[my_p] = prev_slot;
          k += L;
          continue;
        }
        const int64_t r = __shfl_sync(full, my_r, k);
        const int32_t p = __shfl_sync(full, my_p, k);
        ++k;
        prev_r = r;
        prev_slot = -1;
        if (r < 0 || r >= H) {  // reported through err by the key kernel
          if (lane == 0) slots_out[p] = -1;
          continue;
        }
        const unsigned hm = __ballot_sync(full, tag == r);
        if (hm) {
          prev_slot = (int32_t)(base + __ffs(hm) - 1);
          if (lane == 0) slots_out[p] = prev_slot;
          continue;
        }
        const bool cand = lane < ways && st != stamp;
        const unsigned cm = __ballot_sync(full, cand);
        if (!cm) {  // set overflow: a spill slot for the batch
          const unsigned sm = __ballot_sync(full, sp_tag == r);
          if (sm) {
            prev_slot = __shfl_sync(full, sp_slot, __ffs(sm) - 1);
            if (lane == 0) slots_out[p] = prev_slot;
            continue;
          }
          long long idx = -1;
          if (lane == 0 && sp_n < kWarp && spill_cap > 0) {
            idx = (long long)atomicAdd(counters + 4, 1ull);
            if (idx >= spill_cap) idx = -1;
          }
          idx = __shfl_sync(full, idx, 0);
          if (idx < 0) {
            ++over;
            if (lane == 0) slots_out[p] = -1;
            continue;
          }
          const int32_t slot = (int32_t)(num_sets * ways + idx);
          if (lane == sp_n) {
            sp_tag = r;
            sp_slot = slot;
          }
          ++sp_n;
          ++misses;
          prev_slot = slot;
          if (lane == 0) {
            spill_list[2 * idx] = slot;
            spill_list[2 * idx + 1] = r;
            const unsigned long long x = atomicAdd(counters + 3, 1ull);
            xfer[3 * x + 0] = slot;
            xfer[3 * x + 1] = -1;  // nothing to write back now
            xfer[3 * x + 2] = r;
            slots_out[p] = slot;
          }
          continue;
        }
        const uint32_t smin = __reduce_min_sync(full, cand ? st : 0xffffffffu);
        const int v = __ffs(__ballot_sync(full, cand && st == smin)) - 1;
        const int64_t old = __shfl_sync(full, tag, v);
        ++misses;
        if (old >= 0) ++wbs;
        if (lane == v) {
          tag = r;
          st = stamp;
        }
        prev_slot = (int32_t)(base + v);
        if (lane == 0) {
          const unsigned long long x = atomicAdd(counters + 3, 1ull);
          xfer[3 * x + 0] = base + v;
          xfer[3 * x + 1] = old;
          xfer[3 * x + 2] = r;
          slots_out[p] = prev_slot;
        }
      }
      prev_r = __shfl_sync(full, my_r, mm - 1);
    }
    if (lane < ways) {
      tags[base + lane] = tag;
      stamps[base + lane] = st;
    }
  }
  if (lane == 0 && (misses | wbs | over)) {
    atomicAdd(counters + 0, misses);
    atomicAdd(counters + 1, wbs);
    atomicAdd(counters + 2, over);
  }
}

// copy `bytes` (a multiple of 4) from src to dst with the warp's lanes
__device__ __forceinline__ void warp_copy(void* dst, const void* src, int64_t bytes, int lane) {
  if ((bytes & 15) == 0 && aligned16(dst) && aligned16(src)) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint4* s = reinterpret_cast<const uint4*>(src);
    for (int64_t i = lane; i < bytes / 16; i += kWarp) d[i] = s[i];
  } else {
    unsigned* d = reinterpret_cast<unsigned*>(dst);
    const unsigned* s = reinterpret_cast<const unsigned*>(src);
    for (int64_t i = lane; i < bytes / 4; i += kWarp) d[i] = s[i];
  }
}

__global__ void __launch_bounds__(256)
tier_transfer_kernel(const int64_t* __restrict__ xfer, const unsigned long long* __restrict__ counters,
                     unsigned char* cache_w, unsigned char* cache_m, unsigned char* host_w, unsigned char* host_m,
                     int64_t row_bytes, int64_t mom_bytes) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / kWarp;
  const int64_t nx = (int64_t)counters[3];
  constexpr int U = 4;  // transfers per warp step: U host rows in flight per lane
  const bool fast = row_bytes <= 16 * kWarp && (row_bytes & 15) == 0 && (mom_bytes == 0 || mom_bytes == 4) &&
                    aligned16(cache_w) && aligned16(host_w);
  if (fast) {
    const bool act = lane * 16 < row_bytes;
    for (int64_t i0 = warp * U; i0 < nx; i0 += nwarps * U) {
      int64_t slot[U], old[U], r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = i0 + u < nx;
        slot[u] = ok ? xfer[3 * (i0 + u)] : -1;
        old[u] = ok ? xfer[3 * (i0 + u) + 1] : -1;
        r[u] = ok ? xfer[3 * (i0 + u) + 2] : -1;
      }
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)  // write back the evicted rows (HBM -> host)
        if (act && old[u] >= 0) v[u] = *reinterpret_cast<const uint4*>(cache_w + slot[u] * row_bytes + lane * 16);
      float mv = 0.f;
      if (mom_bytes && lane < U && old[lane] >= 0)
        mv = *reinterpret_cast<const float*>(cache_m + slot[lane] * 4);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act && old[u] >= 0) *reinterpret_cast<uint4*>(host_w + old[u] * row_bytes + lane * 16) = v[u];
      if (mom_bytes && lane < U && old[lane] >= 0) *reinterpret_cast<float*>(host_m + old[lane] * 4) = mv;
#pragma unroll
      for (int u = 0; u < U; ++u)  // fetch (host -> HBM): U loads in flight per lane
        if (act && r[u] >= 0) v[u] = *reinterpret_cast<const uint4*>(host_w + r[u] * row_bytes + lane * 16);
      if (mom_bytes && lane < U && r[lane] >= 0) mv = *reinterpret_cast<const float*>(host_m + r[lane] * 4);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act && r[u] >= 0) *reinterpret_cast<uint4*>(cache_w + slot[u] * row_bytes + lane * 16) = v[u];
      if (mom_bytes && lane < U && r[lane] >= 0) *reinterpret_cast<float*>(cache_m + slot[lane] * 4) = mv;
    }
    return;
  }
  for (int64_t i = warp; i < nx; i += nwarps) {
    const int64_t slot = xfer[3 * i], old = xfer[3 * i + 1], r = xfer[3 * i + 2];
    if (old >= 0) {  // write back the evicted row and its optimizer state
      warp_copy(host_w + old * row_bytes, cache_w + slot * row_bytes, row_bytes, lane);
      if (mom_bytes) warp_copy(host_m + old * mom_bytes, cache_m + slot * mom_bytes, mom_bytes, lane);
    }
    warp_copy(cache_w + slot * row_bytes, host_w + r * row_bytes, row_bytes, lane);
    if (mom_bytes) warp_copy(cache_m + slot * mom_bytes, host_m + r * mom_bytes, mom_bytes, lane);
  }
}

__global__ void __launch_bounds__(256)
tier_flush_kernel(int64_t num_slots, const int64_t* __restrict__ tags, const unsigned char* cache_w,
                  const unsigned char* cache_m, unsigned char* host_w, unsigned char* host_m, int64_t row_bytes,
                  int64_t mom_bytes) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / kWarp;
  for (int64_t slot = warp; slot < num_slots; slot += nwarps) {
    const int64_t r = tags[slot];
    if (r < 0) continue;
    warp_copy(host_w + r * row_bytes, cache_w + slot * row_bytes, row_bytes, lane);
    if (mom_bytes) warp_copy(host_m + r * mom_bytes, cache_m + slot * mom_bytes, mom_bytes, lane);
  }
}

__global__ void __launch_bounds__(256)
tier_spill_writeback_kernel(const int64_t* __restrict__ spill_list, const unsigned long long* __restrict__ counters,
                            int64_t spill_cap, const unsigned char* cache_w, const unsigned char* cache_m,
                            unsigned char* host_w, unsigned char* host_m, int64_t row_bytes, int64_t mom_bytes) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / kWarp;
  const int64_t n = min64((int64_t)counters[4], spill_cap);
  for (int64_t i = warp; i < n; i += nwarps) {
    const int64_t slot = spill_list[2 * i], r = spill_list[2 * i + 1];
    warp_copy(host_w + r * row_bytes, cache_w + slot * row_bytes, row_bytes, lane);
    if (mom_bytes) warp_copy(host_m + r * mom_bytes, cache_m + slot * mom_bytes, mom_bytes, lane);
  }
}

static size_t tier_ws(int64_t n) { return cache_ws(n) + a256(3 * 8 * (size_t)n); }

static unsigned sm_grid(int64_t warps_wanted) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (warps_wanted + 7) / 8;
  return (unsigned)(blocks < 1 ? 1 : (blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8));
}

}  // namespace neo

extern "C" size_t neo_tier_workspace_bytes(int64_t num_ids) { return neo::tier_ws(num_ids < 1 ? 1 : num_ids); }

extern "C" int neo_tier_prepare_spill(int64_t num_rows, int64_t num_sets, int32_t ways, const void* ids,
                                      int32_t index_dtype, int64_t num_ids, int64_t* tags, uint32_t* stamps,
                                      uint32_t stamp, void* cache_weights, void* cache_moments, void* host_weights,
                                      void* host_moments, int64_t row_bytes, int64_t moment_bytes,
                                      int32_t* slots_out, int64_t* counters, int64_t spill_cap, int64_t* spill_list,
                                      void* workspace, size_t workspace_bytes, neo_error* err, void* stream);

extern "C" int neo_tier_prepare(int64_t num_rows, int64_t num_sets, int32_t ways, const void* ids,
                                int32_t index_dtype, int64_t num_ids, int64_t* tags, uint32_t* stamps,
                                uint32_t stamp, void* cache_weights, void* cache_moments, void* host_weights,
                                void* host_moments, int64_t row_bytes, int64_t moment_bytes, int32_t* slots_out,
                                int64_t* counters, void* workspace, size_t workspace_bytes, neo_error* err,
                                void* stream) {
  return neo_tier_prepare_spill(num_rows, num_sets, ways, ids, index_dtype, num_ids, tags, stamps, stamp,
                                cache_weights, cache_moments, host_weights, host_moments, row_bytes, moment_bytes,
                                slots_out, counters, 0, nullptr, workspace, workspace_bytes, err, stream);
}

extern "C" int neo_tier_prepare_spill(int64_t num_rows, int64_t num_sets, int32_t ways, const void* ids,
                                      int32_t index_dtype, int64_t num_ids, int64_t* tags, uint32_t* stamps,
                                      uint32_t stamp, void* cache_weights, void* cache_moments, void* host_weights,
                                      void* host_moments, int64_t row_bytes, int64_t moment_bytes,
                                      int32_t* slots_out, int64_t* counters, int64_t spill_cap, int64_t* spill_list,
                                      void* workspace, size_t workspace_bytes, neo_error* err, void* stream) {
  using namespace neo;
  if (spill_cap < 0 || (spill_cap > 0 && !spill_list)) return fail(NEO_E_ARG, "neo_tier_prepare: spill list");
  cudaStream_t s = as_stream(stream);
  if (num_rows < 1 || num_sets < 1 || num_sets > (int64_t)UINT32_MAX) return fail(NEO_E_ARG, "num_sets/num_rows");
  if (ways < 1 || ways > kWarp) return fail(NEO_E_ARG, "ways: 1..32 (one way per lane)");
  if (index_dtype != NEO_I32 && index_dtype != NEO_I64) return fail(NEO_E_ARG, "index dtype must be I32 or I64");
  if (num_ids < 0 || num_ids >= INT_MAX) return fail(NEO_E_ARG, "num_ids: 0 .. 2^31-1");
  if (row_bytes < 4 || (row_bytes & 3) || (moment_bytes & 3) || stamp == 0)
    return fail(NEO_E_ARG, "row/moment bytes must be multiples of 4; stamp >= 1");
  if (!tags || !stamps || !cache_weights || !host_weights || !slots_out || !counters)
    return fail(NEO_E_ARG, "neo_tier_prepare: null pointer");
  if (cudaMemsetAsync(counters, 0, (spill_cap > 0 ? 5 : 4) * sizeof(int64_t), s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tier_prepare: memset failed");
  const int64_t n = num_ids;
  if (n == 0) return NEO_OK;
  if (workspace_bytes < tier_ws(n)) return fail(NEO_E_ARG, "neo_tier_prepare: workspace too small");
  unsigned char* w = static_cast<unsigned char*>(workspace);
  uint32_t* k0 = reinterpret_cast<uint32_t*>(w); w += a256(4 * (size_t)n);
  uint32_t* k1 = reinterpret_cast<uint32_t*>(w); w += a256(4 * (size_t)n);
  int32_t* v0 = reinterpret_cast<int32_t*>(w); w += a256(4 * (size_t)n);
  int32_t* v1 = reinterpret_cast<int32_t*>(w); w += a256(4 * (size_t)n);
  int32_t* starts = reinterpret_cast<int32_t*>(w); w += a256(4 * (size_t)n);
  int64_t* nseg = reinterpret_cast<int64_t*>(w); w += a256(8);
  void* temp = w; w += a256(cub_bytes(n));
  int64_t* xfer = reinterpret_cast<int64_t*>(w);
  const unsigned kgrid = (unsigned)min64((n + 255) / 256, 148 * 32);
  if (index_dtype == NEO_I32)
    tier_keys_kernel<int32_t><<<kgrid, 256, 0, s>>>((const int32_t*)ids, n, num_rows, num_sets, k0, v0, err);
  else
    tier_keys_kernel<int64_t><<<kgrid, 256, 0, s>>>((const int64_t*)ids, n, num_rows, num_sets, k0, v0, err);
  int rc = check_launch("neo_tier_prepare(keys)");
  if (rc) return rc;
  int bits = 1;
  while (bits < 32 && (uint64_t(1) << bits) < (uint64_t)num_sets) ++bits;
  size_t tb = cub_bytes(n);
  cub::DoubleBuffer<uint32_t> kbuf(k0, k1);
  cub::DoubleBuffer<int32_t> vbuf(v0, v1);
  if (cub::DeviceRadixSort::SortPairs(temp, tb, kbuf, vbuf, (int)n, 0, bits, s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tier_prepare: radix sort failed");
  tb = cub_bytes(n);
  cub::CountingInputIterator<int32_t> it(0);
  if (cub::DeviceSelect::If(temp, tb, it, starts, nseg, (int)n, CacheHead{kbuf.Current()}, s) != cudaSuccess)
    return fail(NEO_E_CUDA, "neo_tier_prepare: segment select failed");
  auto* cnt = reinterpret_cast<unsigned long long*>(counters);
  const unsigned agrid = sm_grid(min64(n, num_sets));
  if (index_dtype == NEO_I32)
    tier_assign_kernel<int32_t><<<agrid, 256, 0, s>>>((const int32_t*)ids, vbuf.Current(), starts, nseg, n, num_rows,
                                                       num_sets, ways, tags, stamps, stamp, slots_out, xfer, cnt,
                                                       spill_cap, spill_list);
  else
    tier_assign_kernel<int64_t><<<agrid, 256, 0, s>>>((const int64_t*)ids, vbuf.Current(), starts, nseg, n, num_rows,
                                                       num_sets, ways, tags, stamps, stamp, slots_out, xfer, cnt,
                                                       spill_cap, spill_list);
  rc = check_launch("neo_tier_prepare(assign)");
  if (rc) return rc;
  tier_transfer_kernel<<<sm_grid(n), 256, 0, s>>>(xfer, cnt, (unsigned char*)cache_weights,
                                                   (unsigned char*)cache_moments, (unsigned char*)host_weights,
                                                   (unsigned char*)host_moments, row_bytes, moment_bytes);
  return check_launch("neo_tier_prepare(transfer)");
}

extern "C" int neo_tier_flush(int64_t num_slots, const int64_t* tags, const void* cache_weights,
                              const void* cache_moments, void* host_weights, void* host_moments, int64_t row_bytes,
                              int64_t moment_bytes, void* stream) {
  using namespace neo;
  if (num_slots < 0 || row_bytes < 4 || (row_bytes & 3) || (moment_bytes & 3))
    return fail(NEO_E_ARG, "neo_tier_flush: bad sizes");
  if (num_slots == 0) return NEO_OK;
  tier_flush_kernel<<<sm_grid(num_slots), 256, 0, as_stream(stream)>>>(
      num_slots, tags, (const unsigned char*)cache_weights, (const unsigned char*)cache_moments,
      (unsigned char*)host_weights, (unsigned char*)host_moments, row_bytes, moment_bytes);
  return check_launch("neo_tier_flush");
}

extern "C" int neo_tier_spill_writeback(const int64_t* spill_list, const int64_t* counters, int64_t spill_cap,
                                        const void* cache_weights, const void* cache_moments, void* host_weights,
                                        void* host_moments, int64_t row_bytes, int64_t moment_bytes, void* stream) {
  using namespace neo;
  if (spill_cap < 0 || row_bytes < 4 || (row_bytes & 3) || (moment_bytes & 3))
    return fail(NEO_E_ARG, "neo_tier_spill_writeback: bad sizes");
  if (spill_cap == 0) return NEO_OK;
  if (!spill_list || !counters) return fail(NEO_E_ARG, "neo_tier_spill_writeback: null pointer");
  tier_spill_writeback_kernel<<<sm_grid(spill_cap), 256, 0, as_stream(stream)>>>(
      spill_list, reinterpret_cast<const unsigned long long*>(counters), spill_cap,
      (const unsigned char*)cache_weights, (const unsigned char*)cache_moments, (unsigned char*)host_weights,
      (unsigned char*)host_moments, row_bytes, moment_bytes);
  return check_launch("neo_tier_spill_writeback");
}
