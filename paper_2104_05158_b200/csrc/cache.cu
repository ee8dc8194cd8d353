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
  const unsigned waymask = ways >= 32 ? full : ((1u << ways) - 1u);
  unsigned long long h = 0, m = 0, e = 0;
  for (int64_t seg = warp; seg < S; seg += nwarps) {
    const int64_t s0 = starts[seg];
    const int64_t s1 = seg + 1 < S ? (int64_t)starts[seg + 1] : n;
    int64_t row = -1;          // this lane's way
    uint32_t last = 0, freq = 0;
    bool valid = false;
    int cnt = 0;
    int64_t prev_r = -1;  // row of the set's previous access (resident after it)
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
          const unsigned hm = __ballot_sync(full, valid && row == r);
          if (lane == __ffs(hm) - 1) {
            last = clock_end;
            freq += (uint32_t)L;
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
        const unsigned hm = __ballot_sync(full, valid && row == r);
        if (hm) {
          if (lane == __ffs(hm) - 1) {
            last = clock;
            freq += 1;
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
        int tgt;
        if (cnt < ways) {
          tgt = __ffs(~__ballot_sync(full, valid) & waymask) - 1;
          ++cnt;
        } else {
          uint32_t key = valid ? last : UINT_MAX;
          if (lfu) {
            const uint32_t fmin = __reduce_min_sync(full, valid ? freq : UINT_MAX);
            key = (valid && freq == fmin) ? last : UINT_MAX;
          }
          const uint32_t lmin = __reduce_min_sync(full, key);
          tgt = __ffs(__ballot_sync(full, valid && last == lmin)) - 1;
          ev = __shfl_sync(full, row, tgt);
          ++e;
        }
        if (lane == tgt) {
          row = r;
          last = clock;
          freq = 1;
          valid = true;
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
  if (ways > kWarp) return fail(NEO_E_ARG, "ways: this implementation holds one way per lane (<= 32)");
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
  cache_replay_kernel<<<grid, 256, 0, s>>>(trace, vbuf.Current(), starts, nseg, n, ways,
                                           policy == NEO_CACHE_LFU ? 1 : 0, hit, evicted,
                                           reinterpret_cast<unsigned long long*>(stats));
  rc = check_launch("neo_cache_simulate(replay)");
  if (rc) return rc;
  return NEO_OK;
}
