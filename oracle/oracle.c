/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's arithmetic for the hot path, used
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the checker.  Never linked into or called by the product library.
 *
 * Every loop follows the evaluation order of the numpy primitive the
 * reference uses, so results are bit-identical to /root/reference (pinned
 * in tests/test_oracle.py against fixtures produced by the reference):
 *   forward   embedding.py:147-150  np.add.at(out, sample_ids, values[idx]):
 *             per output row, a sequential sum from +0.0 in buffer order
 *   backward  embedding.py:188-191  np.unique + np.add.at: stable grouping by
 *             row id, sequential sum from +0.0 in buffer order
 *   rowwise   embedding.py:225-231  np.mean(g*g, axis=1) = numpy pairwise
 *             sum (8 accumulators, blocks of 128) / D; m += mean;
 *             w -= (lr*g) / (sqrt(m) + eps); zero rows skipped
 *   adagrad   embedding.py:241-246; sgd embedding.py:253
 *   bucketize comms.py:131-140 searchsorted(ends, idx, 'right') + masks
 *   cache     cache.py:68-98 access(): set = row % num_sets; hit refreshes
 *             last_used (global clock) and frequency; a miss into a full set
 *             evicts argmin (last_used, i) [LRU] or (frequency, last_used, i)
 *             [LFU] and appends the new line
 * Compiled with -ffp-contract=off so no a*b+c is fused.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* forward_pooled: returns the first out-of-range position or -1 */
int64_t or_forward_f64(int64_t n, const int64_t* offsets, const int64_t* idx, int64_t H, int64_t D,
                       const double* values, double* out) {
  int64_t total = offsets[n] - offsets[0];
  for (int64_t p = 0; p < total; ++p) {
    int64_t v = idx[offsets[0] + p];
    if (v < 0 || v >= H) return offsets[0] + p;
  }
  for (int64_t s = 0; s < n; ++s) {
    double* o = out + s * D;
    for (int64_t j = 0; j < D; ++j) o[j] = 0.0;
    for (int64_t p = offsets[s]; p < offsets[s + 1]; ++p) {
      const double* row = values + idx[p] * D;
      for (int64_t j = 0; j < D; ++j) o[j] = o[j] + row[j];
    }
  }
  return -1;
}

/* backward_sort_aggregate over ids in [lo, lo+range): counting sort by id
 * (stable), then per id a sequential sum of upstream rows in buffer order.
 * out_ids/out_grads sized for the number of distinct ids; returns U. */
int64_t or_backward_aggregate_f64(int64_t n, const int64_t* offsets, const int64_t* idx,
                                  int64_t lo, int64_t range, int64_t D, const double* upstream,
                                  int64_t* out_ids, double* out_grads) {
  int64_t base = offsets[0], N = offsets[n] - base;
  int64_t* count = (int64_t*)calloc((size_t)range + 1, sizeof(int64_t));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N ? N : 1));
  int64_t* sample = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N ? N : 1));
  for (int64_t s = 0; s < n; ++s)
    for (int64_t p = offsets[s]; p < offsets[s + 1]; ++p) sample[p - base] = s;
  for (int64_t p = 0; p < N; ++p) count[idx[base + p] - lo + 1]++;
  for (int64_t r = 0; r < range; ++r) count[r + 1] += count[r];
  for (int64_t p = 0; p < N; ++p) order[count[idx[base + p] - lo]++] = p; /* stable */
  int64_t U = 0;
  for (int64_t q = 0; q < N;) {
    int64_t id = idx[base + order[q]];
    double* g = out_grads + U * D;
    for (int64_t j = 0; j < D; ++j) g[j] = 0.0;
    for (; q < N && idx[base + order[q]] == id; ++q) {
      const double* u = upstream + sample[order[q]] * D;
      for (int64_t j = 0; j < D; ++j) g[j] = g[j] + u[j];
    }
    out_ids[U++] = id;
  }
  free(count);
  free(order);
  free(sample);
  return U;
}

/* numpy pairwise_sum (umath loops_utils.h.src) of x_i = g_i*g_i */
static double pairwise_sq(const double* g, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = r + g[i] * g[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = g[j] * g[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = r[j] + g[i + j] * g[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + g[i] * g[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sq(g, n2) + pairwise_sq(g + n2, n - n2);
}

static int row_is_zero(const double* g, int64_t D) {
  for (int64_t j = 0; j < D; ++j)
    if (g[j] != 0.0) return 0;
  return 1;
}

/* kind: 0 sgd, 1 rowwise adagrad, 2 adagrad (embedding.py:212-254) */
void or_apply_f64(int kind, int64_t U, const int64_t* ids, const double* grads, int64_t D,
                  double* values, double* moment, double lr, double eps) {
  for (int64_t u = 0; u < U; ++u) {
    const double* g = grads + u * D;
    double* w = values + ids[u] * D;
    if (kind == 0) {
      for (int64_t j = 0; j < D; ++j) w[j] = w[j] - lr * g[j];
      continue;
    }
    if (row_is_zero(g, D)) continue;
    if (kind == 1) {
      double m = moment[ids[u]] + pairwise_sq(g, D) / (double)D;
      moment[ids[u]] = m;
      double denom = sqrt(m) + eps;
      for (int64_t j = 0; j < D; ++j) w[j] = w[j] - (lr * g[j]) / denom;
    } else {
      double* m = moment + ids[u] * D;
      for (int64_t j = 0; j < D; ++j) {
        m[j] = m[j] + g[j] * g[j];
        w[j] = w[j] - (lr * g[j]) / (sqrt(m[j]) + eps);
      }
    }
  }
}

/* bucketize_rowwise: shard s owns [starts[s], starts[s+1]); out_lengths
 * (k x n), out_indices grouped by shard (shard-major, buffer order kept);
 * returns first bad position or -1 */
int64_t or_bucketize(int64_t n, const int64_t* offsets, const int64_t* idx, int k,
                     const int64_t* starts, int64_t* out_lengths, int64_t* out_indices) {
  int64_t base = offsets[0], N = offsets[n] - base, H = starts[k];
  for (int64_t p = 0; p < N; ++p)
    if (idx[base + p] < 0 || idx[base + p] >= H) return base + p;
  memset(out_lengths, 0, sizeof(int64_t) * (size_t)k * (size_t)n);
  int64_t w = 0;
  for (int s = 0; s < k; ++s) {
    for (int64_t b = 0; b < n; ++b) {
      for (int64_t p = offsets[b]; p < offsets[b + 1]; ++p) {
        int64_t v = idx[p];
        /* searchsorted(ends, v, 'right'): first shard whose end exceeds v */
        int sh = 0;
        while (sh < k - 1 && v >= starts[sh + 1]) ++sh;
        if (sh != s) continue;
        out_lengths[(int64_t)s * n + b]++;
        out_indices[w++] = v - starts[s];
      }
    }
  }
  return -1;
}


/* cache.py:68-98 access() over a whole trace (cache.py:117-126
 * simulate_trace).  Lines of a set are kept in the reference's list order
 * (append on insert, delete the victim).  Returns the first position with a
 * negative row (the reference raises there), else -1.  hit/evicted may be
 * NULL; evicted[p] = -1 when access p evicted nothing. */
int64_t or_cache_simulate(int64_t num_sets, int64_t ways, int lfu, int64_t n, const int64_t* trace,
                          uint8_t* hit, int64_t* evicted, int64_t* stats) {
  int64_t* row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(num_sets * ways));
  int64_t* last = (int64_t*)malloc(sizeof(int64_t) * (size_t)(num_sets * ways));
  int64_t* freq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(num_sets * ways));
  int64_t* len = (int64_t*)calloc((size_t)num_sets, sizeof(int64_t));
  int64_t hits = 0, misses = 0, evictions = 0, clock = 0, bad = -1;
  for (int64_t p = 0; p < n; ++p) {
    const int64_t r = trace[p];
    if (r < 0) { bad = p; break; }
    const int64_t s = r % num_sets;
    int64_t* R = row + s * ways; int64_t* Lu = last + s * ways; int64_t* F = freq + s * ways;
    clock += 1;
    int64_t i, found = -1;
    for (i = 0; i < len[s]; ++i) if (R[i] == r) { found = i; break; }
    if (found >= 0) {
      Lu[found] = clock; F[found] += 1; hits += 1;
      if (hit) hit[p] = 1;
      if (evicted) evicted[p] = -1;
      continue;
    }
    misses += 1;
    int64_t ev = -1;
    if (len[s] >= ways) {
      int64_t v = 0;
      for (i = 1; i < len[s]; ++i) {
        if (lfu) {
          if (F[i] < F[v] || (F[i] == F[v] && Lu[i] < Lu[v])) v = i;
        } else if (Lu[i] < Lu[v]) v = i;
      }
      ev = R[v];
      for (i = v; i + 1 < len[s]; ++i) { R[i] = R[i + 1]; Lu[i] = Lu[i + 1]; F[i] = F[i + 1]; }
      len[s] -= 1; evictions += 1;
    }
    R[len[s]] = r; Lu[len[s]] = clock; F[len[s]] = 1; len[s] += 1;
    if (hit) hit[p] = 0;
    if (evicted) evicted[p] = ev;
  }
  stats[0] = hits; stats[1] = misses; stats[2] = evictions;
  free(row); free(last); free(freq); free(len);
  return bad;
}
