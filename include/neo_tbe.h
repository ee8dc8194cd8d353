/*
 * neo_tbe.h — C ABI of libneob200.so, the B200-native hot path of Neo
 * (arXiv 2104.05158): table-batched embedding-bag (TBE) forward, the
 * sort/segment-reduce backward fused with the sparse optimizer, row-wise
 * bucketisation, the (W,T,B)<->(T,W,B) block permute and the pooled-row
 * piece copies used around the all-to-all.
 *
 * Every entry point is stream-ordered and asynchronous: all buffers are
 * caller-allocated DEVICE memory unless a parameter says "host"; the library
 * never allocates and never synchronises on the success path.  Return value
 * is a status code (NEO_OK or NEO_E_*): argument errors are detected on the
 * host before any launch; data errors (an out-of-range row id) are recorded
 * on the device in a caller-provided neo_error record that the caller reads
 * after the stream completes.  neo_last_error() returns a thread-local
 * message for the last non-OK status.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/neosim):
 *   neo_tbe_forward            embedding.py:136-151 forward_pooled,
 *                              embedding.py:154-168 fused_forward
 *   neo_tbe_backward (AGGREGATE) embedding.py:175-192 backward_sort_aggregate
 *   neo_tbe_backward (UPDATE)  embedding.py:270-281 fused_backward_update
 *                              (+ embedding.py:212-254 the three optimizers)
 *   neo_tbe_backward (DENSE)   embedding.py:195-205 merge_row_gradients input
 *                              (dense DP gradient for the all-reduce)
 *   neo_apply_row_updates      embedding.py:212-267 apply_rowwise_adagrad /
 *                              apply_adagrad / apply_sgd / apply_optimizer
 *   neo_fp16_roundtrip         embedding.py:288-305 quantize_fp16_roundtrip,
 *                              storage_roundtrip
 *   neo_cast                   comms.py:521-540 quantized communication
 *                              (fp16 fwd / bf16 bwd payloads)
 *   neo_lengths_to_offsets     model.py:365-370 lengths_to_offsets
 *   neo_bucketize_rowwise      comms.py:107-141 bucketize_rowwise
 *   neo_bucketize_rowwise_multi comms.py:107-141 (every row-wise table of a batch in one call)
 *   neo_permute_blocks         comms.py:222-257 permute_WTB_to_TWB /
 *                              permute_TWB_to_WTB (and to_wtb, comms.py:197)
 *   neo_copy_pieces            comms.py:692-711 pooled assembly (TW copy,
 *                              CW column placement, RW partial sum)
 *   neo_copy_chunks            comms.py:692-711 (the same, narrow blocks lane-parallel)
 *   neo_gather_blocks          comms.py:292-353 alltoall_redistribute send
 *                              packing; comms.py:164-172 replicate_columnwise
 */
#ifndef NEO_TBE_H
#define NEO_TBE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
enum {
  NEO_OK = 0,
  NEO_E_INDEX_RANGE = 1, /* errors.py:43 IndexOutOfRange  */
  NEO_E_LAYOUT = 2,      /* errors.py:50 LayoutMismatch   */
  NEO_E_ARG = 3,         /* errors.py:18 InvalidValue     */
  NEO_E_CUDA = 4         /* launch / runtime failure      */
};

/* ---- element types --------------------------------------------------- */
enum { NEO_F32 = 0, NEO_F16 = 1, NEO_F64 = 2, NEO_BF16 = 3 };
enum { NEO_I32 = 0, NEO_I64 = 1 };
enum { NEO_POOL_SUM = 0, NEO_POOL_MEAN = 1 };
/* embedding.py:24-27 OptimizerKind */
enum { NEO_OPT_SGD = 0, NEO_OPT_ROWWISE_ADAGRAD = 1, NEO_OPT_ADAGRAD = 2, NEO_OPT_NONE = 3 };
/* backward modes */
enum {
  NEO_BWD_UPDATE = 0,    /* aggregate + exactly one optimizer step per touched row */
  NEO_BWD_AGGREGATE = 1, /* emit RowGradients (ids ascending, grads) only */
  NEO_BWD_DENSE = 2      /* write aggregated rows into dense per-table gradients */
};
/* optional layout promises OR-ed into `mode` (UPDATE fast path):
 * ALIGNED: every table's D is a multiple of the 16-byte vector, weight rows
 *          and the gradient (base, stride, column offsets) are 16-byte aligned;
 * FULL_ROWS: additionally every D equals 32 vectors (128 f32 / 256 f16). */
enum { NEO_BWD_FLAG_ALIGNED = 0x100, NEO_BWD_FLAG_FULL_ROWS = 0x200 };
/* optional phase split of an UPDATE on the streamed path (same arguments
 * and workspace for both calls): PREPARE builds and sorts the (row, bag)
 * pairs; APPLY (later, possibly on another stream once PREPARE's work is
 * ordered before it) runs the segment walk + optimizer.  Lets the sort of
 * one table group overlap the update of another. */
enum { NEO_BWD_FLAG_PREPARE = 0x400, NEO_BWD_FLAG_APPLY = 0x800 };
/* DIM8: every table's D is a multiple of 8 elements, the weight rows, the
 * gradient base and its row stride are 16-byte aligned.  With SUM pooling,
 * f32/f16 tables, UPDATE (or DENSE on f32) and D <= 256 this selects the
 * bucketed backward (hand-written stable two-level counting sort by row +
 * fused sub-warp-per-row reduce/optimizer); its workspace size is
 * neo_tbe_bucket_workspace_bytes. */
enum { NEO_BWD_FLAG_DIM8 = 0x1000 };

/* Device-side error record (caller allocates sizeof(neo_error) bytes of
 * device memory).  position = first offending position in index-buffer
 * order (INT64_MAX when clean), value = the offending row id, table = the
 * table (or bag group) it belongs to. */
typedef struct neo_error {
  int64_t position;
  int64_t value;
  int32_t table;
  int32_t code;
} neo_error;

int neo_version(void);
const char* neo_last_error(void);
/* number of SMs of the current device (0 if no device) */
int neo_device_sm_count(void);
int neo_error_reset(neo_error* err, void* stream);

/* ---- TBE forward (embedding.py:136-168) -------------------------------
 * T tables, B bags per table.  Bag (t, b) covers positions
 * offsets[t*B+b] .. offsets[t*B+b+1] of the concatenated index buffer
 * (model.py:301-337 CombinedBatch: table-major, then sample-major).
 * Table t: rows row_offsets[t+1]-row_offsets[t], dim dim_offsets[t+1]-
 * dim_offsets[t], values at weights[t] (row-major, weight_dtype).
 * out[b*out_stride + dim_offsets[t] + j] = sum over the bag (SUM) or the bag
 * mean (MEAN; empty bag -> 0).  F64 weights accumulate in f64, sequentially in
 * buffer order (bit-identical to np.add.at); F32/F16 accumulate in f32. */
int neo_tbe_forward(int32_t num_tables, int64_t batch,
                    const int64_t* row_offsets,  /* [T+1] */
                    const int32_t* dim_offsets,  /* [T+1] */
                    int32_t max_dim,
                    const uint64_t* weights,     /* [T] device pointers */
                    int32_t weight_dtype,
                    const void* indices, int32_t index_dtype,
                    const int64_t* offsets,      /* [T*B+1] */
                    int32_t pooling,
                    void* out, int32_t out_dtype, int64_t out_stride,
                    neo_error* err,              /* may be NULL */
                    void* stream);

/* Cap the forward's grid at ctas_per_sm CTAs per SM (grid-stride over bags;
 * 0 = uncapped, the default).  A capped, DRAM-bound forward leaves SM
 * resources to a concurrent side-stream kernel, e.g. the next backward's key
 * build + radix sort (NEO_BWD_FLAG_PREPARE).  Process-wide setting; no
 * reference counterpart (scheduling knob of this implementation). */
int neo_set_forward_residency(int32_t ctas_per_sm);

/* Same, with the pooled all-to-all fused into the store: bag row b (of the
 * batch rows) is written to out_ptrs[b / rows_per_dst] at row b %
 * rows_per_dst (out_ptrs: device array of destination base pointers, e.g.
 * peer GPUs' symmetric receive buffers mapped over NVLink; comms.py:366-392
 * pooled AlltoAll). */
int neo_tbe_forward_scatter(int32_t num_tables, int64_t batch,
                            const int64_t* row_offsets, const int32_t* dim_offsets, int32_t max_dim,
                            const uint64_t* weights, int32_t weight_dtype,
                            const void* indices, int32_t index_dtype,
                            const int64_t* offsets, int32_t pooling,
                            const uint64_t* out_ptrs, int64_t rows_per_dst,
                            int32_t out_dtype, int64_t out_stride,
                            neo_error* err, void* stream);

/* ---- TBE backward (embedding.py:175-281) ------------------------------
 * Sort (table row, bag) pairs stably by row, run-length segment them, then
 * one warp per touched row sums the upstream rows of its occurrences in
 * buffer order and, in UPDATE mode, applies exactly one optimizer step in
 * place (no dense gradient is materialised).
 *   grad: upstream gradient, row b of table t at grad[b*grad_stride +
 *         dim_offsets[t] ..], grad_dtype F32/BF16/F16 (F64 with F64 weights)
 *   moments[t]: row-wise (H_t) or element-wise (H_t x D_t) state, f32 for
 *         F32/F16 weights, f64 for F64 weights; ignored for SGD
 *   AGGREGATE: out_ids[u] = row_offsets[t] + row (ascending), out_grads
 *         (U x max_dim, accumulator type), *out_count = U (device int64)
 *   DENSE: dense_grads[t] (H_t x D_t, accumulator type, pre-zeroed) get the
 *         aggregated rows.
 * num_indices must equal offsets[T*B] - offsets[0] (the ids the bags cover).
 * Workspace size: neo_tbe_backward_workspace_bytes. */
size_t neo_tbe_backward_workspace_bytes(int64_t num_indices, int64_t total_rows, int32_t max_dim);
/* workspace of the bucketed path (NEO_BWD_FLAG_DIM8) for T tables of B bags */
size_t neo_tbe_bucket_workspace_bytes(int32_t num_tables, int64_t batch, int64_t num_indices,
                                      int64_t total_rows, int32_t max_dim);

int neo_tbe_backward(int32_t num_tables, int64_t batch,
                     const int64_t* row_offsets, int64_t total_rows,
                     const int32_t* dim_offsets, int32_t max_dim,
                     const uint64_t* weights, int32_t weight_dtype,
                     const uint64_t* moments,      /* [T] or NULL */
                     const void* indices, int32_t index_dtype,
                     const int64_t* offsets, int64_t num_indices,
                     int32_t pooling,
                     const void* grad, int32_t grad_dtype, int64_t grad_stride,
                     int32_t mode, int32_t optim, double lr, double eps,
                     int64_t* out_ids, void* out_grads, int64_t* out_count,
                     const uint64_t* dense_grads,  /* [T] or NULL */
                     void* workspace, size_t workspace_bytes,
                     neo_error* err, void* stream);

/* ---- sparse optimizer from RowGradients (embedding.py:212-267) ---------
 * ids: n row ids (NULL = rows 0..n-1, the dense-gradient case);
 * grads: n x dim in the accumulator type of weight_dtype (f64 for F64,
 * else f32).  Rows whose gradient is identically zero are skipped for the
 * AdaGrad variants (embedding.py:225-228). */
int neo_apply_row_updates(int64_t n, const int64_t* ids, const void* grads,
                          int32_t dim, void* weight, int32_t weight_dtype,
                          void* moment, int32_t optim, double lr, double eps,
                          void* stream);

/* ---- precision (embedding.py:288-305, comms.py:521-540) --------------- */
/* x (f64, n) -> RNE through binary16 -> f64 in place; overflow[i] = 1 where
 * the result is +-inf (may be NULL); *nonfinite (device int32, may be NULL)
 * set to 1 when an input is non-finite. */
int neo_fp16_roundtrip(int64_t n, double* x, uint8_t* overflow, int32_t* nonfinite,
                       void* stream);
/* element-wise RNE conversion between NEO_F32/F16/BF16/F64 */
int neo_cast(int64_t n, const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype,
             void* stream);

/* ---- jagged metadata (model.py:365-370) -------------------------------- */
int neo_lengths_to_offsets(int64_t n, const int64_t* lengths, int64_t* offsets /* n+1 */,
                           void* workspace, size_t workspace_bytes, void* stream);
size_t neo_scan_workspace_bytes(int64_t n);

/* ---- id range check (model.py:344-348 CombinedBatch validation) -------
 * Table t's ids (positions offsets[t*B] .. offsets[(t+1)*B]) must lie in
 * [0, rows[t]) (rows: device int64 [T]); the first offending position, its
 * value and table are recorded in err (IndexOutOfRange).  T <= 65535. */
int neo_check_indices(int32_t num_tables, int64_t batch, const int64_t* rows, const int64_t* offsets,
                      const void* indices, int32_t index_dtype, neo_error* err, void* stream);

/* ---- row-wise bucketisation (comms.py:107-141) -------------------------
 * n bags with offsets[n+1] over indices; shard s owns rows
 * [shard_starts[s], shard_starts[s+1]) (k+1 host values, tiling [0,H)).
 * Outputs: out_lengths (k x n, shard-major), out_offsets (k*n+1, exclusive
 * scan of out_lengths: shard s occupies out_indices[out_offsets[s*n] ..
 * out_offsets[(s+1)*n])), out_indices (N, rebased to the shard, original
 * order kept inside each shard).  Bit-exact. */
size_t neo_bucketize_workspace_bytes(int64_t n, int32_t k);
int neo_bucketize_rowwise(int64_t n, const int64_t* offsets, const void* indices,
                          int32_t index_dtype, int32_t k, const int64_t* shard_starts_host,
                          int64_t* out_lengths, int64_t* out_offsets, void* out_indices,
                          int32_t table, neo_error* err,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Row-wise bucketisation of many tables in one call (the sharded step's
 * sender side, comms.py:107-141 applied per row-wise table): tables[r]
 * (device, num_rw) names table r's bags in the full batch (offsets over
 * T*batch bags, device); shard_starts (device, num_rw x (kmax+1)) holds table
 * r's shard_counts[r] + 1 boundaries.  out_lengths (num_rw, kmax, batch),
 * out_offsets its exclusive scan (num_rw*kmax*batch + 1), out_indices the ids
 * grouped by (table, shard, bag), rebased to the shard.  Ids outside their
 * table are skipped (validate them first with neo_check_indices).
 * Workspace: neo_bucketize_workspace_bytes(num_rw * batch, kmax). */
int neo_bucketize_rowwise_multi(int32_t num_rw, int64_t batch, const int32_t* tables, const int64_t* offsets,
                                const void* indices, int32_t index_dtype, int32_t kmax, const int64_t* shard_starts,
                                const int32_t* shard_counts, int64_t* out_lengths, int64_t* out_offsets,
                                void* out_indices, void* workspace, size_t workspace_bytes, void* stream);

/* ---- block permute (comms.py:222-264) ----------------------------------
 * lengths: outer*inner*B entries whose (o, i) block of B lengths covers the
 * next sum(lengths) indices; output is the (i, o) block order.  WTB->TWB is
 * outer=W, inner=T; TWB->WTB is outer=T, inner=W. */
size_t neo_permute_workspace_bytes(int32_t outer, int32_t inner);
int neo_permute_blocks(int32_t outer, int32_t inner, int64_t B,
                       const int64_t* lengths, const void* indices, int32_t index_dtype,
                       int64_t* out_lengths, void* out_indices,
                       void* workspace, size_t workspace_bytes, void* stream);

/* ---- pooled-row pieces (comms.py:692-711) ------------------------------
 * For r in [0, rows): dst[r*dst_stride + dst_col + j] (=|+=) cast(src[r*
 * src_stride + src_col + j]) for j < width, pieces applied in array order
 * (so RW partial pools add in shard order).  pieces: device array of
 * neo_piece.  src/dst dtypes F32/F16/BF16/F64. */
typedef struct neo_piece {
  uint64_t src;        /* device pointer */
  uint64_t dst;        /* device pointer */
  int64_t src_stride;  /* elements */
  int64_t dst_stride;  /* elements */
  int32_t src_col;
  int32_t dst_col;
  int32_t width;
  int32_t accumulate;  /* 0 = overwrite, 1 = add */
} neo_piece;
int neo_copy_pieces(int64_t rows, const neo_piece* pieces, int32_t num_pieces,
                    int32_t src_dtype, int32_t dst_dtype, void* stream);
/* The same for pieces cut into 16-byte vectors (on the narrower dtype's
 * side): chunk c moves, for every row r, the vector at src + r*src_stride to
 * dst + r*dst_stride (byte addresses / strides, 16-byte aligned), converting.
 * Chunks are independent (overwrite only, disjoint destinations), so lanes
 * take them in parallel: used for the many narrow column blocks of the
 * sharded exchange (comms.py:692-711); accumulating pieces stay ordered in
 * neo_copy_pieces. */
typedef struct neo_chunk {
  uint64_t src;
  uint64_t dst;
  int64_t src_stride;  /* bytes */
  int64_t dst_stride;  /* bytes */
} neo_chunk;
int neo_copy_chunks(int64_t rows, const neo_chunk* chunks, int32_t num_chunks,
                    int32_t src_dtype, int32_t dst_dtype, void* stream);

/* ---- block gather (comms.py:292-353 send packing, comms.py:164-172) ----
 * dst[dst_off[i] .. dst_off[i]+count[i]) = src_ptr[i][0 .. count[i]) for
 * each of n blocks; elem_bytes 4 or 8 (indices, lengths).  Blocks are
 * device arrays. */
int neo_gather_blocks(int32_t n, const uint64_t* src_ptrs, const int64_t* counts,
                      const int64_t* dst_offsets, void* dst, int32_t elem_bytes,
                      void* stream);

/* ---- software row cache (cache.py:68-133) -------------------------------
 * Replays an access trace through a num_sets x ways set-associative cache
 * (set = row % num_sets) with LRU or LFU replacement exactly as the
 * reference's sequential access() loop does (cache.py:68-98), on the device:
 * hit[p] (uint8, may be NULL) and evicted[p] (int64 row or -1, may be NULL)
 * receive access p's AccessResult; stats[0..2] (device int64) = hits,
 * misses, evictions (cache.py:117-126 TraceStats).  A negative row is
 * recorded in err (first position); the reference raises InvalidValue
 * ("row_id") there.  ways <= 128 (up to four ways per lane).  Replaces
 * neosim.cache.simulate_trace / access over a trace. */
enum { NEO_CACHE_LRU = 0, NEO_CACHE_LFU = 1 };
size_t neo_cache_workspace_bytes(int64_t num_accesses);
int neo_cache_simulate(int64_t num_sets, int32_t ways, int32_t policy, const int64_t* trace,
                       int64_t num_accesses, uint8_t* hit, int64_t* evicted, int64_t* stats,
                       void* workspace, size_t workspace_bytes, neo_error* err, void* stream);

/* ---- HBM tier over host-resident tables -------------
 * One table: rows (row_bytes each, optimizer state moment_bytes each, 0 for
 * SGD) live in host memory the device can address (pinned, UVA); an HBM
 * cache of num_sets x ways slots (cache_weights / cache_moments, slot-major)
 * holds the rows in use.  neo_tier_prepare maps the batch's ids to slots
 * (slots_out, int32, same order as ids), writing evicted slots back to host
 * and fetching missing rows; rows the batch uses are never evicted by it.
 * tags[num_sets*ways] (int64 row or -1) and stamps[...] (uint32, 0 = never)
 * are the caller-owned directory; stamp = this batch's number (>= 1,
 * increasing).  counters[4] (device int64) = misses, write-backs, accesses
 * that found no free way (set overflow: slot -1), transfers.  Out-of-range
 * ids are recorded in err.  neo_tier_flush writes every cached row back.
 * No reference counterpart: the reference models this tier analytically
 * (cache.py:129-136 effective_row_bandwidth, planner.py:512-522 hbm+dram). */
size_t neo_tier_workspace_bytes(int64_t num_ids);
int neo_tier_prepare(int64_t num_rows, int64_t num_sets, int32_t ways, const void* ids, int32_t index_dtype,
                     int64_t num_ids, int64_t* tags, uint32_t* stamps, uint32_t stamp, void* cache_weights,
                     void* cache_moments, void* host_weights, void* host_moments, int64_t row_bytes,
                     int64_t moment_bytes, int32_t* slots_out, int64_t* counters, void* workspace,
                     size_t workspace_bytes, neo_error* err, void* stream);
/* neo_tier_prepare with set-overflow spill: an access whose set has no free
 * way this batch (more than `ways` distinct rows of the set in the batch)
 * takes one of spill_cap extra slots after the cache (slot num_sets*ways + k;
 * cache_weights / cache_moments must hold them), fetched like a miss; its
 * (slot, row) pair goes to spill_list[2k..2k+1] and counters[4] counts the
 * spills (counters: 5 int64).  neo_tier_spill_writeback, issued after the
 * backward, writes the spilled rows (and their optimizer state) back to host.
 * Only spills beyond spill_cap map to slot -1 (counters[2]). */
int neo_tier_prepare_spill(int64_t num_rows, int64_t num_sets, int32_t ways, const void* ids, int32_t index_dtype,
                           int64_t num_ids, int64_t* tags, uint32_t* stamps, uint32_t stamp, void* cache_weights,
                           void* cache_moments, void* host_weights, void* host_moments, int64_t row_bytes,
                           int64_t moment_bytes, int32_t* slots_out, int64_t* counters, int64_t spill_cap,
                           int64_t* spill_list, void* workspace, size_t workspace_bytes, neo_error* err, void* stream);
int neo_tier_spill_writeback(const int64_t* spill_list, const int64_t* counters, int64_t spill_cap,
                             const void* cache_weights, const void* cache_moments, void* host_weights,
                             void* host_moments, int64_t row_bytes, int64_t moment_bytes, void* stream);
int neo_tier_flush(int64_t num_slots, const int64_t* tags, const void* cache_weights, const void* cache_moments,
                   void* host_weights, void* host_moments, int64_t row_bytes, int64_t moment_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NEO_TBE_H */
