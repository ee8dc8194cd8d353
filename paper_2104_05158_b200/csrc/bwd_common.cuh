// Types shared by the backward translation units (tbe_backward.cu: the
// general / streamed / pipelined paths; tbe_bucket.cu: the bucketed path).
#pragma once
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace neo {

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct SegParams {
  int32_t T;
  int64_t B;
  const int64_t* row_offsets;
  int64_t total_rows;
  const int32_t* dim_offsets;
  int32_t max_dim;
  const uint64_t* weights;
  const uint64_t* moments;
  const void* grad;
  int64_t grad_stride;
  int32_t pooling;
  const int64_t* offsets;  // for MEAN pooling: bag lengths
  int32_t mode;
  int32_t optim;
  double lr;
  double eps;
  int64_t* out_ids;
  void* out_grads;
  const uint64_t* dense_grads;
  const void* keys;
  const int32_t* bags;
  const int32_t* seg_starts;
  const int64_t* num_segs;
  int64_t N;
  int32_t flags;   // NEO_BWD_FLAG_* layout promises from the caller
  int64_t* chunk_counter;  // work-queue counter of the streamed kernel (zeroed per launch)
  int32_t* chunk_slot;     // per 128-entry chunk: partial-sum slot if the chunk lies inside one row, else -1
  float* pool;             // partial sums of such chunks (slot x max_dim, f32)
  unsigned* pool_counter;
  int64_t pool_cap;
  int32_t tma;             // pipelined walk: upstream rows staged by TMA gather4 (uniform full rows)
};

// bucketed path (tbe_bucket.cu)
bool bkt_eligible(const SegParams& p, int32_t weight_dtype, int32_t grad_dtype, bool out_count);
size_t bkt_workspace(int32_t T, int64_t B, int64_t N, int64_t total_rows, int32_t max_dim);
int run_bucket_backward(SegParams p, int32_t weight_dtype, int32_t grad_dtype, const void* indices,
                        int32_t index_dtype, void* workspace, size_t ws_bytes, neo_error* err, cudaStream_t s);

}  // namespace neo
