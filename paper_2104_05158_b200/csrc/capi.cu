// Library-wide plumbing: status messages, error record, device queries.
#include <climits>

#include "common.cuh"

namespace neo {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return fail(NEO_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return NEO_OK;
}

// Resolve the first bad position into (value, table).  Bags of table t cover
// positions [offsets[t*B], offsets[(t+1)*B]); when offsets is NULL the
// record's table field is left as set by the caller.
template <typename Idx>
__global__ void error_finalize_kernel(neo_error* err, const Idx* indices, const int64_t* offsets,
                                      int64_t B, int32_t T) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t pos = err->position;
  if (pos == INT64_MAX) return;
  err->value = static_cast<int64_t>(indices[pos]);
  err->code = NEO_E_INDEX_RANGE;
  if (offsets) {
    int32_t lo = 0, hi = T - 1;  // last t with offsets[t*B] <= pos
    while (lo < hi) {
      int32_t mid = (lo + hi + 1) / 2;
      if (offsets[(int64_t)mid * B] <= pos) lo = mid;
      else hi = mid - 1;
    }
    err->table = lo;
  }
}

void launch_error_finalize(neo_error* err, const void* indices, int32_t index_dtype,
                           const int64_t* offsets, int64_t B, int32_t T, cudaStream_t s) {
  if (!err) return;
  if (index_dtype == NEO_I32)
    error_finalize_kernel<int32_t><<<1, 32, 0, s>>>(err, (const int32_t*)indices, offsets, B, T);
  else
    error_finalize_kernel<int64_t><<<1, 32, 0, s>>>(err, (const int64_t*)indices, offsets, B, T);
}

__global__ void error_reset_kernel(neo_error* err) {
  err->position = INT64_MAX;
  err->value = 0;
  err->table = -1;
  err->code = NEO_OK;
}

}  // namespace neo

extern "C" {

int neo_version(void) { return 10000; }

const char* neo_last_error(void) { return neo::g_last_error.c_str(); }

int neo_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int neo_error_reset(neo_error* err, void* stream) {
  if (!err) return neo::fail(NEO_E_ARG, "neo_error_reset: null record");
  neo::error_reset_kernel<<<1, 1, 0, neo::as_stream(stream)>>>(err);
  return neo::check_launch("neo_error_reset");
}

}  // extern "C"
