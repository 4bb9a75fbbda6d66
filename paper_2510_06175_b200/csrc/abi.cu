// ABI plumbing: version, thread-local error strings, status names, device attribute cache.
#include <stdarg.h>
#include <stdio.h>
#include <mutex>

#include "common.cuh"

namespace vecinfer {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

vecinfer_status_t fail(vecinfer_status_t st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

vecinfer_status_t check_paged(const vecinfer_paged_t* pg, int64_t n_cap, const char* who) {
  if (!pg->block_table) return fail(VECINFER_ERR_INVALID_ARG, "%s: paged cache without block_table", who);
  const int ps = pg->page_size;
  if (ps < 32 || (ps & (ps - 1)) != 0)
    return fail(VECINFER_ERR_INVALID_ARG, "%s: page_size %d must be a power of two >= 32", who, ps);
  if (pg->n_pages <= 0) return fail(VECINFER_ERR_SHAPE, "%s: n_pages must be > 0", who);
  if (pg->bt_stride <= 0 || pg->bt_stride * static_cast<int64_t>(ps) < n_cap)
    return fail(VECINFER_ERR_SHAPE, "%s: bt_stride * page_size must cover n_cap", who);
  return VECINFER_OK;
}

vecinfer_status_t check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VECINFER_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return VECINFER_OK;
}

int device_sm_count() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

}  // namespace vecinfer

namespace vecinfer {
static unsigned long long* g_phase = nullptr;
unsigned long long* phase_buffer() { return g_phase; }
}  // namespace vecinfer
#ifdef VECINFER_PHASE_TIMING
// profiling builds only: device buffer of [n_cta][8] u64 globaltimer stamps
extern "C" int vecinfer_debug_set_phase_buffer(void* p) {
  vecinfer::g_phase = static_cast<unsigned long long*>(p);
  return 0;
}
#endif

extern "C" {

int vecinfer_abi_version(void) { return VECINFER_ABI_VERSION; }

const char* vecinfer_last_error(void) { return vecinfer::g_err; }

const char* vecinfer_status_string(vecinfer_status_t s) {
  switch (s) {
    case VECINFER_OK: return "VECINFER_OK";
    case VECINFER_ERR_INVALID_ARG: return "VECINFER_ERR_INVALID_ARG";
    case VECINFER_ERR_SHAPE: return "VECINFER_ERR_SHAPE";
    case VECINFER_ERR_UNSUPPORTED: return "VECINFER_ERR_UNSUPPORTED";
    case VECINFER_ERR_EMPTY: return "VECINFER_ERR_EMPTY";
    case VECINFER_ERR_RANGE: return "VECINFER_ERR_RANGE";
    case VECINFER_ERR_WORKSPACE: return "VECINFER_ERR_WORKSPACE";
    case VECINFER_ERR_CUDA: return "VECINFER_ERR_CUDA";
  }
  return "VECINFER_UNKNOWN_STATUS";
}

}  // extern "C"
