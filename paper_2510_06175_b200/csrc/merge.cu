// N5: log-sum-exp merge of P normalised partials (cross-GPU shards, residual window).
//   L = logsumexp_s L_s;  o = sum_s exp(L_s - L) o_s  in the fixed order s = 0..P-1
// (the online-softmax recurrence of P:745-757 applied to whole partials).
// One CTA per (b, h_q) row, one thread per dim; tiny and latency-bound.
#include <string.h>

#include "common.cuh"

namespace vecinfer {
namespace {

__global__ void merge_lse_kernel(const float* __restrict__ o_parts, const float* __restrict__ lse_parts, int P,
                                 int64_t rows, int D, void* o, int o_f32, float* lse) {
  const int64_t row = blockIdx.x;
  float M = -INFINITY;
  for (int s = 0; s < P; ++s) M = fmaxf(M, lse_parts[s * rows + row]);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float wsum = 0.f, osum = 0.f;
    if (M != -INFINITY) {
      for (int s = 0; s < P; ++s) {
        const float f = __expf(lse_parts[s * rows + row] - M);
        wsum += f;
        osum += f * o_parts[(s * rows + row) * D + d];
      }
    }
    const bool empty = !(wsum > 0.f);
    const float v = empty ? 0.f : osum / wsum;
    if (o_f32) static_cast<float*>(o)[row * D + d] = v;
    else static_cast<__nv_bfloat16*>(o)[row * D + d] = __float2bfloat16_rn(v);
    if (d == 0 && lse) lse[row] = empty ? -INFINITY : M + __logf(wsum);
  }
}

}  // namespace
}  // namespace vecinfer

using namespace vecinfer;

extern "C" vecinfer_status_t vecinfer_merge_lse(const float* o_parts, const float* lse_parts, int32_t P, int32_t B,
                                                int32_t H_q, int32_t D, void* o, vecinfer_dtype_t o_dtype, float* lse,
                                                vecinfer_stream_t stream) {
  if (!o_parts || !lse_parts || !o) return fail(VECINFER_ERR_INVALID_ARG, "merge_lse: NULL pointer");
  if (o_dtype != VECINFER_BF16 && o_dtype != VECINFER_F32) return fail(VECINFER_ERR_INVALID_ARG, "merge_lse: bad o_dtype");
  if (P <= 0 || B <= 0 || H_q <= 0 || D <= 0) return fail(VECINFER_ERR_SHAPE, "merge_lse: non-positive size");
  const int64_t rows = static_cast<int64_t>(B) * H_q;
  if (rows > 2147483647) return fail(VECINFER_ERR_SHAPE, "merge_lse: too many rows");
  const int threads = D >= 128 ? 128 : ((D + 31) / 32) * 32;
  merge_lse_kernel<<<static_cast<unsigned>(rows), threads, 0, as_stream(stream)>>>(o_parts, lse_parts, P, rows, D, o,
                                                                                    o_dtype == VECINFER_F32, lse);
  return check_launch("merge_lse_kernel");
}

// ---------------------------------------------------------------------------------------------
// N5-P2P: the cross-GPU exchange of the sequence-sharded partials fused with their merge, over
// peer memory ("N4's epilogue stores partials straight into peers' windows ... then
// local N5").  Every rank owns one window in its own HBM, mapped by all peers through CUDA IPC
// (NVLink/NVSwitch P2P between GPUs).  One CTA per (b, h_q) row:
//   1. publish: the row's (o_r, L_r) is stored into slot [epoch & 1][rank] of EVERY rank's window
//      (remote stores), then, after a system-scope fence, a release store of flag = epoch;
//   2. wait: thread 0 acquire-polls the P flags of the row in its own window until all equal epoch
//      (bounded by a timeout: VECINFER_FLAG_P2P_TIMEOUT instead of a hang);
//   3. merge: the P partials, read from the own window, combined in rank order with exactly the
//      arithmetic of merge_lse_kernel, so the result is bitwise that of all-gather + merge_lse.
// Epoch parity double-buffers the slots: a peer can run at most one exchange ahead (it cannot
// finish exchange e+1 before this rank publishes e+1, i.e. before this rank has finished e).
namespace vecinfer {
namespace {

// window = [256-byte header: u32 epoch counter, u32 CTA-done counter][data][flags]
struct P2PLayout {
  int64_t rows;
  int P, D;
  static constexpr int64_t kHeader = 256;
  __host__ __device__ int64_t data_off(int par, int src, int64_t row) const {   // floats
    return kHeader / 4 + ((static_cast<int64_t>(par) * P + src) * rows + row) * (D + 1);
  }
  __host__ __device__ int64_t flag_off_bytes(int par, int src, int64_t row) const {
    return kHeader + 2ll * P * rows * (D + 1) * 4 + ((static_cast<int64_t>(par) * P + src) * rows + row) * 4;
  }
  __host__ __device__ int64_t bytes() const { return kHeader + 2ll * P * rows * ((D + 1) * 4 + 4); }
};

__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void merge_lse_p2p_kernel(const float* __restrict__ o_local, const float* __restrict__ lse_local,
                                     void* const* __restrict__ windows, P2PLayout lay, int rank, uint32_t epoch,
                                     void* o, int o_f32, float* lse, uint32_t* err, unsigned long long timeout_ns) {
  // Persistent grid (at most the co-resident CTA count, see the launch): CTA c owns rows c, c+grid,
  // ...; it publishes ALL of its rows before it waits for any, so progress never depends on the
  // hardware dispatching CTAs in any particular order on any rank.
  const int D = lay.D, P = lay.P;
  const int64_t rows = lay.rows;
  __shared__ int s_ok;
  __shared__ uint32_t s_epoch;
  // epoch 0 = automatic: the own window's header counter + 1 (every CTA reads it before the last
  // CTA of this launch advances it; the next launch on the stream starts after this one ends), so
  // the exchange can be captured in a CUDA graph and replayed
  uint32_t* hdr = static_cast<uint32_t*>(windows[rank]);
  if (threadIdx.x == 0) {
    uint32_t e = epoch;
    if (e == 0) { e = *reinterpret_cast<volatile uint32_t*>(hdr) + 1u; if (e == 0) e = 1u; }
    s_epoch = e;
  }
  __syncthreads();
  epoch = s_epoch;
  const int par = static_cast<int>(epoch & 1u);
  // 1. publish this rank's partial rows into every window (own included)
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    for (int p = 0; p < P; ++p) {
      float* dst = static_cast<float*>(windows[p]) + lay.data_off(par, rank, row);
      for (int d = threadIdx.x; d < D; d += blockDim.x) dst[d] = o_local[row * D + d];
      if (threadIdx.x == 0) dst[D] = lse_local[row];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();   // cumulative: the CTA's data stores (ordered by the barrier) first
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x)
      for (int p = 0; p < P; ++p)
        st_release_sys_u32(reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(windows[p]) +
                                                       lay.flag_off_bytes(par, rank, row)), epoch);
  }
  const unsigned long long t0 = globaltimer_ns();
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    // 2. wait for the P partials of this row in the own window
    if (threadIdx.x == 0) {
      const unsigned char* mine = static_cast<const unsigned char*>(windows[rank]);
      int ok = 1;
      for (int q = 0; q < P && ok; ++q) {
        const uint32_t* f = reinterpret_cast<const uint32_t*>(mine + lay.flag_off_bytes(par, q, row));
        while (ld_acquire_sys_u32(f) != epoch) {
          if (globaltimer_ns() - t0 > timeout_ns) { ok = 0; break; }
        }
      }
      if (!ok && err) atomicOr(err, VECINFER_FLAG_P2P_TIMEOUT);
      s_ok = ok;
    }
    __syncthreads();
    // 3. merge in rank order (merge_lse_kernel's arithmetic), reading past L1 (peer-written data)
    const float* win = static_cast<const float*>(windows[rank]);
    float M = -INFINITY;
    for (int s = 0; s < P; ++s) M = fmaxf(M, __ldcg(win + lay.data_off(par, s, row) + D));
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      float wsum = 0.f, osum = 0.f;
      if (M != -INFINITY) {
        for (int s = 0; s < P; ++s) {
          const float* src = win + lay.data_off(par, s, row);
          const float f = __expf(__ldcg(src + D) - M);
          wsum += f;
          osum += f * __ldcg(src + d);
        }
      }
      const bool empty = !(wsum > 0.f) || !s_ok;
      const float v = empty ? 0.f : osum / wsum;
      if (o_f32) static_cast<float*>(o)[row * D + d] = v;
      else static_cast<__nv_bfloat16*>(o)[row * D + d] = __float2bfloat16_rn(v);
      if (d == 0 && lse) lse[row] = empty ? -INFINITY : M + __logf(wsum);
    }
    __syncthreads();   // s_ok is rewritten for the next row
  }
  if (threadIdx.x == 0) {   // the last CTA of the launch records the epoch it used (automatic mode)
    __threadfence();
    if (atomicAdd(hdr + 1, 1u) == gridDim.x - 1) {
      hdr[1] = 0u;
      hdr[0] = epoch;
    }
  }
}

}  // namespace
}  // namespace vecinfer

extern "C" size_t vecinfer_p2p_window_bytes(int32_t P, int64_t rows, int32_t D) {
  if (P <= 0 || rows <= 0 || D <= 0) return 0;
  P2PLayout lay{rows, P, D};
  return static_cast<size_t>(lay.bytes());
}

extern "C" vecinfer_status_t vecinfer_p2p_window_create(size_t bytes, void** window, void* ipc_handle) {
  if (!window || !ipc_handle || bytes == 0) return fail(VECINFER_ERR_INVALID_ARG, "p2p_window_create: bad argument");
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return check_launch("p2p_window_create cudaMalloc");
  if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p);
    return check_launch("p2p_window_create memset");
  }
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaFree(p);
    return check_launch("p2p_window_create cudaIpcGetMemHandle");
  }
  memcpy(ipc_handle, &h, sizeof(h));
  *window = p;
  return VECINFER_OK;
}

extern "C" vecinfer_status_t vecinfer_p2p_window_open(const void* ipc_handle, void** window) {
  if (!window || !ipc_handle) return fail(VECINFER_ERR_INVALID_ARG, "p2p_window_open: NULL pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return check_launch("p2p_window_open cudaIpcOpenMemHandle");
  *window = p;
  return VECINFER_OK;
}

extern "C" vecinfer_status_t vecinfer_p2p_window_close(void* window) {
  if (!window) return fail(VECINFER_ERR_INVALID_ARG, "p2p_window_close: NULL pointer");
  if (cudaIpcCloseMemHandle(window) != cudaSuccess) return check_launch("p2p_window_close");
  return VECINFER_OK;
}

extern "C" vecinfer_status_t vecinfer_p2p_window_destroy(void* window) {
  if (!window) return fail(VECINFER_ERR_INVALID_ARG, "p2p_window_destroy: NULL pointer");
  if (cudaFree(window) != cudaSuccess) return check_launch("p2p_window_destroy");
  return VECINFER_OK;
}

extern "C" vecinfer_status_t vecinfer_merge_lse_p2p(const float* o_local, const float* lse_local, void* const* windows,
                                                    int32_t P, int32_t rank, int32_t B, int32_t H_q, int32_t D,
                                                    uint32_t epoch, void* o, vecinfer_dtype_t o_dtype, float* lse,
                                                    uint32_t* err_flags, vecinfer_stream_t stream) {
  if (!o_local || !lse_local || !windows || !o) return fail(VECINFER_ERR_INVALID_ARG, "merge_lse_p2p: NULL pointer");
  if (o_dtype != VECINFER_BF16 && o_dtype != VECINFER_F32) return fail(VECINFER_ERR_INVALID_ARG, "merge_lse_p2p: bad o_dtype");
  if (P <= 0 || B <= 0 || H_q <= 0 || D <= 0 || D > 1024) return fail(VECINFER_ERR_SHAPE, "merge_lse_p2p: bad size");
  if (rank < 0 || rank >= P) return fail(VECINFER_ERR_SHAPE, "merge_lse_p2p: rank %d outside [0, %d)", rank, P);
  const int64_t rows = static_cast<int64_t>(B) * H_q;
  if (rows > 2147483647) return fail(VECINFER_ERR_SHAPE, "merge_lse_p2p: too many rows");
  const P2PLayout lay{rows, P, D};
  const int threads = D >= 128 ? 128 : ((D + 31) / 32) * 32;
  const unsigned long long timeout_ns = 5000000000ull;   // 5 s: a missing peer flags instead of hanging
  // persistent grid capped at the co-resident CTA count (every CTA spin-waits on peer flags)
  static int cached_threads = 0, resident = 0;   // benign race: idempotent
  if (cached_threads != threads) {
    cached_threads = threads;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge_lse_p2p_kernel, threads, 0) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    resident = per_sm * device_sm_count();
  }
  const unsigned grid = static_cast<unsigned>(rows < resident ? rows : resident);
  merge_lse_p2p_kernel<<<grid, threads, 0, as_stream(stream)>>>(
      o_local, lse_local, windows, lay, rank, epoch, o, o_dtype == VECINFER_F32, lse, err_flags, timeout_ns);
  return check_launch("merge_lse_p2p_kernel");
}
