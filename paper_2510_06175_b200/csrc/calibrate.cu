// N1: smoothing-factor calibration, Eq. 4: lambda_c = sqrt(max_n |K[n,h,c]|).
//
// HBM-bound reduction over the calibration keys (256 x 512 tokens x 8 heads x 128 ch bf16 =
// 256 MiB at the paper's protocol).  Each thread owns 8 consecutive channels (one 16-B
// load per token row), 8 token lanes per block; per-channel maxima are merged with atomicMax
// on the fp32 bit pattern (valid: |x| >= 0, so uint order == float order) and the last block
// finalises lambda = max(RN32(sqrt(amax)), eps), inv_lambda = RN32(1/lambda).
#include "common.cuh"

namespace vecinfer {

namespace {

constexpr int kTokLanes = 8;     // threadIdx.y
constexpr int kColThreads = 32;  // threadIdx.x, 8 channels each -> 256 channels per block column

template <bool kVec>
__global__ void __launch_bounds__(kColThreads* kTokLanes)
    calibrate_kernel(const uint16_t* __restrict__ k, int64_t n_tok, int H, int D, int64_t st_tok,
                     int64_t st_head, uint32_t* __restrict__ amax_bits, uint32_t* __restrict__ counter,
                     float eps, float* __restrict__ lam, float* __restrict__ inv) {
  const int HD = H * D;
  const int cg = (blockIdx.y * kColThreads + threadIdx.x) * 8;  // first global channel of thread
  const bool active = cg < HD;
  const int h = active ? cg / D : 0;
  const int c = active ? cg % D : 0;
  float m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = 0.f;
  if (active) {
    const uint16_t* base = k + h * st_head + c;
    const int64_t step = static_cast<int64_t>(gridDim.x) * kTokLanes;
    int64_t t = static_cast<int64_t>(blockIdx.x) * kTokLanes + threadIdx.y;
    // 4 rows in flight per thread
    for (; t + 3 * step < n_tok; t += 4 * step) {
      uint32_t w[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint16_t* p = base + (t + u * step) * st_tok;
        if (kVec) {
          uint4 v = ldg_nc_u128(p);
          w[u][0] = v.x; w[u][1] = v.y; w[u][2] = v.z; w[u][3] = v.w;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) w[u][i] = static_cast<uint32_t>(p[2 * i]) | (static_cast<uint32_t>(p[2 * i + 1]) << 16);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          m[2 * i] = fmaxf(m[2 * i], fabsf(__uint_as_float(w[u][i] << 16)));
          m[2 * i + 1] = fmaxf(m[2 * i + 1], fabsf(__uint_as_float(w[u][i] & 0xFFFF0000u)));
        }
    }
    for (; t < n_tok; t += step) {
      const uint16_t* p = base + t * st_tok;
#pragma unroll
      for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], fabsf(bf16_bits_to_float(p[i])));
    }
  }
  // reduce the 8 token lanes through shared memory, then one atomicMax per channel
  __shared__ float red[kTokLanes][kColThreads * 8 + 1];
#pragma unroll
  for (int i = 0; i < 8; ++i) red[threadIdx.y][threadIdx.x * 8 + i] = m[i];
  __syncthreads();
  const int tid = threadIdx.y * kColThreads + threadIdx.x;  // 0..255 -> one channel each
  {
    float v = 0.f;
#pragma unroll
    for (int y = 0; y < kTokLanes; ++y) v = fmaxf(v, red[y][tid]);
    const int ch = blockIdx.y * kColThreads * 8 + tid;
    if (ch < HD) atomicMax(&amax_bits[ch], __float_as_uint(v));
  }
  // last block finalises
  __threadfence();
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    const uint32_t total = gridDim.x * gridDim.y;
    last = (atomicAdd(counter, 1u) == total - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int ch = tid; ch < HD; ch += blockDim.x * blockDim.y) {
    const float a = __uint_as_float(atomicAdd(&amax_bits[ch], 0u));
    float l = __fsqrt_rn(a);
    l = fmaxf(l, eps);
    lam[ch] = l;
    inv[ch] = __fdiv_rn(1.0f, l);
  }
}

}  // namespace
}  // namespace vecinfer

using namespace vecinfer;

extern "C" size_t vecinfer_calibrate_workspace_bytes(int32_t n_kv_heads, int32_t head_dim) {
  if (n_kv_heads <= 0 || head_dim <= 0) return 0;
  return (static_cast<size_t>(n_kv_heads) * head_dim + 32) * sizeof(uint32_t);
}

extern "C" vecinfer_status_t vecinfer_calibrate_smooth(const void* k_cal_bf16, int64_t n_tokens,
                                                       int32_t n_kv_heads, int32_t head_dim,
                                                       int64_t stride_tok, int64_t stride_head,
                                                       float eps_floor, float* lambda_out,
                                                       float* inv_lambda_out, void* workspace,
                                                       size_t workspace_bytes,
                                                       vecinfer_stream_t stream) {
  if (!k_cal_bf16 || !lambda_out || !inv_lambda_out)
    return fail(VECINFER_ERR_INVALID_ARG, "calibrate_smooth: NULL pointer");
  if (!(eps_floor > 0.f)) return fail(VECINFER_ERR_INVALID_ARG, "calibrate_smooth: eps_floor must be > 0");
  if (n_kv_heads <= 0 || head_dim <= 0 || head_dim % 8 != 0)
    return fail(VECINFER_ERR_SHAPE, "calibrate_smooth: need n_kv_heads > 0 and head_dim a positive multiple of 8");
  if (n_tokens < 0) return fail(VECINFER_ERR_SHAPE, "calibrate_smooth: n_tokens < 0");
  if (n_tokens == 0) return fail(VECINFER_ERR_EMPTY, "calibrate_smooth: empty calibration set (Eq. 4 undefined)");
  if (stride_tok <= 0 || (n_kv_heads > 1 && stride_head < head_dim))
    return fail(VECINFER_ERR_INVALID_ARG, "calibrate_smooth: bad strides");
  const size_t need = vecinfer_calibrate_workspace_bytes(n_kv_heads, head_dim);
  if (!workspace || workspace_bytes < need)
    return fail(VECINFER_ERR_WORKSPACE, "calibrate_smooth: workspace needs %zu bytes", need);
  if (!aligned(workspace, 4)) return fail(VECINFER_ERR_INVALID_ARG, "calibrate_smooth: workspace misaligned");
  cudaStream_t st = as_stream(stream);
  const int HD = n_kv_heads * head_dim;
  uint32_t* amax = static_cast<uint32_t*>(workspace);
  uint32_t* counter = amax + HD;
  if (cudaMemsetAsync(workspace, 0, need, st) != cudaSuccess) return check_launch("calibrate_smooth memset");
  const bool vec = aligned(k_cal_bf16, 16) && (stride_tok % 8 == 0) && (stride_head % 8 == 0);
  const int gy = (HD / 8 + kColThreads - 1) / kColThreads;
  const int64_t rows_per_block = 64;  // >= 8 iterations of 8 token lanes per block
  int64_t gx64 = (n_tokens + rows_per_block - 1) / rows_per_block;
  const int64_t cap = static_cast<int64_t>(device_sm_count()) * 8 / gy + 1;
  if (gx64 > cap) gx64 = cap;
  if (gx64 < 1) gx64 = 1;
  dim3 grid(static_cast<unsigned>(gx64), gy), block(kColThreads, kTokLanes);
  const uint16_t* k = static_cast<const uint16_t*>(k_cal_bf16);
  if (vec)
    calibrate_kernel<true><<<grid, block, 0, st>>>(k, n_tokens, n_kv_heads, head_dim, stride_tok, stride_head,
                                                   amax, counter, eps_floor, lambda_out, inv_lambda_out);
  else
    calibrate_kernel<false><<<grid, block, 0, st>>>(k, n_tokens, n_kv_heads, head_dim, stride_tok, stride_head,
                                                    amax, counter, eps_floor, lambda_out, inv_lambda_out);
  return check_launch("calibrate_kernel");
}
