// N5: log-sum-exp merge of P normalised partials (cross-GPU shards, residual window).
//   L = logsumexp_s L_s;  o = sum_s exp(L_s - L) o_s  in the fixed order s = 0..P-1
// (the online-softmax recurrence of P:745-757 applied to whole partials).
// One CTA per (b, h_q) row, one thread per dim; tiny and latency-bound.
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
