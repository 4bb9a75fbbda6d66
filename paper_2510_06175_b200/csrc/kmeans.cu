// Codebook k-means on the GPU (NEXT-3): one Lloyd iteration per call, the
// codebook-construction step of the method ("C_k ... via K-means", "K-means ...
// maximum number of iterations set to 30"; empty-cluster re-seeding SPEC S:184).  Offline, not on
// the decode path; written so fitting a b4d4 codebook (65 536 centroids) is a GPU job.
//
//   1. assign (kmeans_assign_kernel): a_i = argmin_j dist(x_i, C_j) with the encoder's pinned fp32
//      distance (Eq. 2 / reading R9: e_t = x_t - c_t, ((e_0^2 + e_1^2) + e_2^2) + ..., every op RN,
//      no FMA), strict < scan in index order -> lowest index on ties.  Centroids are staged in
//      shared memory in 32 KiB chunks and read as broadcasts; every thread keeps 8 points (2 for
//      small n) in registers.  The same thread then adds its points into the cluster sums and counts
//      and its best distance into the objective (global atomics).  Sums and objective are exact
//      int64 fixed-point sums (scale 2^e chosen from max|x|, max|C| and n by kmeans_bound_kernel so
//      no sum can overflow): integer addition is associative, so the result does not depend on the
//      order the atomics land in -- the step is bitwise reproducible run to run.
//   2. finalize (kmeans_finalize_kernel): C'_j = RN32((sum_j / 2^e) / n_j) (fp64) for n_j > 0.
//   3. reseed (kmeans_reseed_kernel, one CTA): the empty clusters, in increasing j, take the points
//      of largest best_i (ties: lowest i), one each -- E rounds of a block-wide max over the key
//      (best_bits << 32 | ~i) restricted to keys below the previous pick.  No-op when E = 0.
// Parity: oracle/vecinfer_oracle.py kmeans_lloyd_step (assignments and best bit-exact, counts
// exact, C' within one fp32 ulp: the per-point fixed-point rounding is <= 2^-(e+1), far below an
// fp32 ulp of the mean at the data scales used, but not zero).
#include "common.cuh"

namespace vecinfer {
namespace {

constexpr int kKmThreads = 256;
constexpr int kKmChunkBytes = 32768;      // centroid chunk staged in shared memory

template <int D>
__device__ __forceinline__ float pinned_dist(const float (&x)[D], const float* c) {
  float acc = 0.f;
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const float e = __fsub_rn(x[t], c[t]);
    const float e2 = __fmul_rn(e, e);
    acc = t == 0 ? e2 : __fadd_rn(acc, e2);
  }
  return acc;
}

// max |x| over the points and max |c| over the centroids as fp32 bits (|v| >= 0: unsigned order
// of the bits is the float order), for the fixed-point scales of the sums and the objective
__global__ void kmeans_bound_kernel(const float* __restrict__ X, int64_t nx, const float* __restrict__ C, int64_t nc,
                                    uint32_t* __restrict__ bound) {
  uint32_t mx = 0u, mc = 0u;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nx;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mx = max(mx, __float_as_uint(fabsf(X[e])));
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nc;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mc = max(mc, __float_as_uint(fabsf(C[e])));
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(bound, mx);
    atomicMax(bound + 1, mc);
  }
}

// Power-of-two scales 2^e_sum (cluster sums) and 2^e_obj (objective) such that n addends of
// magnitude <= bound stay below 2^62 in int64: e = 61 - ceil(log2 n) - ceil(log2 bound), clamped.
struct KmScale {
  double s_sum, s_obj;
};
__device__ __forceinline__ int km_exp_for(double bound, int64_t n) {
  int eb = 0, en = 0;
  frexp(bound > 0.0 ? bound : 1.0, &eb);               // bound < 2^eb
  frexp(static_cast<double>(n), &en);                  // n < 2^en
  int e = 61 - en - eb;
  return e > 200 ? 200 : (e < -200 ? -200 : e);
}
__device__ __forceinline__ KmScale km_scale(const uint32_t* bound, int64_t n, int D) {
  const double xm = static_cast<double>(__uint_as_float(bound[0]));
  const double cm = static_cast<double>(__uint_as_float(bound[1]));
  KmScale sc;
  sc.s_sum = ldexp(1.0, km_exp_for(xm, n));
  sc.s_obj = ldexp(1.0, km_exp_for(static_cast<double>(D) * (xm + cm) * (xm + cm) * 1.0001, n));
  return sc;
}
__device__ __forceinline__ long long to_fixed(double v, double scale) { return __double2ll_rn(v * scale); }

template <int D, int kKmPts>   // kKmPts: points per thread (8, or 2 for small n: more CTAs)
__global__ void __launch_bounds__(kKmThreads) kmeans_assign_kernel(const float* __restrict__ X, int64_t n,
                                                                    const float* __restrict__ C, int k,
                                                                    int32_t* __restrict__ assign,
                                                                    float* __restrict__ best,
                                                                    unsigned long long* __restrict__ sums,
                                                                    int32_t* __restrict__ counts,
                                                                    unsigned long long* __restrict__ obj_fx,
                                                                    const uint32_t* __restrict__ bound) {
  constexpr int kChunk = kKmChunkBytes / (4 * D);
  __shared__ __align__(16) float sc[kChunk * D];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kKmThreads * kKmPts;
  float x[kKmPts][D];
  float bd[kKmPts];
  int bi[kKmPts];
#pragma unroll
  for (int p = 0; p < kKmPts; ++p) {
    const int64_t i = base + p * kKmThreads + threadIdx.x;   // coalesced rows
#pragma unroll
    for (int t = 0; t < D; ++t) x[p][t] = i < n ? X[i * D + t] : 0.f;
    bd[p] = __int_as_float(0x7f800000);
    bi[p] = 0;
  }
  for (int c0 = 0; c0 < k; c0 += kChunk) {
    const int nc = min(kChunk, k - c0);
    __syncthreads();
    if constexpr (D == 4) {
      // d = 4: centroid pairs in the FADD2 / FMUL2 layout (pinned_dist4_x2: the same per-element
      // RN ops, two centroids per instruction); an odd last centroid is paired with itself
      uint4* sp = reinterpret_cast<uint4*>(sc);
      for (int q = threadIdx.x; q < (nc + 1) / 2; q += kKmThreads) {
        const float* a = C + static_cast<int64_t>(c0 + 2 * q) * 4;
        const float* b = (2 * q + 1 < nc) ? a + 4 : a;
        sp[2 * q] = make_uint4(__float_as_uint(a[0]), __float_as_uint(b[0]), __float_as_uint(a[1]), __float_as_uint(b[1]));
        sp[2 * q + 1] = make_uint4(__float_as_uint(a[2]), __float_as_uint(b[2]), __float_as_uint(a[3]), __float_as_uint(b[3]));
      }
      __syncthreads();
      for (int q = 0; q < nc / 2; ++q) {
        const uint4 p01 = sp[2 * q], p23 = sp[2 * q + 1];
#pragma unroll
        for (int p = 0; p < kKmPts; ++p) {
          const float2 d = pinned_dist4_x2(x[p][0], x[p][1], x[p][2], x[p][3], p01, p23);
          if (d.x < bd[p]) { bd[p] = d.x; bi[p] = c0 + 2 * q; }
          if (d.y < bd[p]) { bd[p] = d.y; bi[p] = c0 + 2 * q + 1; }
        }
      }
      if (nc & 1) {
        const int q = nc / 2;
        const uint4 p01 = sp[2 * q], p23 = sp[2 * q + 1];
#pragma unroll
        for (int p = 0; p < kKmPts; ++p) {
          const float2 d = pinned_dist4_x2(x[p][0], x[p][1], x[p][2], x[p][3], p01, p23);
          if (d.x < bd[p]) { bd[p] = d.x; bi[p] = c0 + 2 * q; }
        }
      }
    } else {
      for (int e = threadIdx.x; e < nc * D; e += kKmThreads) sc[e] = C[static_cast<int64_t>(c0) * D + e];
      __syncthreads();
      for (int j = 0; j < nc; ++j) {
        float cj[D];
#pragma unroll
        for (int t = 0; t < D; ++t) cj[t] = sc[j * D + t];
#pragma unroll
        for (int p = 0; p < kKmPts; ++p) {
          const float dd = pinned_dist<D>(x[p], cj);
          if (dd < bd[p]) { bd[p] = dd; bi[p] = c0 + j; }
        }
      }
    }
  }
  const KmScale scl = km_scale(bound, n, D);
  long long obj = 0;
#pragma unroll
  for (int p = 0; p < kKmPts; ++p) {
    const int64_t i = base + p * kKmThreads + threadIdx.x;
    if (i >= n) continue;
    assign[i] = bi[p];
    best[i] = bd[p];
    obj += to_fixed(static_cast<double>(bd[p]), scl.s_obj);
    atomicAdd(&counts[bi[p]], 1);
#pragma unroll
    for (int t = 0; t < D; ++t)   // two's complement wrap-around add == exact signed int64 add
      atomicAdd(&sums[static_cast<int64_t>(bi[p]) * D + t],
                static_cast<unsigned long long>(to_fixed(static_cast<double>(x[p][t]), scl.s_sum)));
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) obj += __shfl_xor_sync(0xffffffffu, obj, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(obj_fx, static_cast<unsigned long long>(obj));
}

template <int D>
__global__ void kmeans_finalize_kernel(const float* __restrict__ C, int k, int64_t n,
                                       const unsigned long long* __restrict__ sums,
                                       const int32_t* __restrict__ counts, float* __restrict__ Cn,
                                       const uint32_t* __restrict__ bound, const unsigned long long* __restrict__ obj_fx,
                                       double* __restrict__ objective) {
  const KmScale scl = km_scale(bound, n, D);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) *objective = static_cast<double>(static_cast<long long>(*obj_fx)) / scl.s_obj;
  if (j >= k) return;
  const int cnt = counts[j];
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const int64_t e = static_cast<int64_t>(j) * D + t;
    const double sum = static_cast<double>(static_cast<long long>(sums[e])) / scl.s_sum;   // /2^e: exact
    Cn[e] = cnt > 0 ? __double2float_rn(__ddiv_rn(sum, static_cast<double>(cnt))) : C[e];
  }
}

// one CTA of 1024 threads
template <int D>
__global__ void __launch_bounds__(1024) kmeans_reseed_kernel(const float* __restrict__ X, int64_t n,
                                                             const float* __restrict__ best, int k,
                                                             const int32_t* __restrict__ counts,
                                                             int32_t* __restrict__ empty_list,
                                                             float* __restrict__ Cn) {
  __shared__ int s_warp[32];
  __shared__ int s_total;
  __shared__ unsigned long long s_red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 1. ordered list of the empty clusters (block-wide exclusive scan per 1024-cluster chunk)
  int E = 0;
  for (int c0 = 0; c0 < k; c0 += 1024) {
    const int c = c0 + tid;
    const bool emp = c < k && counts[c] == 0;
    const unsigned m = __ballot_sync(0xffffffffu, emp);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int w = 0; w < 32; ++w) { const int v = s_warp[w]; s_warp[w] = run; run += v; }
      s_total = run;
    }
    __syncthreads();
    if (emp) empty_list[E + s_warp[warp] + __popc(m & ((1u << lane) - 1u))] = c;
    E += s_total;
    __syncthreads();
  }
  if (E == 0) return;
  __threadfence_block();
  __syncthreads();
  // 2. E rounds: the point of largest key = (best bits << 32 | ~i) below the previous pick
  unsigned long long prev = ~0ull;
  for (int r = 0; r < E; ++r) {
    unsigned long long mx = 0ull;
    bool any = false;
    for (int64_t i = tid; i < n; i += 1024) {
      const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(best[i])) << 32) |
                                     (0xFFFFFFFFull - static_cast<unsigned long long>(i));
      if (key < prev && (!any || key > mx)) { mx = key; any = true; }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, off);
      mx = o > mx ? o : mx;
    }
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    if (warp == 0) {
      unsigned long long v = s_red[lane];
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o > v ? o : v;
      }
      if (lane == 0) s_red[0] = v;
    }
    __syncthreads();
    prev = s_red[0];
    __syncthreads();
    const int64_t pick = static_cast<int64_t>(0xFFFFFFFFull - (prev & 0xFFFFFFFFull));
    if (tid < D) Cn[static_cast<int64_t>(empty_list[r]) * D + tid] = X[pick * D + tid];
  }
}

struct KmWs {
  size_t sums, counts, misc, empty, total;   // misc: u32 bound[2] (max|x|, max|c|) + u64 objective sum
};
KmWs km_ws(int32_t k, int32_t d) {
  KmWs w;
  w.sums = 0;
  w.counts = (static_cast<size_t>(k) * d * sizeof(unsigned long long) + 255) & ~size_t(255);
  w.misc = w.counts + ((static_cast<size_t>(k) * sizeof(int32_t) + 255) & ~size_t(255));
  w.empty = w.misc + 256;
  w.total = w.empty + static_cast<size_t>(k) * sizeof(int32_t);
  return w;
}

template <int D>
cudaError_t launch_kmeans(const float* X, int64_t n, const float* C, int k, float* Cn, int32_t* assign, float* best,
                          double* obj, unsigned char* ws, cudaStream_t st) {
  const KmWs w = km_ws(k, D);
  unsigned long long* sums = reinterpret_cast<unsigned long long*>(ws + w.sums);
  int32_t* counts = reinterpret_cast<int32_t*>(ws + w.counts);
  uint32_t* bound = reinterpret_cast<uint32_t*>(ws + w.misc);
  unsigned long long* obj_fx = reinterpret_cast<unsigned long long*>(ws + w.misc + 8);
  int32_t* empty = reinterpret_cast<int32_t*>(ws + w.empty);
  if (cudaMemsetAsync(ws, 0, w.empty, st) != cudaSuccess) return cudaGetLastError();
  kmeans_bound_kernel<<<2 * device_sm_count(), 256, 0, st>>>(X, n * D, C, static_cast<int64_t>(k) * D, bound);
  // 8 points per thread amortise the shared-memory centroid stream; below ~2 CTAs per SM at 8,
  // 2 points per thread keep every SM busy
  const bool big = n >= static_cast<int64_t>(device_sm_count()) * kKmThreads * 8 * 2;
  const int64_t per = static_cast<int64_t>(kKmThreads) * (big ? 8 : 2);
  const unsigned g = static_cast<unsigned>((n + per - 1) / per);
  if (big) kmeans_assign_kernel<D, 8><<<g, kKmThreads, 0, st>>>(X, n, C, k, assign, best, sums, counts, obj_fx, bound);
  else kmeans_assign_kernel<D, 2><<<g, kKmThreads, 0, st>>>(X, n, C, k, assign, best, sums, counts, obj_fx, bound);
  kmeans_finalize_kernel<D><<<(k + 255) / 256, 256, 0, st>>>(C, k, n, sums, counts, Cn, bound, obj_fx, obj);
  kmeans_reseed_kernel<D><<<1, 1024, 0, st>>>(X, n, best, k, counts, empty, Cn);
  return cudaPeekAtLastError();
}

}  // namespace
}  // namespace vecinfer

using namespace vecinfer;

extern "C" size_t vecinfer_kmeans_workspace_bytes(int32_t k, int32_t d) {
  if (k <= 0 || d <= 0) return 0;
  return km_ws(k, d).total;
}

extern "C" vecinfer_status_t vecinfer_kmeans_step(const float* X, int64_t n, int32_t d, const float* C, int32_t k,
                                                  float* C_new, int32_t* assign, float* best, double* objective,
                                                  void* workspace, size_t workspace_bytes, vecinfer_stream_t stream) {
  if (!X || !C || !C_new || !assign || !best || !objective)
    return fail(VECINFER_ERR_INVALID_ARG, "kmeans_step: NULL pointer");
  if (d != 2 && d != 4 && d != 8) return fail(VECINFER_ERR_UNSUPPORTED, "kmeans_step: sub-vector dim d must be 2, 4 or 8");
  if (k <= 0 || k > 65536) return fail(VECINFER_ERR_SHAPE, "kmeans_step: need 0 < k <= 65536");
  if (n <= 0) return fail(VECINFER_ERR_EMPTY, "kmeans_step: no points");
  if (n < k) return fail(VECINFER_ERR_SHAPE, "kmeans_step: fewer points (%lld) than clusters (%d)", (long long)n, k);
  if (n >= (int64_t(1) << 32) - 1) return fail(VECINFER_ERR_SHAPE, "kmeans_step: n must be < 2^32 - 1");
  if (!aligned(X, 4) || !aligned(C, 4) || !aligned(C_new, 4) || !aligned(objective, 8))
    return fail(VECINFER_ERR_INVALID_ARG, "kmeans_step: misaligned pointer");
  const size_t need = vecinfer_kmeans_workspace_bytes(k, d);
  if (!workspace || workspace_bytes < need)
    return fail(VECINFER_ERR_WORKSPACE, "kmeans_step: workspace needs %zu bytes", need);
  if (!aligned(workspace, 256)) return fail(VECINFER_ERR_INVALID_ARG, "kmeans_step: workspace must be 256-byte aligned");
  cudaStream_t st = as_stream(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  if (d == 2) launch_kmeans<2>(X, n, C, k, C_new, assign, best, objective, ws, st);
  else if (d == 4) launch_kmeans<4>(X, n, C, k, C_new, assign, best, objective, ws, st);
  else launch_kmeans<8>(X, n, C, k, C_new, assign, best, objective, ws, st);
  return check_launch("kmeans_step");
}
