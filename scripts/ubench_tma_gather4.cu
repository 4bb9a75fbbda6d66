// Microbenchmark: random 16-byte row gathers from a 512 KiB / 1 MiB table (a b4d4 / d8b16 codebook
// viewed as rows of 16 B), L1/L2 path (LDG.128 per lane) vs the TMA engine (cp.async.bulk.tensor
// tile::gather4: four rows per request into shared memory, mbarrier completion).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_g4 scripts/ubench_tma_gather4.cu -lcuda
// Prints rows per clock per SM for both paths (the attention needs 64 centroid rows per token-head).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kWarps = 8;
constexpr int kRounds = 256;   // per warp: 128 rows per round

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(kWarps * 32) gather_ldg(const uint4* table, const uint32_t* rows, int nrows_mask,
                                                           uint32_t* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp;
  uint32_t acc = 0;
  for (int it = 0; it < kRounds; ++it) {
    const uint32_t* r = rows + ((static_cast<uint64_t>(gw) * kRounds + it) * 128 & 0xFFFFFF);
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      const uint4* p = table + (r[32 * q + lane] & nrows_mask);
      asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(p));
      v[q] = w;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += v[q].x ^ v[q].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

constexpr int kTW = 4;   // TMA kernel warps per CTA (8 KiB of stages each)
__global__ void __launch_bounds__(kTW * 32) gather_tma(const __grid_constant__ CUtensorMap tmap, const uint32_t* rows,
                                                           int nrows_mask, uint32_t* out) {
  // per warp: 2 stages x 32 requests; a request's 4 rows x 16 B land at a 128-byte aligned slot (TMA)
  __shared__ __align__(128) uint4 stage[kTW][2][32][8];
  __shared__ __align__(8) uint64_t bar[kTW][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kTW + warp;
  if (lane < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[warp][lane])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int it) {
    const int st = it & 1;
    const uint32_t* r = rows + ((static_cast<uint64_t>(gw) * kRounds + it) * 128 & 0xFFFFFF);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[warp][st])), "r"(128 * 16) : "memory");
    __syncwarp();
    const int4 rr = make_int4(r[4 * lane] & nrows_mask, r[4 * lane + 1] & nrows_mask, r[4 * lane + 2] & nrows_mask,
                              r[4 * lane + 3] & nrows_mask);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        :: "r"(smem_u32(&stage[warp][st][lane][0])), "l"(&tmap), "r"(0), "r"(rr.x), "r"(rr.y), "r"(rr.z), "r"(rr.w),
           "r"(smem_u32(&bar[warp][st]))
        : "memory");
  };
  uint32_t acc = 0;
  issue(0);
  for (int it = 0; it < kRounds; ++it) {
    if (it + 1 < kRounds) issue(it + 1);
    const int st = it & 1;
    const uint32_t par = (it >> 1) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar[warp][st])), "r"(par) : "memory");
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += stage[warp][st][(32 * q + lane) >> 2][(32 * q + lane) & 3].x ^ stage[warp][st][(32 * q + lane) >> 2][(32 * q + lane) & 3].w;
    __syncwarp();
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  cudaSetDevice(0);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int nrows_list[2] = {32768, 65536};   // 512 KiB (b4d4 book as 16-byte rows), 1 MiB
  uint4* table;
  cudaMalloc(&table, 65536 * 16);
  cudaMemset(table, 1, 65536 * 16);
  const size_t nr = 1 << 24;
  std::vector<uint32_t> h(nr);
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < nr; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = static_cast<uint32_t>(s); }
  uint32_t *rows, *out;
  cudaMalloc(&rows, nr * 4);
  cudaMalloc(&out, 16);
  cudaMemcpy(rows, h.data(), nr * 4, cudaMemcpyHostToDevice);
  for (int t = 0; t < 2; ++t) {
    const int nrows = nrows_list[t];
    CUtensorMap tmap;
    cuuint64_t gdim[2] = {8, static_cast<cuuint64_t>(nrows)};
    cuuint64_t gstr[1] = {16};
    cuuint32_t box[2] = {8, 1};
    cuuint32_t est[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, table, gdim, gstr, box, est,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("tensor map encode failed: %d\n", static_cast<int>(cr)); return 1; }
    for (int ctas_per_sm : {1, 2, 4}) {
      const int grid = sms * ctas_per_sm;
      const double rows_total = static_cast<double>(grid) * kWarps * kRounds * 128;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int path = 0; path < 2; ++path) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (path == 0) gather_ldg<<<grid, kWarps * 32>>>(table, rows, nrows - 1, out);
          else gather_tma<<<grid * (kWarps / kTW), kTW * 32>>>(tmap, rows, nrows - 1, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaError_t err = cudaGetLastError();
          if (err != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(err)); return 1; }
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep == 1)
            printf("table %4d KiB  %s  CTAs/SM %d (%2d warps/SM): %7.3f ms  %.2f rows/clk/SM (%.0f GB/s of 16-B rows)\n",
                   nrows * 16 / 1024, path ? "TMA gather4" : "LDG.128    ", ctas_per_sm, ctas_per_sm * kWarps, ms,
                   rows_total / (ms * 1e-3) / (clk * 1e3) / sms, rows_total * 16 / (ms * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
