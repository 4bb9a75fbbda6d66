// Microbenchmark for the b4d4 design question (DESIGN.md §9 item 2): random 8-byte gathers from a
// 512 KiB table (65536 x 8 B, one b4d4 codebook stream) served
//   (a) from global memory through L1/L2 (the current b4d4 path),
//   (b) from distributed shared memory: the table split over an 8-CTA cluster, 64 KiB per CTA,
//       gathered with ld.shared::cluster at mapa(addr, code >> 13),
//   (c) from local shared memory (64 KiB slice, same random pattern; the best case of (b)).
// Every thread runs ITERS dependent-free gathers (4 independent streams) from an LCG; reports
// gathers/s and bytes/clk/SM at the measured SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_dsmem r01_ubench_dsmem.cu && ./ubench_dsmem
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int kThreads = 512, kIters = 4096, kEntriesPerCta = 8192;

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s >> 16; }

__global__ void __launch_bounds__(kThreads) gather_global(const uint2* __restrict__ tab, uint32_t* out) {
  uint32_t s0 = blockIdx.x * kThreads + threadIdx.x, s1 = s0 ^ 0x9e3779b9u, s2 = s0 * 7u + 3u, s3 = ~s0;
  uint32_t acc = 0;
  for (int i = 0; i < kIters; i += 4) {
    const uint2 a = __ldg(tab + lcg(s0)), b = __ldg(tab + lcg(s1)), c = __ldg(tab + lcg(s2)), d = __ldg(tab + lcg(s3));
    acc ^= a.x ^ b.y ^ c.x ^ d.y;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(kThreads) gather_dsmem(const uint2* __restrict__ tab, uint32_t* out, int local_only) {
  extern __shared__ uint2 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  for (int j = threadIdx.x; j < kEntriesPerCta; j += kThreads) sm[j] = tab[rank * kEntriesPerCta + j];
  cl.sync();
  uint32_t s0 = blockIdx.x * kThreads + threadIdx.x, s1 = s0 ^ 0x9e3779b9u, s2 = s0 * 7u + 3u, s3 = ~s0;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  uint32_t acc = 0;
  auto g = [&](uint32_t code) -> uint32_t {
    const uint32_t r = local_only ? rank : (code >> 13);
    const uint32_t addr = base + (code & (kEntriesPerCta - 1)) * 8;
    uint32_t ra, x, y;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(r));
    asm volatile("ld.shared::cluster.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(ra));
    return x ^ y;
  };
  for (int i = 0; i < kIters; i += 4) acc ^= g(lcg(s0)) ^ g(lcg(s1)) ^ g(lcg(s2)) ^ g(lcg(s3));
  cl.sync();
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint2* tab;
  uint32_t* out;
  cudaMalloc(&tab, 65536 * 8);
  cudaMalloc(&out, 4);
  cudaMemset(tab, 1, 65536 * 8);
  cudaFuncSetAttribute(gather_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, kEntriesPerCta * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grids[] = {sms, 2 * sms / 8 * 8};
  for (int gi = 0; gi < 2; ++gi) {
    const int grid = grids[gi] / 8 * 8;
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) gather_global<<<grid, kThreads>>>(tab, out);
        else gather_dsmem<<<grid, kThreads, kEntriesPerCta * 8>>>(tab, out, mode == 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gathers = double(grid) * kThreads * kIters;
      const double per_sm_clk = gathers * 8.0 / (ms * 1e-3) / sms / (clk_khz * 1e3);
      printf("%-28s grid %4d: %8.3f ms  %7.1f G gathers/s  %6.2f B/clk/SM (max clock %d MHz)  err=%s\n",
             mode == 0 ? "global L1/L2 (512 KiB)" : mode == 1 ? "DSMEM 8-CTA cluster" : "local smem (64 KiB slice)",
             grid, ms, gathers / (ms * 1e-3) / 1e9, per_sm_clk, clk_khz / 1000, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
