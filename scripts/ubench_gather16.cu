// Gather bound of the b4d4 attention path (65 536-entry bf16 codebooks, 512 KiB per book, K + V):
// every cached (token, KV head) needs 32 K + 32 V random 8-byte centroid gathers = 512 B, served by
// L1/L2 (the books do not fit shared memory).  This kernel does ONLY that work, with the attention
// kernel's launch shape (one 512-thread CTA per SM, 16 warps) and code stream (16-bit codes read
// from HBM, 64 B K + 64 B V per token-head), and reports the achieved gather rate: the ceiling the
// b4d4 attention kernel is compared against.  Variants: codes from HBM or hashed in registers,
// ld.global.nc (L1-allocating) vs ld.global.nc.L1::no_allocate, 1 or 2 tables.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gather16 scripts/ubench_gather16.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint2 ld_nc(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ld_nc_na(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
// centroid ci of a book whose entries [0, kSlice) also sit in shared memory (slice, 8 B each):
// a predicated LDS for those, a predicated LDG for the rest (no branch)
__device__ __forceinline__ uint2 ld_split(const void* g, uint32_t s, uint32_t ci, uint32_t n_slice) {
  uint2 v;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %2, %3;\n\t@p ld.shared.v2.u32 {%0,%1}, [%4];\n\t"
               "@!p ld.global.nc.v2.u32 {%0,%1}, [%5];\n\t}"
               : "=r"(v.x), "=r"(v.y) : "r"(ci), "r"(n_slice), "r"(s), "l"(g));
  return v;
}
__device__ __forceinline__ uint4 ld_codes(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// one warp-step = 32 token-heads x (K or V) half-rows: lane l reads 16 B of codes (8 codes) and
// gathers 8 centroids; two steps (K, V) per 32 token-half-rows.  Per token-head: 32 K + 32 V codes.
// kSlice > 0: entries [0, kSlice) of each book are staged in shared memory first (K slice, then V)
template <bool kHbmCodes, bool kNoAlloc, bool kTwoTables, int kSlice = 0>
__global__ void __launch_bounds__(512, 1) gather_kernel(const uint8_t* kcodes, const uint8_t* vcodes,
                                                        const uint16_t* ck, const uint16_t* cv,
                                                        long long rows_per_cta, unsigned* sink) {
  extern __shared__ __align__(16) uint8_t slice_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint16_t* cvv = kTwoTables ? cv : ck;
  uint32_t acc = 0;
  const uint32_t sk = static_cast<uint32_t>(__cvta_generic_to_shared(slice_smem));
  const uint32_t sv = sk + kSlice * 8;
  if (kSlice > 0) {
    for (int i = threadIdx.x; i < kSlice / 2; i += 512) {
      reinterpret_cast<uint4*>(slice_smem)[i] = reinterpret_cast<const uint4*>(ck)[i];
      reinterpret_cast<uint4*>(slice_smem + kSlice * 8)[i] = reinterpret_cast<const uint4*>(cvv)[i];
    }
    __syncthreads();
  }
  // each CTA streams its own contiguous code rows (64 B per row = one token-head's K or V codes)
  const long long row0 = blockIdx.x * rows_per_cta;
  uint32_t h = blockIdx.x * 7919u + threadIdx.x * 104729u;
  for (long long rw = warp * 8; rw < rows_per_cta; rw += 16 * 8) {   // 8 rows per warp-step: 4 lanes per row
    const long long row = row0 + rw + (lane >> 2);
    uint4 kc, vc;
    if (kHbmCodes) {
      kc = ld_codes(kcodes + row * 64 + 16 * (lane & 3));
      vc = ld_codes(vcodes + row * 64 + 16 * (lane & 3));
    } else {
      h = h * 1664525u + 1013904223u; kc.x = h; h = h * 1664525u + 1013904223u; kc.y = h;
      h = h * 1664525u + 1013904223u; kc.z = h; h = h * 1664525u + 1013904223u; kc.w = h;
      h = h * 1664525u + 1013904223u; vc.x = h; h = h * 1664525u + 1013904223u; vc.y = h;
      h = h * 1664525u + 1013904223u; vc.z = h; h = h * 1664525u + 1013904223u; vc.w = h;
    }
    const uint32_t kw[4] = {kc.x, kc.y, kc.z, kc.w}, vw[4] = {vc.x, vc.y, vc.z, vc.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t ci = (kw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
      const uint32_t di = (vw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
      uint2 a, b;
      if (kSlice > 0) {
        a = ld_split(ck + 4 * ci, sk + 8 * ci, ci, kSlice);
        b = ld_split(cvv + 4 * di, sv + 8 * di, di, kSlice);
      } else {
        a = kNoAlloc ? ld_nc_na(ck + 4 * ci) : ld_nc(ck + 4 * ci);
        b = kNoAlloc ? ld_nc_na(cvv + 4 * di) : ld_nc(cvv + 4 * di);
      }
      acc += a.x ^ a.y ^ b.x ^ b.y;
    }
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, acc);
}

template <bool H, bool N, bool T, int SL = 0>
void run(const char* name, const uint8_t* kc, const uint8_t* vc, const uint16_t* ck, const uint16_t* cv,
         long long rows_per_cta, int sms, unsigned* sink, int clk_mhz) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = SL * 16;
  cudaFuncSetAttribute(gather_kernel<H, N, T, SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel<H, N, T, SL>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxL1);
  gather_kernel<H, N, T, SL><<<sms, 512, smem>>>(kc, vc, ck, cv, rows_per_cta, sink);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gather_kernel<H, N, T, SL><<<sms, 512, smem>>>(kc, vc, ck, cv, rows_per_cta, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double s = ms / 1e3 / reps;
  const double token_heads = static_cast<double>(rows_per_cta) * sms;   // one K row + one V row each
  const double gather_bytes = token_heads * 64 * 8;                     // 32 K + 32 V gathers of 8 B
  const double clk = s * clk_mhz * 1e6;
  printf("%-44s %8.1f us  %6.2f B/clk/SM gathered  %6.1f clk/token-head/SM  (%.2f G token-heads/s)\n", name,
         s * 1e6, gather_bytes / sms / clk, clk * sms / token_heads, token_heads / s / 1e9);
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int clk_mhz = clk_khz / 1000;
  const long long rows_per_cta = 65536LL * 8 / 148 * 18 / 8;    // ~ the steady-state b4d4 launch: 8 x 65536 token-heads
  const long long rows = rows_per_cta * sms;
  uint8_t *kc, *vc;
  uint16_t *ck, *cv;
  unsigned* sink;
  cudaMalloc(&kc, rows * 64);
  cudaMalloc(&vc, rows * 64);
  cudaMalloc(&ck, 65536 * 8);
  cudaMalloc(&cv, 65536 * 8);
  cudaMalloc(&sink, 4);
  std::vector<uint8_t> h(rows * 64);
  uint32_t s = 12345;
  for (auto& x : h) { s = s * 1664525u + 1013904223u; x = s >> 24; }
  cudaMemcpy(kc, h.data(), h.size(), cudaMemcpyHostToDevice);
  for (auto& x : h) { s = s * 1664525u + 1013904223u; x = s >> 24; }
  cudaMemcpy(vc, h.data(), h.size(), cudaMemcpyHostToDevice);
  cudaMemset(ck, 0x3c, 65536 * 8);
  cudaMemset(cv, 0x3d, 65536 * 8);
  printf("SMs %d, SM clock %d MHz, %lld token-heads per launch\n", sms, clk_mhz, rows);
  run<true, false, true>("HBM codes, L1-allocating, K+V books", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<true, true, true>("HBM codes, L1::no_allocate, K+V books", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<false, false, true>("hashed codes, L1-allocating, K+V books", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<true, false, false>("HBM codes, L1-allocating, one book (K=V)", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<true, false, true, 4096>("HBM codes, K+V books, 2x 32 KiB in smem", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<true, false, true, 8192>("HBM codes, K+V books, 2x 64 KiB in smem", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<true, false, true, 11776>("HBM codes, K+V books, 2x 92 KiB in smem", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  run<true, false, true, 14336>("HBM codes, K+V books, 2x 112 KiB in smem", kc, vc, ck, cv, rows_per_cta, sms, sink, clk_mhz);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
