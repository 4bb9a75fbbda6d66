// Microbenchmarks to validate the decode-kernel design on B200 (scratch, not product).
#include <cstdio>
#include <cuda_fp16.h>
#include <cstdint>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__global__ void hmma_bench(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0*3, a2 = a0*5, a3 = a0*7, b0 = a0*11, b1 = a0*13;
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// conflict-free replicated gather: table [256][16 copies] of 8B
__global__ void lds_bench(float* out, int iters, uint32_t seed) {
  extern __shared__ uint2 tab[];
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) tab[i] = make_uint2(i, i * 7);
  __syncthreads();
  uint32_t x = seed ^ (threadIdx.x * 2654435761u);
  uint32_t acc0 = 0, acc1 = 0;
  const int lane = threadIdx.x & 15;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      uint32_t j = (x >> (k & 7) * 3) & 255;   // pseudo-random index
      uint2 v = tab[j * 16 + lane];
      acc0 += v.x; acc1 ^= v.y;
      x = x * 1664525u + 1013904223u + v.x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc0 + acc1);
}

// same but non-replicated (random conflicts)
__global__ void lds_bench_norep(float* out, int iters, uint32_t seed) {
  extern __shared__ uint2 tab[];
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) tab[i] = make_uint2(i, i * 7);
  __syncthreads();
  uint32_t x = seed ^ (threadIdx.x * 2654435761u);
  uint32_t acc0 = 0, acc1 = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      uint32_t j = (x >> (k & 7) * 3) & 255;
      uint2 v = tab[j];
      acc0 += v.x; acc1 ^= v.y;
      x = x * 1664525u + 1013904223u + v.x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc0 + acc1);
}

__global__ void copy_bench(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void read_bench(const int4* __restrict__ a, int* out, size_t n) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { int4 v = __ldg(a + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("name %s SMs %d smemPerSM %zu smemOptin %zu L2 %d regsPerSM %d clock_khz %d cc %d.%d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.l2CacheSize, p.regsPerMultiprocessor, clk, p.major, p.minor);
  float* out; CK(cudaMalloc(&out, 148 * 1024 * 8 * sizeof(float)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4000;
    hmma_bench<<<sms, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    hmma_bench<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n_mma = (double)sms * warps * iters * 8;
    printf("HMMA m16n8k16 f16->f32 warps/SM %2d: %.3f ms, %.1f TFLOP/s, %.3f MMA/clk/SM(at %d MHz)\n", warps, ms,
           n_mma * 4096 / ms / 1e9, n_mma / sms / (ms * 1e-3 * clk * 1e3), clk / 1000);
  }
  CK(cudaFuncSetAttribute(lds_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  CK(cudaFuncSetAttribute(lds_bench_norep, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for (int warps : {8, 16, 32}) {
    int iters = 4000;
    lds_bench<<<sms, warps * 32, 32768>>>(out, 10, 1);
    cudaEventRecord(e0);
    lds_bench<<<sms, warps * 32, 32768>>>(out, iters, 1);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)sms * warps * 32 * iters * 16 * 8;
    printf("LDS.64 replicated gather warps/SM %2d: %.3f ms, %.1f TB/s, %.1f B/clk/SM\n", warps, ms, bytes / ms / 1e9, bytes / sms / (ms * 1e-3 * clk * 1e3));
    lds_bench_norep<<<sms, warps * 32, 32768>>>(out, 10, 1);
    cudaEventRecord(e0);
    lds_bench_norep<<<sms, warps * 32, 32768>>>(out, iters, 1);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDS.64 NON-replicated gather warps/SM %2d: %.3f ms, %.1f TB/s, %.1f B/clk/SM\n", warps, ms, bytes / ms / 1e9, bytes / sms / (ms * 1e-3 * clk * 1e3));
  }
  size_t nbytes = 1ull << 30; int4 *a, *b; CK(cudaMalloc(&a, nbytes)); CK(cudaMalloc(&b, nbytes));
  cudaMemset(a, 1, nbytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy_bench<<<sms * 8, 512>>>(a, b, nbytes / 16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("copy 1GiB: %.1f GB/s (r+w)\n", 2.0 * nbytes / ms / 1e6);
    cudaEventRecord(e0); read_bench<<<sms * 8, 512>>>(a, (int*)out, nbytes / 16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("read 1GiB: %.1f GB/s\n", 1.0 * nbytes / ms / 1e6);
  }
  // launch latency: back-to-back empty-ish kernels
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int i = 0; i < 1000; ++i) read_bench<<<sms, 128>>>(a, (int*)out, 0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("empty launch back-to-back: %.2f us each\n", ms);
  }
  return 0;
}
