// Probe of the tcgen05 pieces the attention score path uses (sm_100a), checked against the host:
//  1. tcgen05.st.32x32b (lane t -> TMEM lane t, consecutive columns) then tcgen05.ld.16x256b: which
//     (TMEM lane, column) each thread receives;
//  2. D[128 x 16] = A[128 x 128] (fp16, A in TMEM: lane = row, column c = elements 2c, 2c+1) x
//     B^T (B = [16 x 128] fp16 in shared memory, K-major, no swizzle: core matrices of 8 rows x 16 B,
//     LBO = next 8 K-elements, SBO = next 8 rows), fp32 accumulate, 8 MMAs of K = 16, committed to
//     an mbarrier; D read back with tcgen05.ld.32x32b and compared with a host fp64 product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_tcgen05 scripts/probe_tcgen05.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(uint32_t* ld_out, const __half* A, const __half* Bm, float* D) {
  __shared__ uint32_t tmem_base;
  __shared__ __align__(128) unsigned char bsm[4096];
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // B into shared memory: element (n, k) at ((k/8)*2 + n/8)*128 + (n%8)*16 + (k%8)*2
  for (int e = tid; e < 16 * 128; e += blockDim.x) {
    const int n = e / 128, k = e % 128;
    *reinterpret_cast<__half*>(bsm + ((k / 8) * 2 + n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = Bm[n * 128 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  const uint32_t lane_base = static_cast<uint32_t>(32 * (warp & 3)) << 16;

  // ---- 1. layout probe on columns [200, 208): value = (TMEM lane << 8) | column
  {
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) v[c] = ((32 * warp + lane) << 8) | c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(tb + lane_base + 200), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                    "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tb + lane_base + 200));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; ++i) ld_out[tid * 4 + i] = r[i];
  }

  // ---- 2. MMA: A rows into TMEM columns [0, 64), D at columns [64, 80)
  {
    const int row = 32 * warp + lane;
    uint32_t w[16];
    for (int cc = 0; cc < 4; ++cc) {
      for (int c = 0; c < 16; ++c) {
        const int col = 16 * cc + c;
        const __half lo = A[row * 128 + 2 * col], hi = A[row * 128 + 2 * col + 1];
        w[c] = static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                   :: "r"(tb + lane_base + 16 * cc), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]),
                      "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                      "r"(w[14]), "r"(w[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 17) | (8u << 24);   // f32 D, f16 A/B, K-major, N = 16, M = 128
    const uint32_t bs = smem_u32(bsm);
    for (int s = 0; s < 8; ++s) {
      const uint64_t desc = (static_cast<uint64_t>(((bs + 512 * s) >> 4) & 0x3FFF)) |
                            (static_cast<uint64_t>(256 >> 4) << 16) | (static_cast<uint64_t>(128 >> 4) << 32) |
                            (1ull << 46);
      const uint32_t acc = s > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                   :: "r"(tb + 64), "r"(tb + 8 * s), "l"(desc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tb + lane_base + 64));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * warp + lane;
    for (int n = 0; n < 16; ++n) D[row * 16 + n] = __uint_as_float(r[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "r"(256));
}

int main() {
  __half *A, *B;
  float* D;
  uint32_t* ldo;
  cudaMallocManaged(&A, 128 * 128 * 2);
  cudaMallocManaged(&B, 16 * 128 * 2);
  cudaMallocManaged(&D, 128 * 16 * 4);
  cudaMallocManaged(&ldo, 128 * 4 * 4);
  srand(1);
  for (int i = 0; i < 128 * 128; ++i) A[i] = __float2half((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < 16 * 128; ++i) B[i] = __float2half((rand() % 13 - 6) / 4.0f);
  probe<<<1, 128>>>(ldo, A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  // 1. 16x256b mapping
  int ok1 = 1;
  for (int t = 0; t < 128; ++t) {
    const int w = t / 32, l = t % 32;
    for (int i = 0; i < 4; ++i) {
      const uint32_t v = ldo[t * 4 + i];
      const int tl = v >> 8, col = v & 255;
      const int exp_l = 32 * w + l / 4 + (i >= 2 ? 8 : 0), exp_c = 2 * (l % 4) + (i & 1);
      if (tl != exp_l || col != exp_c) {
        if (ok1) printf("16x256b: thread %d reg %d got (lane %d, col %d), expected (%d, %d)\n", t, i, tl, col, exp_l, exp_c);
        ok1 = 0;
      }
    }
  }
  printf("16x256b layout (r0,r1 = lane l/4 cols 2(l%%4)+{0,1}; r2,r3 = lane l/4+8): %s\n", ok1 ? "OK" : "MISMATCH");
  // 2. MMA
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      double s = 0;
      for (int k = 0; k < 128; ++k) s += (double)__half2float(A[m * 128 + k]) * (double)__half2float(B[n * 128 + k]);
      maxerr = fmax(maxerr, fabs(s - D[m * 16 + n]));
    }
  printf("tcgen05.mma A-in-TMEM x B(smem, K-major, no swizzle) max |err| = %.3e -> %s\n", maxerr, maxerr < 1e-3 ? "OK" : "MISMATCH");
  if (maxerr >= 1e-3) {
    for (int n = 0; n < 4; ++n) {
      double s = 0;
      for (int k = 0; k < 128; ++k) s += (double)__half2float(A[k]) * (double)__half2float(B[n * 128 + k]);
      printf("  D[0][%d] = %f expected %f\n", n, D[n], s);
    }
  }
  return (ok1 && maxerr < 1e-3) ? 0 : 2;
}
