// Shared internals of libvecinfer (sm_100a).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>
#include <utility>
#include <type_traits>

#include "../../include/vecinfer.h"

namespace vecinfer {

// ------------------------------------------------------------------ host-side error helpers
void set_error(const char* fmt, ...);
vecinfer_status_t fail(vecinfer_status_t st, const char* fmt, ...);
vecinfer_status_t check_launch(const char* what);
int device_sm_count();  // cached per device

inline cudaStream_t as_stream(vecinfer_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
// Launch with programmatic dependent launch enabled: the kernel may start while its predecessor
// on the stream drains; it must call griddep_wait() before touching anything the predecessor
// may write (our kernels read only static weights -- codebooks, lambda -- before the wait).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// validation of a paged-cache descriptor (include/vecinfer.h, vecinfer_paged_t)
vecinfer_status_t check_paged(const vecinfer_paged_t* pg, int64_t n_cap, const char* who);

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// pack two floats into an fp16x2 register: lo -> bits [0,16), hi -> bits [16,32)
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// D(16x8 f32) += A(16x16 f16, row) * B(16x8 f16, col)
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// transpose an 8x8 b16 matrix held in mma fragment layout across the warp
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t ldg_nc_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ldg_nc_u64(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ldg_nc_u128(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t ldg_nc_u16(const void* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint32_t>(v);
}
__device__ __forceinline__ uint32_t ldg_nc_u8(const void* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint32_t>(v);
}
// read-only load that may allocate in L1 (codebook gathers)
__device__ __forceinline__ uint2 ldg_ro_u64(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// read-only loads that may allocate in L1 (sub-word code chunks of the NEXT-2 formats: the bytes
// of one chunk are fetched by several loads, the first brings the sector into L1)
__device__ __forceinline__ uint32_t ldg_ro_u8(const void* p) {
  unsigned short v;
  asm volatile("ld.global.nc.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint32_t>(v);
}
__device__ __forceinline__ uint32_t ldg_ro_u16(const void* p) {
  unsigned short v;
  asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint32_t>(v);
}
__device__ __forceinline__ uint32_t ldg_ro_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// compile-time unrolled loop: f(std::integral_constant<int, I>) for I in [B, E)
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint4 lds_u128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint2 lds_u64(uint32_t saddr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(saddr));
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// bulk async copy global -> shared (the TMA engine; no registers, no LSU instructions per byte):
// completion is signalled on an mbarrier whose transaction count was raised by expect_tx.
// dst, src and bytes must be multiples of 16.
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

// bulk L2 prefetch of [p, p + bytes) (bytes a multiple of 16): no registers, no completion tracking
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// gpu-scope acq_rel atomic add (returns the old value).  After a CTA barrier, thread 0's release
// is cumulative over the CTA's prior global stores (PTX memory model), and its acquire, followed
// by a CTA barrier, orders the CTA's later loads after the other CTAs' released stores.
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// floor(x / d) for 0 <= x < 2^24, 1 <= d < 2^24: float reciprocal estimate + exact fix-up
__device__ __forceinline__ int div_small(int x, int d) {
  int q = __float2int_rz(__int2float_rn(x) * __frcp_rn(__int2float_rn(d)));
  int rr = x - q * d;
  while (rr < 0) { --q; rr += d; }
  while (rr >= d) { ++q; rr -= d; }
  return q;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// weak global load that never allocates in L1 (workspace partials: ordering comes from an acquire
// + CTA barrier; no L1 line of the workspace is ever allocated, so none can be stale)
__device__ __forceinline__ float ld_na_f32(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// ---- thread-block clusters / distributed shared memory
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// split cluster barrier: arrive early (relaxed), wait later -- used to guarantee every CTA of the
// cluster has started before any distributed-shared-memory access
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// ---- programmatic dependent launch (no-ops when the launch did not enable PDL)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Pinned fp32 squared distance of reading R9: ((e0^2 + e1^2) + e2^2) + e3^2, RN, no FMA.
__device__ __forceinline__ float pinned_dist4(float x0, float x1, float x2, float x3, float c0,
                                              float c1, float c2, float c3) {
  const float e0 = __fsub_rn(x0, c0), e1 = __fsub_rn(x1, c1);
  const float e2 = __fsub_rn(x2, c2), e3 = __fsub_rn(x3, c3);
  float s = __fadd_rn(__fmul_rn(e0, e0), __fmul_rn(e1, e1));
  s = __fadd_rn(s, __fmul_rn(e2, e2));
  return __fadd_rn(s, __fmul_rn(e3, e3));
}

// The same pinned distance for two centroids j, j+1 at once with Blackwell's paired fp32 ops for
// the differences and squares (FADD2 / FMUL2: IEEE round-to-nearest per element, subnormals kept)
// and scalar __fadd_rn for the ordered sums -- the exact per-element results of pinned_dist4 in 14
// instructions for 2 pairs instead of 22.  Centroid
// pair layout (32 B): p01 = {c_j.x, c_j+1.x, c_j.y, c_j+1.y}, p23 = {c_j.z, c_j+1.z, c_j.w, c_j+1.w};
// returns {dist_j, dist_j+1}.
__device__ __forceinline__ unsigned long long f32x2_pack(uint32_t lo, uint32_t hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ unsigned long long f32x2_splat(float x) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float2 pinned_dist4_x2(float x0, float x1, float x2, float x3, const uint4& p01,
                                                  const uint4& p23) {
  unsigned long long e0, e1, e2, e3;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e0) : "l"(f32x2_splat(x0)), "l"(f32x2_pack(p01.x, p01.y)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e1) : "l"(f32x2_splat(x1)), "l"(f32x2_pack(p01.z, p01.w)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e2) : "l"(f32x2_splat(x2)), "l"(f32x2_pack(p23.x, p23.y)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e3) : "l"(f32x2_splat(x3)), "l"(f32x2_pack(p23.z, p23.w)));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(e0) : "l"(e0));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(e1) : "l"(e1));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(e2) : "l"(e2));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(e3) : "l"(e3));
  // the sums stay scalar __fadd_rn: ptxas contracts mul.rn.f32x2 followed by add.rn.f32x2 into
  // FFMA2 (even with -fmad=false), which would round e_t^2 + s once instead of twice
  float q0x, q0y, q1x, q1y, q2x, q2y, q3x, q3y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(q0x), "=f"(q0y) : "l"(e0));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(q1x), "=f"(q1y) : "l"(e1));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(q2x), "=f"(q2y) : "l"(e2));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(q3x), "=f"(q3y) : "l"(e3));
  const float d0 = __fadd_rn(__fadd_rn(__fadd_rn(q0x, q1x), q2x), q3x);
  const float d1 = __fadd_rn(__fadd_rn(__fadd_rn(q0y, q1y), q2y), q3y);
  return make_float2(d0, d1);
}
// stage the bf16 centroid pair (j, j+1) of a [n][4] codebook into the 32-byte paired layout
__device__ __forceinline__ void stage_centroid_pair(const uint16_t* cb, int j, uint4* dst) {
  const uint2 a = *reinterpret_cast<const uint2*>(cb + 4 * j);
  const uint2 b = *reinterpret_cast<const uint2*>(cb + 4 * (j + 1));
  dst[0] = make_uint4(a.x << 16, b.x << 16, a.x & 0xFFFF0000u, b.x & 0xFFFF0000u);
  dst[1] = make_uint4(a.y << 16, b.y << 16, a.y & 0xFFFF0000u, b.y & 0xFFFF0000u);
}

// Key side of the dual transform for the 4 dims [4*lane, 4*lane+4) held by this lane (one warp =
// one 128-dim key), on the pinned exact fixed point (R10):
//   A = rint_even(k * inv_lambda * 2^24) in int64 (the f64 product bf16 x fp32 is exact),
//   X = A H_pm  (2 in-register + 5 warp-shuffle butterfly stages, exact integer arithmetic),
//   x = RN32(RN32(X) * 2^-24) * RN32(1/sqrt(D)).
// krow4/inv4 point at this lane's 4 elements.  Returns true (warp-uniform) if any |k*inv| >= 2^32.
// nlanes = D / 4 lanes hold the key (32 for D = 128, 16 for D = 64; with 16 the upper half-warp
// computes a duplicate of the lower one and the butterflies never cross the halves).
__device__ __forceinline__ bool key_transform_lane(const uint16_t* krow4, const float* inv4, float inv_sqrt_d,
                                                   int lane, float (&x)[4], int nlanes = 32) {
  const uint2 kw = *reinterpret_cast<const uint2*>(krow4);
  const float kf[4] = {__uint_as_float(kw.x << 16), __uint_as_float(kw.x & 0xFFFF0000u),
                       __uint_as_float(kw.y << 16), __uint_as_float(kw.y & 0xFFFF0000u)};
  const float4 il = *reinterpret_cast<const float4*>(inv4);
  const float ilv[4] = {il.x, il.y, il.z, il.w};
  long long A[4];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double p = __dmul_rn(static_cast<double>(kf[i]), static_cast<double>(ilv[i]));  // exact
    bad |= !(fabs(p) < 4294967296.0);
    A[i] = __double2ll_rn(__dmul_rn(p, 16777216.0));  // ties-to-even, exact scaling
  }
  long long s0 = A[0] + A[1], s1 = A[0] - A[1], s2 = A[2] + A[3], s3 = A[2] - A[3];
  A[0] = s0 + s2; A[2] = s0 - s2; A[1] = s1 + s3; A[3] = s1 - s3;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    if (m >= nlanes) break;
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long o = __shfl_xor_sync(0xffffffffu, A[i], m);
      A[i] = upper ? (o - A[i]) : (A[i] + o);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    x[i] = __fmul_rn(__fmul_rn(__ll2float_rn(A[i]), 5.9604644775390625e-08f), inv_sqrt_d);
  return __any_sync(0xffffffffu, bad);
}

__device__ __forceinline__ float4 bf16x4_to_float4(uint2 w) {
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u), __uint_as_float(w.y << 16),
                     __uint_as_float(w.y & 0xFFFF0000u));
}

// Phase timestamps for profiling builds (-DVECINFER_PHASE_TIMING): thread 0 of each CTA writes
// %globaltimer (ns) at phase boundaries into a device buffer set with vecinfer_debug_set_phase_buffer.
unsigned long long* phase_buffer();  // host: set by vecinfer_debug_set_phase_buffer (profiling builds)
#ifdef VECINFER_PHASE_TIMING
__device__ __forceinline__ void phase_mark(unsigned long long* buf, int cta, int slot) {
  if (threadIdx.x == 0 && buf) {
    unsigned long long t, c;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    buf[cta * 32 + slot] = t;        // 16 slots per CTA: globaltimer (ns, coarse, comparable across SMs)
    buf[cta * 32 + 16 + slot] = c;   // and the SM cycle counter (fine, within the CTA)
    if (slot == 0) {                 // slot 15: the SM the CTA runs on
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      buf[cta * 32 + 15] = sm;
    }
  }
}
#else
__device__ __forceinline__ void phase_mark(unsigned long long*, int, int) {}
#endif

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace vecinfer
