// Paper-faithful variant of N4: Algorithm 1 of VecInfer on sm_100a, LUT algorithm.
//
// Grid (num_splits, H_kv, B) with 128 threads per CTA as in the paper.  Per CTA:
//   l.4   lut[m][j][g] = q~'_g[m] . C_k[j]  (fp32, all G heads interleaved, 128 KiB of smem)
//   l.7   C_v -> shared memory
//   l.8-17 tiles of B = 128 tokens: key codes of tile i+1 and value codes of tile i are
//          prefetched with cp.async (the paper's memcpy_async double buffer, l.10 / l.15);
//          s = lookup(K_q, lut) (l.11; one float4 LUT read per sub-vector), online softmax
//          (l.12-13), o = diag(e^{m-m_new}) o + p VQ^-1(V_q, C_v) (l.16) with thread = dim.
//   l.19-22 o / l, L = m + log l; splits merged by the shared last-CTA epilogue.
// This kernel exists to evidence the design choice of the DEQUANT_MMA default: its key path
// reads 16 B of shared memory per (token, sub-vector) (vs 8 B for a dequantised gather) and
// its P.V runs on CUDA cores.
#include "attn_common.cuh"

namespace vecinfer {
namespace {

constexpr int kT = 128;  // threads per CTA == tokens per tile == head_dim
constexpr int kRow = 32; // 8-bit code row bytes

struct SmemLut {
  float4 lut[32 * 256];           // [m][j] -> 4 heads
  float cv[256][4];
  float q[4][128];
  uint8_t kc[2][kT * kRow];       // double-buffered key code tiles
  uint8_t vc[2][kT * kRow];       // double-buffered value code tiles
  float p[4][kT];
  float red[4][4];
  float wm[4], wl[4];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = smem_u32(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// copy the 128 code rows (32 B each) of a tile: 256 x 16-byte chunks, 2 per thread
__device__ __forceinline__ void issue_tile(uint8_t* dst, const uint8_t* src, int64_t t0, int64_t r1, int tid) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int c = tid + i * kT;
    const int64_t tok = t0 + (c >> 1);
    cp_async16(dst + c * 16, src + (tok < r1 ? tok : 0) * kRow + (c & 1) * 16, tok < r1);
  }
}

__global__ void __launch_bounds__(kT, 1) attn_lut8_kernel(const AttnArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemLut& sm = *reinterpret_cast<SmemLut*>(smem_raw);
  const int s = blockIdx.x, h = blockIdx.y, b = blockIdx.z;   // (non-persistent grid)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  griddep_wait();
  int64_t r0, r1;
  split_range(a, b, s, r0, r1);
  const int64_t ntile = (r1 - r0 + kT - 1) / kT;
  const int64_t unit = static_cast<int64_t>(b) * a.Hkv + h;
  const uint8_t* kb = a.kcodes + unit * a.n_cap * kRow;
  const uint8_t* vb = a.vcodes + unit * a.n_cap * kRow;

  if (ntile > 0) { issue_tile(sm.kc[0], kb, r0, r1, tid); }   // l.9: K_q^(1)
  cp_async_commit();

  // l.2: q~ (scaled by 1/sqrt(D) * softmax_scale * log2 e); l.7: C_v
  query_transform_warp(a, b, h, warp, sm.q[warp]);
  {
    const uint16_t* cv = a.cv + h * a.cv_hs;
    for (int j = tid; j < 256; j += kT) {
      const uint2 w = *reinterpret_cast<const uint2*>(cv + 4 * j);
      sm.cv[j][0] = __uint_as_float(w.x << 16);
      sm.cv[j][1] = __uint_as_float(w.x & 0xFFFF0000u);
      sm.cv[j][2] = __uint_as_float(w.y << 16);
      sm.cv[j][3] = __uint_as_float(w.y & 0xFFFF0000u);
    }
  }
  __syncthreads();
  // l.4: lut = q~' C_k^T for the 4 heads
  {
    const uint16_t* ck = a.ck + h * a.ck_hs;
    for (int idx = tid; idx < 32 * 256; idx += kT) {
      const int m = idx >> 8, jj = idx & 255;
      const uint2 w = *reinterpret_cast<const uint2*>(ck + 4 * jj);
      const float c0 = __uint_as_float(w.x << 16), c1 = __uint_as_float(w.x & 0xFFFF0000u);
      const float c2 = __uint_as_float(w.y << 16), c3 = __uint_as_float(w.y & 0xFFFF0000u);
      float4 e;
      e.x = sm.q[0][4 * m] * c0 + sm.q[0][4 * m + 1] * c1 + sm.q[0][4 * m + 2] * c2 + sm.q[0][4 * m + 3] * c3;
      e.y = sm.q[1][4 * m] * c0 + sm.q[1][4 * m + 1] * c1 + sm.q[1][4 * m + 2] * c2 + sm.q[1][4 * m + 3] * c3;
      e.z = sm.q[2][4 * m] * c0 + sm.q[2][4 * m + 1] * c1 + sm.q[2][4 * m + 2] * c2 + sm.q[2][4 * m + 3] * c3;
      e.w = sm.q[3][4 * m] * c0 + sm.q[3][4 * m + 1] * c1 + sm.q[3][4 * m + 2] * c2 + sm.q[3][4 * m + 3] * c3;
      sm.lut[idx] = e;
    }
  }
  float o[4] = {0.f, 0.f, 0.f, 0.f};   // thread = output dim `tid`, all 4 heads
  float m_run[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  float l_run[4] = {0.f, 0.f, 0.f, 0.f};

  for (int64_t i = 0; i < ntile; ++i) {
    const int buf = static_cast<int>(i & 1);
    const int64_t t0 = r0 + i * kT;
    issue_tile(sm.vc[buf], vb, t0, r1, tid);            // l.10: prefetch V_q^(i)
    cp_async_commit();
    cp_async_wait<1>();                                  // K_q^(i) landed
    __syncthreads();
    // l.11: s = lookup(K_q^(i), lut); thread = token
    const int64_t tok = t0 + tid;
    float sg[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const uint32_t* row = reinterpret_cast<const uint32_t*>(sm.kc[buf] + tid * kRow);
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const uint32_t cw = row[w];
#pragma unroll
        for (int by = 0; by < 4; ++by) {
          const float4 e = sm.lut[(4 * w + by) * 256 + ((cw >> (8 * by)) & 255)];
          sg[0] += e.x; sg[1] += e.y; sg[2] += e.z; sg[3] += e.w;
        }
      }
    }
    // l.12-13: block max per head
    float mloc[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      sg[g] = tok < r1 ? sg[g] : -INFINITY;
      float v = sg[g];
      for (int off = 16; off; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
      mloc[g] = v;
    }
    if (lane == 0) for (int g = 0; g < 4; ++g) sm.red[warp][g] = mloc[g];
    __syncthreads();
    float alpha[4], mnew[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float mt = fmaxf(fmaxf(sm.red[0][g], sm.red[1][g]), fmaxf(sm.red[2][g], sm.red[3][g]));
      mnew[g] = fmaxf(m_run[g], mt);
      alpha[g] = mnew[g] == -INFINITY ? 1.f : ex2_approx(m_run[g] - mnew[g]);
      const float mu = mnew[g] == -INFINITY ? 0.f : mnew[g];
      sm.p[g][tid] = ex2_approx(sg[g] - mu);
    }
    if (i + 1 < ntile) issue_tile(sm.kc[buf ^ 1], kb, t0 + kT, r1, tid);   // l.15: prefetch K_q^(i+1)
    cp_async_commit();
    cp_async_wait<1>();                                  // l.14: V_q^(i) landed
    __syncthreads();
    // l.13 row sums + l.16 o update; thread = dim d, sub-vector d/4, component d%4
    const int m = tid >> 2, comp = tid & 3;
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, psum[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < kT; ++t) {
      const float c = sm.cv[sm.vc[buf][t * kRow + m]][comp];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const float p = sm.p[g][t];
        psum[g] += p;
        acc[g] += p * c;
      }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      o[g] = alpha[g] * o[g] + acc[g];
      l_run[g] = alpha[g] * l_run[g] + psum[g];
      m_run[g] = mnew[g];
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
  // hand the (m, l, o) of this CTA to the shared epilogue as a single "warp"
  float* wm = reinterpret_cast<float*>(smem_raw);   // reuse the LUT region
  float* wl = wm + 4;
  float* wacc = wl + 4;
  float* scratch = wacc + 4 * 128;
  if (tid < 4) { wm[tid] = m_run[tid]; wl[tid] = l_run[tid]; }
#pragma unroll
  for (int g = 0; g < 4; ++g) wacc[g * 128 + tid] = o[g];
  __syncthreads();
  cta_finish<kT, 1>(a, b, h, s, wm, wl, wacc, scratch);
}

}  // namespace

void launch_attn_lut(const AttnArgs& a, int kbits, int vbits, cudaStream_t st) {
  (void)kbits; (void)vbits;
  const size_t smem = sizeof(SmemLut);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_lut8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr_set = true;
  }
  attn_lut8_kernel<<<dim3(a.S, a.Hkv, a.B), kT, smem, st>>>(a);
}

}  // namespace vecinfer
