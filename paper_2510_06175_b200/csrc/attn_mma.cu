// N3+N4+N5: split-KV fused VQ decode attention, DEQUANT_MMA algorithm (default on sm_100a).
//
// Implements Eq. 10 with Algorithm 1's online softmax:
//   s = q~ VQ^-1(K~_q)^T / sqrt(D),  o = softmax(s) VQ^-1(V_q),  L = logsumexp(s).
// CTA = (split, KV head, batch); each of its NW warps streams 32-token tiles of packed codes
// straight from HBM into registers (LDG, one tile of prefetch) -- no dequantised cache, no
// shared-memory staging of codes.  Per warp and 16-token sub-tile:
//  score:  the key codes index a 16x-replicated fp16 copy of C_k in shared memory (lane l
//          reads copy l%16, so every 8-byte gather is bank-conflict-free); the gathered
//          centroids ARE the A fragments of mma.m16n8k16 (tokens x 16 dims, dims permuted so
//          that one gather = one fragment pair) against B = q~ for the G=4 heads of the GQA
//          group split into fp16 hi + lo parts (N = 8 = 4 heads x {hi, lo}): s = D[.,2g]+D[.,2g+1].
//  softmax: per-head running max with lazy rescaling (only when the max grows by > 2^8),
//          exp2 with log2(e) folded into q~; p split into fp16 hi/lo and moved from the
//          accumulator layout to the B-operand layout with movmatrix.trans.
//  P.V:    V^T (16 dims x 16 tokens) built from replicated C_v gathers (PRMT pairs tokens)
//          times P (16 tokens x 8 = 4 heads x {hi, lo}); fp32 accumulators in registers.
// Epilogue: warps combine through shared memory; splits merge by log-sum-exp in the last CTA
// of each (b, h_kv) (fixed order => deterministic).  See DESIGN.md "Kernel N4".
#include "attn_common.cuh"

namespace vecinfer {
namespace {

constexpr int kNW = 16;            // warps per CTA (1 CTA per SM)
constexpr int kThreads = kNW * 32;
constexpr float kTau = 8.0f;       // lazy-rescale threshold (log2 units): p <= 2^8
constexpr int kRep = 16;           // codebook replicas (one per half-warp lane)
constexpr int kRowBytes = 32;      // 8-bit codes, D/d = 32 sub-vectors

struct Smem8 {
  uint2 ck[256 * kRep];  // fp16x4 centroids, entry j copy c at [j*16 + c]
  uint2 cv[256 * kRep];
  float q[4][128];
};

__device__ __forceinline__ void fill_codebook(uint2* dst, const uint16_t* src, int tid) {
  // thread j converts centroid j (bf16 -> fp16, exact for |c| in the fp16 normal range) and
  // writes its 16 replicas as 8 x 16-byte stores, rotated so a quarter-warp hits 8 banks groups
  if (tid < 256) {
    const uint2 w = *reinterpret_cast<const uint2*>(src + 4 * tid);
    uint2 e;
    e.x = pack_half2(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u));
    e.y = pack_half2(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
    uint4 v = make_uint4(e.x, e.y, e.x, e.y);
#pragma unroll
    for (int u0 = 0; u0 < 8; ++u0) {
      const int u = (u0 + tid) & 7;
      *reinterpret_cast<uint4*>(&dst[tid * kRep + 2 * u]) = v;
    }
  }
}

struct TileCodes {
  uint2 k[2][2];     // [sub-tile][row r / r+8]: 8 key codes (sub-vectors 8j..8j+7)
  uint32_t v[2][4];  // [sub-tile][token 2j, 2j+1, 2j+8, 2j+9]: 4 value codes (sub-vectors 4r..4r+3)
};

__device__ __forceinline__ void load_tile(TileCodes& tc, const uint8_t* kb, const uint8_t* vb, int64_t t0,
                                          int64_t r1, int r, int j) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int64_t base = t0 + 16 * q;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int64_t tok = base + r + 8 * hh;
      tc.k[q][hh] = tok < r1 ? ldg_nc_u64(kb + tok * kRowBytes + 8 * j) : make_uint2(0u, 0u);
    }
    const int toks[4] = {2 * j, 2 * j + 1, 2 * j + 8, 2 * j + 9};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t tok = base + toks[i];
      tc.v[q][i] = tok < r1 ? ldg_nc_u32(vb + tok * kRowBytes + 4 * r) : 0u;
    }
  }
}

// byte t of a code word pair -> shared-memory byte offset of that centroid's replica row
__device__ __forceinline__ uint32_t code_off(uint32_t w, int byte) {
  return byte == 0 ? ((w << 7) & 0x7f80u) : ((w >> (8 * byte - 7)) & 0x7f80u);
}

__global__ void __launch_bounds__(kThreads, 1) attn_mma8_kernel(const AttnArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem8& sm = *reinterpret_cast<Smem8*>(smem_raw);
  const int s = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, j = lane & 3;

  int64_t r0, r1;
  split_range(a, b, s, r0, r1);
  const int64_t ntile = (r1 - r0 + 31) / 32;
  const int64_t unit = static_cast<int64_t>(b) * a.Hkv + h;
  const uint8_t* kb = a.kcodes + unit * a.n_cap * kRowBytes;
  const uint8_t* vb = a.vcodes + unit * a.n_cap * kRowBytes;

  // issue the first tile's loads before the prologue so HBM latency overlaps it
  TileCodes nxt;
  if (warp < ntile) load_tile(nxt, kb, vb, r0 + 32 * warp, r1, r, j);

  fill_codebook(sm.ck, a.ck + h * a.ck_hs, tid);
  if (tid >= 256) fill_codebook(sm.cv, a.cv + h * a.cv_hs, tid - 256);
  if (warp < 4) query_transform_warp(a, b, h, warp, sm.q[warp]);
  __syncthreads();

  // B fragments of the score MMA: column n = lane/4 <-> (head n/2, part n%2); rows k
  // <-> sub-vector 8j+t, components {0,1} (b0) and {2,3} (b1)
  uint32_t bq0[8], bq1[8];
  {
    const int gq = r >> 1, part = r & 1;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float4 v = *reinterpret_cast<const float4*>(&sm.q[gq][4 * (8 * j + t)]);
      const float in[4] = {v.x, v.y, v.z, v.w};
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __half hi = __float2half_rn(in[i]);
        o[i] = part == 0 ? __half2float(hi) : (in[i] - __half2float(hi));
      }
      bq0[t] = pack_half2(o[0], o[1]);
      bq1[t] = pack_half2(o[2], o[3]);
    }
  }

  const uint32_t ck_base = smem_u32(sm.ck) + (lane & 15) * 8;
  const uint32_t cv_base = smem_u32(sm.cv) + (lane & 15) * 8;

  float acc[8][4];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;

  for (int64_t it = warp; it < ntile; it += kNW) {
    const TileCodes cur = nxt;
    const int64_t t0 = r0 + 32 * it;
    if (it + kNW < ntile) load_tile(nxt, kb, vb, t0 + 32 * kNW, r1, r, j);

    // ---- scores (log2 units) for tokens t0 + 16q + {r, r+8}, head j
    float sc[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t wa = t < 4 ? cur.k[q][0].x : cur.k[q][0].y;
        const uint32_t wb = t < 4 ? cur.k[q][1].x : cur.k[q][1].y;
        const uint2 ea = lds_u64(ck_base + code_off(wa, t & 3));
        const uint2 eb = lds_u64(ck_base + code_off(wb, t & 3));
        mma_16816(d, ea.x, eb.x, ea.y, eb.y, bq0[t], bq1[t]);
      }
      const int64_t tok = t0 + 16 * q + r;
      sc[q][0] = tok < r1 ? d[0] + d[1] : -INFINITY;
      sc[q][1] = tok + 8 < r1 ? d[2] + d[3] : -INFINITY;
    }

    // ---- online softmax (Alg. 1 l.12-13, 18), lazy rescale
    float mx = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    const bool need = mx > m_run + kTau;
    if (__any_sync(0xffffffffu, need)) {
      const float m_new = need ? mx : m_run;
      const float alpha = need ? ex2_approx(m_run - m_new) : 1.f;  // 0 when m_run was -inf
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        acc[t][0] *= alpha; acc[t][1] *= alpha; acc[t][2] *= alpha; acc[t][3] *= alpha;
      }
      l_run *= alpha;
      m_run = m_new;
    }
    const float m_use = m_run == -INFINITY ? 0.f : m_run;

#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float p0 = ex2_approx(sc[q][0] - m_use);
      const float p1 = ex2_approx(sc[q][1] - m_use);
      l_run += p0 + p1;
      const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
      const __half l0 = __float2half_rn(p0 - __half2float(h0));
      const __half l1 = __float2half_rn(p1 - __half2float(h1));
      const uint32_t x0 = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(l0)) << 16);
      const uint32_t x1 = static_cast<uint32_t>(__half_as_ushort(h1)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
      const uint32_t bp0 = movmatrix_trans(x0);  // P^T rows (slots) x tokens 0..7
      const uint32_t bp1 = movmatrix_trans(x1);  // tokens 8..15

      // ---- P.V (Alg. 1 l.16): m-tile t <-> sub-vector 4r + t/2, components 2(t%2) + {0,1}
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint2 g0 = lds_u64(cv_base + code_off(cur.v[q][0], u));
        const uint2 g1 = lds_u64(cv_base + code_off(cur.v[q][1], u));
        const uint2 g2 = lds_u64(cv_base + code_off(cur.v[q][2], u));
        const uint2 g3 = lds_u64(cv_base + code_off(cur.v[q][3], u));
        mma_16816(acc[2 * u], prmt(g0.x, g1.x, 0x5410), prmt(g0.x, g1.x, 0x7632), prmt(g2.x, g3.x, 0x5410),
                  prmt(g2.x, g3.x, 0x7632), bp0, bp1);
        mma_16816(acc[2 * u + 1], prmt(g0.y, g1.y, 0x5410), prmt(g0.y, g1.y, 0x7632), prmt(g2.y, g3.y, 0x5410),
                  prmt(g2.y, g3.y, 0x7632), bp0, bp1);
      }
    }
  }

  // ---- warp partials -> shared memory (reusing the codebook region)
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 4);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 8);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
  __syncthreads();
  float* wm = reinterpret_cast<float*>(smem_raw);
  float* wl = wm + kNW * 4;
  float* wacc = wl + kNW * 4;
  if (r == 0) {
    wm[warp * 4 + j] = m_run;
    wl[warp * 4 + j] = l_run;
  }
  float* dst = wacc + (warp * 4 + j) * 128 + 16 * r;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    dst[2 * t] = acc[t][0] + acc[t][1];      // dim 16r + 2t     (h = 0: hi + lo slot)
    dst[2 * t + 1] = acc[t][2] + acc[t][3];  // dim 16r + 2t + 1 (h = 1)
  }
  __syncthreads();
  cta_finish<kThreads>(a, b, h, s, kNW, wm, wl, wacc);
}

}  // namespace

void launch_attn_mma(const AttnArgs& a, int kbits, int vbits, cudaStream_t st) {
  (void)kbits; (void)vbits;  // dispatch validated by the caller (8/8 only in v1)
  const size_t smem = sizeof(Smem8);
  static bool attr_set = false;  // benign race: idempotent attribute
  if (!attr_set) {
    cudaFuncSetAttribute(attn_mma8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr_set = true;
  }
  attn_mma8_kernel<<<dim3(a.S, a.Hkv, a.B), kThreads, smem, st>>>(a);
}

}  // namespace vecinfer
