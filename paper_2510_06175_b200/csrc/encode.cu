// N2: KV encode + cache store (Eq. 8 prefill / Eq. 9 decode append).
//
// One warp per (b, t, h) token-head; lane l owns dims [4l, 4l+4) = sub-vector l (d = 4).
//  key:   A = rint(k * inv_lambda * 2^24) (exact f64 product -> int64)       [smooth, Eq. 3]
//         X = A H_pm: 2 in-register butterfly stages + 5 warp-shuffle stages, int64 (exact,
//             so the result is independent of the butterfly order)            [Hadamard, Eq. 6]
//         x = RN32(RN32(X) * 2^-24) * RN32(1/sqrt(D))                         [reading R10]
//         code = argmin_j pinned_dist(x, C_k[j])  (lowest index on ties)      [Eq. 2, R9]
//  value: code = argmin_j pinned_dist(v, C_v[j])                                [Eq. 8]
// 4/8-bit codebooks live in shared memory as fp32 (all lanes read the same centroid ->
// broadcast, conflict-free).  16-bit codebooks (65536 entries, 512 KiB bf16) are scanned by
// centroid-split CTAs (1024 centroids staged per CTA) whose per-lane minima are combined
// with 64-bit atomicMin on (dist_bits << 32 | j) -- exact argmin with lowest-index ties,
// since dist >= 0 makes the fp32 bit pattern order-preserving.
#include "common.cuh"

namespace vecinfer {
namespace {

constexpr int kEncWarps = 8;
constexpr int kChunk16 = 1024;  // centroids per CTA for 16-bit codebooks

struct EncArgs {
  const uint16_t* k;
  const uint16_t* v;
  int B, T, H;
  int64_t ks_b, ks_t, ks_h, vs_b, vs_t, vs_h;
  const float* inv_lambda;
  const uint16_t* ck;
  const uint16_t* cv;
  int64_t ck_hs, cv_hs;
  int kbits, vbits;
  int ksub, vsub;             // sub-vector dims (4; NEXT-2 formats: 8 / 4 / 2)
  uint8_t* kcodes;
  uint8_t* vcodes;
  int64_t n_cap;
  const int32_t* bt;          // paged cache: block table (NULL: contiguous [B, H, n_cap, row])
  int64_t bt_stride;
  int page_shift, n_pages;
  const int32_t* write_pos;
  uint32_t* err;
  float inv_sqrt_d;
  int D, nsub;             // head dim (64 or 128) and sub-vectors (lanes holding the key) = D / 4
  unsigned long long* ws;  // 16-bit path: [B*T*H][2][32] packed minima
};

// Smoothing + exact integer FWHT + fixed-point -> fp32 (key_transform_lane), flags range errors.
__device__ __forceinline__ void transform_key_lane(const EncArgs& a, int b, int t, int h, int lane,
                                                   float (&x)[4]) {
  const int le = lane & (a.nsub - 1);   // D = 64: the upper half-warp duplicates the lower one
  const bool bad = key_transform_lane(a.k + b * a.ks_b + t * a.ks_t + h * a.ks_h + 4 * le,
                                      a.inv_lambda + h * a.D + 4 * le, a.inv_sqrt_d, lane, x, a.nsub);
  if (bad && lane == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_RANGE);
}

__device__ __forceinline__ void load_value_lane(const EncArgs& a, int b, int t, int h, int lane, float (&x)[4]) {
  const uint16_t* vp = a.v + b * a.vs_b + t * a.vs_t + h * a.vs_h + 4 * (lane & (a.nsub - 1));
  const uint2 w = *reinterpret_cast<const uint2*>(vp);
  x[0] = __uint_as_float(w.x << 16);
  x[1] = __uint_as_float(w.x & 0xFFFF0000u);
  x[2] = __uint_as_float(w.y << 16);
  x[3] = __uint_as_float(w.y & 0xFFFF0000u);
}

__device__ __forceinline__ void store_code(uint8_t* codes, int bits, int64_t row, int lane, uint32_t code,
                                           int nsub = 32) {
  const int row_bytes = nsub * bits / 8;
  uint8_t* p = codes + row * row_bytes;
  if (bits == 8) {
    if (lane < nsub) p[lane] = static_cast<uint8_t>(code);
  } else if (bits == 4) {
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, code, 1);
    if ((lane & 1) == 0 && lane < nsub) p[lane >> 1] = static_cast<uint8_t>(code | (hi << 4));
  } else {
    if (lane < nsub) reinterpret_cast<uint16_t*>(p)[lane] = static_cast<uint16_t>(code);
  }
}

__device__ __forceinline__ bool cache_row(const EncArgs& a, int b, int t, int h, int lane, int64_t& row) {
  const int64_t pos = static_cast<int64_t>(a.write_pos[b]) + t;
  if (pos < 0 || pos >= a.n_cap) {
    if (lane == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_WRITE_POS);
    return false;
  }
  if (a.bt) {   // paged: [n_pages, H, page_size, row]
    const int pg = a.bt[b * a.bt_stride + (pos >> a.page_shift)];
    if (pg < 0 || pg >= a.n_pages) {
      if (lane == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_WRITE_POS);
      return false;
    }
    row = ((static_cast<int64_t>(pg) * a.H + h) << a.page_shift) + (pos & ((int64_t(1) << a.page_shift) - 1));
    return true;
  }
  row = (static_cast<int64_t>(b) * a.H + h) * a.n_cap + pos;
  return true;
}

// ------------------------------------------------------------------ 4/8-bit: smem codebooks
// centroids staged as pairs (32 B per 2 entries, pinned_dist4_x2 layout): one FADD2 / FMUL2 per
// component for two centroids, same per-element rounding as the scalar pinned distance
template <int N>
__device__ __forceinline__ void scan_pairs(const uint4* sp, const float (&x)[4], uint32_t& bi) {
  float best = __int_as_float(0x7f800000);
  bi = 0;
#pragma unroll 4
  for (int p = 0; p < N / 2; ++p) {
    const float2 d = pinned_dist4_x2(x[0], x[1], x[2], x[3], sp[2 * p], sp[2 * p + 1]);
    if (d.x < best) { best = d.x; bi = 2 * p; }       // j = 2p first: lowest index on ties
    if (d.y < best) { best = d.y; bi = 2 * p + 1; }
  }
}

template <int KBITS, int VBITS>
__global__ void __launch_bounds__(kEncWarps * 32) encode_small_kernel(EncArgs a) {
  constexpr int NK = 1 << KBITS, NV = 1 << VBITS;
  __shared__ uint4 sck[NK];   // NK / 2 pairs x 32 B
  __shared__ uint4 scv[NV];
  griddep_launch_dependents();
  const int h = blockIdx.y;
  const uint16_t* ck = a.ck + h * a.ck_hs;
  const uint16_t* cv = a.cv + h * a.cv_hs;
  for (int p = threadIdx.x; p < NK / 2; p += blockDim.x) stage_centroid_pair(ck, 2 * p, sck + 2 * p);
  for (int p = threadIdx.x; p < NV / 2; p += blockDim.x) stage_centroid_pair(cv, 2 * p, scv + 2 * p);
  __syncthreads();
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int64_t bt = static_cast<int64_t>(blockIdx.x) * kEncWarps + (threadIdx.x >> 5);
  if (bt >= static_cast<int64_t>(a.B) * a.T) return;
  const int b = static_cast<int>(bt / a.T), t = static_cast<int>(bt % a.T);
  int64_t row;
  if (!cache_row(a, b, t, h, lane, row)) return;
  float x[4];
  transform_key_lane(a, b, t, h, lane, x);
  uint32_t bi;
  scan_pairs<NK>(sck, x, bi);
  store_code(a.kcodes, KBITS, row, lane, bi, a.nsub);
  load_value_lane(a, b, t, h, lane, x);
  scan_pairs<NV>(scv, x, bi);
  store_code(a.vcodes, VBITS, row, lane, bi, a.nsub);
}

// ------------------------------------------------------------------ 4/8-bit decode append
// Few token-heads (decode append, T = 1): one CTA of 16 warps per token-head.  Warps 0-7 search
// C_k, warps 8-15 search C_v, each over 1/8 of the centroids (staged by that warp only, so no
// CTA barrier before the scan); per-lane (dist, index) minima are reduced in warp order, which
// keeps the lowest-index tie rule (strict < within a warp, ascending centroid ranges across).
template <int KBITS, int VBITS>
__global__ void __launch_bounds__(512) encode_append_kernel(EncArgs a) {
  constexpr int NK = 1 << KBITS, NV = 1 << VBITS;
  constexpr int PK = (NK + 7) / 8, PV = (NV + 7) / 8;  // centroids per warp
  __shared__ float4 sc[8 * (PK > PV ? PK : PV) * 2];
  __shared__ float sbest[16][32];
  __shared__ uint32_t sidx[16][32];
  griddep_launch_dependents();
  const int h = blockIdx.y;
  const int64_t bt = blockIdx.x;
  const int b = static_cast<int>(bt / a.T), t = static_cast<int>(bt % a.T);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool isv = warp >= 8;
  const int w8 = warp & 7;
  const int P = isv ? PV : PK;
  const int n_ent = isv ? NV : NK;
  const int j0 = w8 * P;
  float4* mine = sc + (isv ? 8 * PK : 0) + w8 * P;
  const uint16_t* cb = isv ? (a.cv + h * a.cv_hs) : (a.ck + h * a.ck_hs);
  for (int i = lane; i < P; i += 32) {
    if (j0 + i < n_ent) {
      const uint2 w = *reinterpret_cast<const uint2*>(cb + 4 * (j0 + i));
      mine[i] = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                            __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
    }
  }
  griddep_wait();
  float x[4];
  if (isv) load_value_lane(a, b, t, h, lane, x);
  else transform_key_lane(a, b, t, h, lane, x);
  __syncwarp();
  float best = __int_as_float(0x7f800000);
  uint32_t bi = 0;
  const int cnt = min(P, n_ent - j0);
#pragma unroll 8
  for (int i = 0; i < cnt; ++i) {
    const float4 c = mine[i];
    const float dd = pinned_dist4(x[0], x[1], x[2], x[3], c.x, c.y, c.z, c.w);
    if (dd < best) { best = dd; bi = j0 + i; }
  }
  sbest[warp][lane] = best;
  sidx[warp][lane] = bi;
  __syncthreads();
  if (warp == 0 || warp == 8) {
    float bb = sbest[warp][lane];
    uint32_t ii = sidx[warp][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const float c = sbest[warp + w][lane];
      if (c < bb) { bb = c; ii = sidx[warp + w][lane]; }
    }
    int64_t row;
    if (cache_row(a, b, t, h, lane, row)) store_code(isv ? a.vcodes : a.kcodes, isv ? VBITS : KBITS, row, lane, ii, a.nsub);
  }
}

// ------------------------------------------------------------------ 16-bit: centroid split
// grid (ceil(B*T / kEncWarps), 65536 / kChunk16, H); stage one chunk of C_k and C_v.
// kSplit (few token-heads, e.g. the decode append): one token-head per CTA and its 8 warps split
// the chunk (128 centroids each); the K and V chunks are staged together (one barrier) and the
// last of the 64 chunk CTAs of a token-head finalises its codes (no separate finalize launch).
// Otherwise one token-head per warp scanning the whole chunk, finalised by encode_nn16_finalize.
__device__ __forceinline__ void finalize_token_head(const EncArgs& a, int64_t bt, int b, int t, int h, int lane);

template <bool kSplit>
__global__ void __launch_bounds__(kEncWarps * 32) encode_nn16_kernel(EncArgs a) {
  __shared__ uint4 sc[kSplit ? 2 * kChunk16 : kChunk16];   // per stream: kChunk16 / 2 pairs x 32 B
  __shared__ bool s_last;
  griddep_wait();
  const int h = blockIdx.z;
  const int j0 = blockIdx.y * kChunk16;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t bt = kSplit ? static_cast<int64_t>(blockIdx.x) : static_cast<int64_t>(blockIdx.x) * kEncWarps + warp;
  constexpr int kSpan = kSplit ? kChunk16 / kEncWarps : kChunk16;
  const int jw = kSplit ? warp * kSpan : 0;
  const bool live = bt < static_cast<int64_t>(a.B) * a.T;
  const int b = live ? static_cast<int>(bt / a.T) : 0, t = live ? static_cast<int>(bt % a.T) : 0;
  auto stage = [&](int which, uint4* dst) {   // centroid pairs (pinned_dist4_x2 layout)
    const int n_ent = 1 << (which ? a.vbits : a.kbits);
    if (j0 < n_ent) {
      const uint16_t* cb = which ? (a.cv + h * a.cv_hs) : (a.ck + h * a.ck_hs);
      for (int p = threadIdx.x; p < kChunk16 / 2; p += blockDim.x) stage_centroid_pair(cb, j0 + 2 * p, dst + 2 * p);
    }
  };
  if constexpr (kSplit) {
    stage(0, sc);
    stage(1, sc + kChunk16);
    __syncthreads();
  }
  for (int which = 0; which < 2; ++which) {
    const int bits = which ? a.vbits : a.kbits;
    const int n_ent = 1 << bits;
    const uint4* tab = sc;
    if constexpr (kSplit) {
      tab = sc + which * kChunk16;
    } else {
      __syncthreads();
      stage(which, sc);
      __syncthreads();
    }
    if (!live || j0 >= n_ent || bits != 16) continue;
    float x[4];
    if (which == 0) transform_key_lane(a, b, t, h, lane, x);
    else load_value_lane(a, b, t, h, lane, x);
    uint32_t bi;
    scan_pairs<kSpan>(tab + jw, x, bi);   // pairs of the warp's span (jw even)
    bi += jw;
    float best;
    {   // the pinned distance of the chosen centroid (exact: same per-element ops)
      const int pp = static_cast<int>(bi) & ~1;
      const float2 d = pinned_dist4_x2(x[0], x[1], x[2], x[3], tab[pp], tab[pp + 1]);
      best = (bi & 1) ? d.y : d.x;
    }
    const unsigned long long packed =
        (static_cast<unsigned long long>(__float_as_uint(best)) << 32) | static_cast<unsigned long long>(j0 + bi);
    atomicMin(a.ws + ((bt * a.H + h) * 2 + which) * 32 + lane, packed);
  }
  if constexpr (kSplit) {
    // the last chunk CTA of this token-head finalises it: counters start at 0xFFFFFFFF (the
    // per-call 0xFF fill), so arrival k sees k - 1 and the last one (k = gridDim.y - 1) sees
    // gridDim.y - 2
    uint32_t* cnt = reinterpret_cast<uint32_t*>(a.ws + static_cast<int64_t>(a.B) * a.T * a.H * 64);
    __syncthreads();   // every warp's atomicMin precedes thread 0's arrival
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = live && (atomicAdd(cnt + bt * a.H + h, 1u) + 2u == gridDim.y);
    }
    __syncthreads();
    if (!s_last || warp != 0) return;
    __threadfence();
    if (lane == 0) cnt[bt * a.H + h] = 0u;   // every arrival is in: the word is left zero on exit
    finalize_token_head(a, bt, b, t, h, lane);
  }
}

// finalize 16-bit codes (and encode the other stream if it is 4/8-bit)
template <int OBITS>
__device__ __forceinline__ void small_nn_global(const uint16_t* cb, const float (&x)[4], uint32_t& bi) {
  float best = __int_as_float(0x7f800000);
  bi = 0;
  for (int j = 0; j < (1 << OBITS); ++j) {
    const uint2 w = *reinterpret_cast<const uint2*>(cb + 4 * j);
    const float dd = pinned_dist4(x[0], x[1], x[2], x[3], __uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                                  __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
    if (dd < best) { best = dd; bi = j; }
  }
}

__device__ __forceinline__ void finalize_token_head(const EncArgs& a, int64_t bt, int b, int t, int h, int lane) {
  // consume the 16-bit minima first (zeroed even when the write row is invalid: the workspace is
  // left zero on exit; it may be part of a vecinfer_decode_step workspace that other calls lay out
  // differently)
  uint32_t code16[2] = {0u, 0u};
  for (int which = 0; which < 2; ++which) {
    if ((which ? a.vbits : a.kbits) != 16) continue;
    unsigned long long* slot = a.ws + ((bt * a.H + h) * 2 + which) * 32 + lane;
    code16[which] = static_cast<uint32_t>(__ldcg(slot) & 0xFFFFFFFFull);
    *slot = 0ull;
  }
  int64_t row;
  if (!cache_row(a, b, t, h, lane, row)) return;
  for (int which = 0; which < 2; ++which) {
    const int bits = which ? a.vbits : a.kbits;
    uint8_t* codes = which ? a.vcodes : a.kcodes;
    uint32_t code;
    if (bits == 16) {
      code = code16[which];
    } else {
      float x[4];
      if (which == 0) transform_key_lane(a, b, t, h, lane, x);
      else load_value_lane(a, b, t, h, lane, x);
      const uint16_t* cb = which ? (a.cv + h * a.cv_hs) : (a.ck + h * a.ck_hs);
      if (bits == 8) small_nn_global<8>(cb, x, code);
      else small_nn_global<4>(cb, x, code);
    }
    store_code(codes, bits, row, lane, code, a.nsub);
  }
}

__global__ void __launch_bounds__(kEncWarps * 32) encode_nn16_finalize(EncArgs a) {
  griddep_wait();
  const int h = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t bt = static_cast<int64_t>(blockIdx.x) * kEncWarps + (threadIdx.x >> 5);
  if (bt >= static_cast<int64_t>(a.B) * a.T) return;
  finalize_token_head(a, bt, static_cast<int>(bt / a.T), static_cast<int>(bt % a.T), h, lane);
}

// ------------------------------------------------------------------ NEXT-2 formats
// d8b8 / d8b12 / d4b10 / d2b8, D = 128.  One CTA of 256 threads
// per (token-head, K or V): warp 0 produces the row (key: the pinned smooth + integer FWHT above;
// value: raw) into shared memory; for each sub-vector m every thread scans centroids j = tid,
// tid + 256, ... with the pinned distance (fp32, RN, no FMA, summed left to right over the d
// dims: reading R9), minima travel as (dist_bits << 32 | j) -- dist >= 0, so the minimum is the
// nearest centroid with the lowest index on ties.  The codes are then packed into the row's
// little-endian bit string (code m in bits [m b, m b + b), reading R11).
constexpr int kGenThreads = 256;

__global__ void __launch_bounds__(kGenThreads) encode_generic_kernel(EncArgs a) {
  __shared__ __align__(16) float xs[128];
  __shared__ unsigned long long best[64];
  griddep_launch_dependents();
  const int which = blockIdx.z, h = blockIdx.y;
  const int64_t bt = blockIdx.x;
  const int b = static_cast<int>(bt / a.T), t = static_cast<int>(bt % a.T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = which ? a.vsub : a.ksub, bits = which ? a.vbits : a.kbits;
  const int M = 128 / sub, n_ent = 1 << bits;
  const uint16_t* cb = which ? (a.cv + h * a.cv_hs) : (a.ck + h * a.ck_hs);
  if (tid < 64) best[tid] = ~0ull;
  griddep_wait();
  int64_t row;
  if (!cache_row(a, b, t, h, lane, row)) return;   // uniform over the CTA
  if (warp == 0) {
    float x[4];
    if (which == 0) transform_key_lane(a, b, t, h, lane, x);
    else load_value_lane(a, b, t, h, lane, x);
    *reinterpret_cast<float4*>(xs + 4 * lane) = make_float4(x[0], x[1], x[2], x[3]);
  }
  __syncthreads();
  for (int m = 0; m < M; ++m) {
    const float* xm = xs + m * sub;
    unsigned long long key = ~0ull;
    for (int j = tid; j < n_ent; j += kGenThreads) {
      const uint16_t* c = cb + static_cast<int64_t>(j) * sub;
      float e = __fsub_rn(xm[0], __uint_as_float(static_cast<uint32_t>(c[0]) << 16));
      float dsum = __fmul_rn(e, e);
      for (int u = 1; u < sub; ++u) {
        e = __fsub_rn(xm[u], __uint_as_float(static_cast<uint32_t>(c[u]) << 16));
        dsum = __fadd_rn(dsum, __fmul_rn(e, e));
      }
      const unsigned long long k = (static_cast<unsigned long long>(__float_as_uint(dsum)) << 32) | static_cast<uint32_t>(j);
      key = k < key ? k : key;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
      key = o < key ? o : key;
    }
    if (lane == 0) atomicMin(&best[m], key);
  }
  __syncthreads();
  const int rb = M * bits / 8;
  uint8_t* dst = (which ? a.vcodes : a.kcodes) + row * rb;
  for (int i = tid; i < rb; i += kGenThreads) {   // byte i = row bits [8i, 8i + 8): <= 2 codes (b >= 8)
    const int p = 8 * i, c0 = p / bits, off = p - c0 * bits;
    uint32_t w = static_cast<uint32_t>(best[c0] & 0xFFFFFFFFull);
    if (c0 + 1 < M) w |= static_cast<uint32_t>(best[c0 + 1] & 0xFFFFFFFFull) << bits;
    dst[i] = static_cast<uint8_t>(w >> off);
  }
}

bool vq_d4(const vecinfer_vq_t& c) {
  return (c.head_dim == 128 || c.head_dim == 64) && c.sub_dim == 4 &&
         (c.code_bits == 4 || c.code_bits == 8 || c.code_bits == 16);
}
bool vq_next2(const vecinfer_vq_t& c) {
  return c.head_dim == 128 && ((c.sub_dim == 8 && (c.code_bits == 8 || c.code_bits == 12 || c.code_bits == 16)) ||
                               (c.sub_dim == 4 && c.code_bits == 10) || (c.sub_dim == 2 && c.code_bits == 8));
}
bool vq_supported(const vecinfer_vq_t& c) { return vq_d4(c) || vq_next2(c); }

}  // namespace
}  // namespace vecinfer

using namespace vecinfer;

extern "C" size_t vecinfer_encode_workspace_bytes(int32_t B, int32_t T, int32_t H_kv, vecinfer_vq_t kcfg,
                                                  vecinfer_vq_t vcfg) {
  if (B <= 0 || T <= 0 || H_kv <= 0) return 0;
  if (kcfg.code_bits != 16 && vcfg.code_bits != 16) return 0;
  // packed minima [B*T*H][2][32] u64, then one arrival counter per token-head (decode append path)
  return static_cast<size_t>(B) * T * H_kv * (2 * 32 * sizeof(unsigned long long) + sizeof(uint32_t));
}

static vecinfer_status_t encode_impl(const void* k_bf16, const void* v_bf16, int32_t B, int32_t T,
                                     int32_t H_kv, const int64_t k_strides[3], const int64_t v_strides[3],
                                     const float* inv_lambda, const void* ck_bf16, const void* cv_bf16,
                                     int64_t ck_head_stride, int64_t cv_head_stride, vecinfer_vq_t kcfg,
                                     vecinfer_vq_t vcfg, uint8_t* k_codes, uint8_t* v_codes, int64_t n_cap,
                                     const int32_t* write_pos, uint32_t* err_flags, void* workspace,
                                     size_t workspace_bytes, vecinfer_stream_t stream, const vecinfer_paged_t* pg) {
  if (!k_bf16 || !v_bf16 || !k_strides || !v_strides || !inv_lambda || !ck_bf16 || !cv_bf16 || !k_codes ||
      !v_codes || !write_pos)
    return fail(VECINFER_ERR_INVALID_ARG, "encode_kv: NULL pointer");
  if (B <= 0 || T <= 0 || H_kv <= 0 || n_cap <= 0) return fail(VECINFER_ERR_SHAPE, "encode_kv: non-positive size");
  if (!vq_supported(kcfg) || !vq_supported(vcfg))
    return fail(VECINFER_ERR_UNSUPPORTED, "encode_kv: supported configs are D in {64, 128} with d=4, code_bits in "
                "{4,8,16}, and D = 128 d8b8 / d8b12 / d4b10 / d2b8");
  if (kcfg.head_dim != vcfg.head_dim) return fail(VECINFER_ERR_SHAPE, "encode_kv: K and V head_dim differ");
  if (!aligned(k_bf16, 8) || !aligned(v_bf16, 8) || !aligned(inv_lambda, 16) || !aligned(ck_bf16, 8) ||
      !aligned(cv_bf16, 8) || !aligned(k_codes, 2) || !aligned(v_codes, 2))
    return fail(VECINFER_ERR_INVALID_ARG, "encode_kv: misaligned pointer (k/v/codebooks 8 B, inv_lambda 16 B)");
  for (int i = 0; i < 3; ++i)
    if (k_strides[i] % 4 != 0 || v_strides[i] % 4 != 0 || k_strides[i] < 0 || v_strides[i] < 0)
      return fail(VECINFER_ERR_INVALID_ARG, "encode_kv: strides must be non-negative multiples of 4 elements");
  if (ck_head_stride < 0 || cv_head_stride < 0 || ck_head_stride % 4 || cv_head_stride % 4)
    return fail(VECINFER_ERR_INVALID_ARG, "encode_kv: codebook head stride must be a non-negative multiple of 4");
  EncArgs a;
  a.k = static_cast<const uint16_t*>(k_bf16);
  a.v = static_cast<const uint16_t*>(v_bf16);
  a.B = B; a.T = T; a.H = H_kv;
  a.ks_b = k_strides[0]; a.ks_t = k_strides[1]; a.ks_h = k_strides[2];
  a.vs_b = v_strides[0]; a.vs_t = v_strides[1]; a.vs_h = v_strides[2];
  a.inv_lambda = inv_lambda;
  a.ck = static_cast<const uint16_t*>(ck_bf16);
  a.cv = static_cast<const uint16_t*>(cv_bf16);
  a.ck_hs = ck_head_stride; a.cv_hs = cv_head_stride;
  a.kbits = kcfg.code_bits; a.vbits = vcfg.code_bits;
  a.ksub = kcfg.sub_dim; a.vsub = vcfg.sub_dim;
  a.kcodes = k_codes; a.vcodes = v_codes;
  a.n_cap = n_cap; a.write_pos = write_pos; a.err = err_flags;
  a.bt = nullptr; a.bt_stride = 0; a.page_shift = 0; a.n_pages = 0;
  if (pg) {
    const vecinfer_status_t v = check_paged(pg, n_cap, "encode_kv");
    if (v != VECINFER_OK) return v;
    a.bt = pg->block_table; a.bt_stride = pg->bt_stride; a.n_pages = pg->n_pages;
    a.page_shift = __builtin_ctz(static_cast<unsigned>(pg->page_size));
  }
  a.inv_sqrt_d = static_cast<float>(1.0 / sqrt(static_cast<double>(kcfg.head_dim)));
  a.D = kcfg.head_dim;
  a.nsub = kcfg.head_dim / 4;
  a.ws = static_cast<unsigned long long*>(workspace);
  cudaStream_t st = as_stream(stream);
  const int64_t nbt = static_cast<int64_t>(B) * T;
  const int64_t gx = (nbt + kEncWarps - 1) / kEncWarps;
  if (gx > 2147483647) return fail(VECINFER_ERR_SHAPE, "encode_kv: too many tokens");
  if (H_kv > 65535) return fail(VECINFER_ERR_SHAPE, "encode_kv: too many heads");
  if (vq_next2(kcfg) || vq_next2(vcfg)) {   // one generic launch encodes both streams
    if (nbt > 2147483647) return fail(VECINFER_ERR_SHAPE, "encode_kv: too many tokens");
    const cudaError_t e = launch_pdl(encode_generic_kernel, dim3(static_cast<unsigned>(nbt), H_kv, 2),
                                     dim3(kGenThreads), 0, st, a);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(VECINFER_ERR_CUDA, "encode_generic_kernel: %s", cudaGetErrorString(e)); }
    return check_launch("encode_generic_kernel");
  }
  if (kcfg.code_bits == 16 || vcfg.code_bits == 16) {
    const size_t need = vecinfer_encode_workspace_bytes(B, T, H_kv, kcfg, vcfg);
    if (!workspace || workspace_bytes < need || !aligned(workspace, 8))
      return fail(VECINFER_ERR_WORKSPACE, "encode_kv: 16-bit codebooks need %zu bytes of workspace", need);
    // minima start at ~0 and the arrival counters at 0xFFFFFFFF; the kernels zero every word they
    // consume, and the finalize-kernel path (no counters) fills only the minima
    const size_t minima = static_cast<size_t>(B) * T * H_kv * 2 * 32 * sizeof(unsigned long long);
    if (cudaMemsetAsync(workspace, 0xFF, nbt * H_kv <= 4096 ? need : minima, st) != cudaSuccess)
      return check_launch("encode_kv memset");
    if (nbt * H_kv <= 4096) {   // decode append: the last chunk CTA of each token-head finalises it
      encode_nn16_kernel<true><<<dim3(static_cast<unsigned>(nbt), 65536 / kChunk16, H_kv), kEncWarps * 32, 0, st>>>(a);
      return check_launch("encode_nn16_kernel");
    }
    encode_nn16_kernel<false><<<dim3(static_cast<unsigned>(gx), 65536 / kChunk16, H_kv), kEncWarps * 32, 0, st>>>(a);
    vecinfer_status_t s = check_launch("encode_nn16_kernel");
    if (s != VECINFER_OK) return s;
    encode_nn16_finalize<<<dim3(static_cast<unsigned>(gx), H_kv), kEncWarps * 32, 0, st>>>(a);
    return check_launch("encode_nn16_finalize");
  }
  if (nbt * H_kv <= 4096) {   // decode append: centroid-split search, 16 warps per token-head
    dim3 g2(static_cast<unsigned>(nbt), H_kv);
    cudaError_t e;
    if (kcfg.code_bits == 8 && vcfg.code_bits == 8) e = launch_pdl(encode_append_kernel<8, 8>, g2, dim3(512), 0, st, a);
    else if (kcfg.code_bits == 4 && vcfg.code_bits == 4) e = launch_pdl(encode_append_kernel<4, 4>, g2, dim3(512), 0, st, a);
    else if (kcfg.code_bits == 8 && vcfg.code_bits == 4) e = launch_pdl(encode_append_kernel<8, 4>, g2, dim3(512), 0, st, a);
    else e = launch_pdl(encode_append_kernel<4, 8>, g2, dim3(512), 0, st, a);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(VECINFER_ERR_CUDA, "encode_append_kernel: %s", cudaGetErrorString(e)); }
    return check_launch("encode_append_kernel");
  }
  dim3 grid(static_cast<unsigned>(gx), H_kv);
  const dim3 blk(kEncWarps * 32);
  cudaError_t e;
  if (kcfg.code_bits == 8 && vcfg.code_bits == 8) e = launch_pdl(encode_small_kernel<8, 8>, grid, blk, 0, st, a);
  else if (kcfg.code_bits == 4 && vcfg.code_bits == 4) e = launch_pdl(encode_small_kernel<4, 4>, grid, blk, 0, st, a);
  else if (kcfg.code_bits == 8 && vcfg.code_bits == 4) e = launch_pdl(encode_small_kernel<8, 4>, grid, blk, 0, st, a);
  else e = launch_pdl(encode_small_kernel<4, 8>, grid, blk, 0, st, a);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(VECINFER_ERR_CUDA, "encode_small_kernel: %s", cudaGetErrorString(e)); }
  return check_launch("encode_small_kernel");
}

extern "C" vecinfer_status_t vecinfer_encode_kv(const void* k_bf16, const void* v_bf16, int32_t B, int32_t T,
                                                int32_t H_kv, const int64_t k_strides[3], const int64_t v_strides[3],
                                                const float* inv_lambda, const void* ck_bf16, const void* cv_bf16,
                                                int64_t ck_head_stride, int64_t cv_head_stride, vecinfer_vq_t kcfg,
                                                vecinfer_vq_t vcfg, uint8_t* k_codes, uint8_t* v_codes, int64_t n_cap,
                                                const int32_t* write_pos, uint32_t* err_flags, void* workspace,
                                                size_t workspace_bytes, vecinfer_stream_t stream) {
  return encode_impl(k_bf16, v_bf16, B, T, H_kv, k_strides, v_strides, inv_lambda, ck_bf16, cv_bf16, ck_head_stride,
                     cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, write_pos, err_flags, workspace,
                     workspace_bytes, stream, nullptr);
}

extern "C" vecinfer_status_t vecinfer_encode_kv_paged(const void* k_bf16, const void* v_bf16, int32_t B, int32_t T,
                                                      int32_t H_kv, const int64_t k_strides[3],
                                                      const int64_t v_strides[3], const float* inv_lambda,
                                                      const void* ck_bf16, const void* cv_bf16,
                                                      int64_t ck_head_stride, int64_t cv_head_stride,
                                                      vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                                      uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                                      uint32_t* err_flags, void* workspace, size_t workspace_bytes,
                                                      vecinfer_stream_t stream, const vecinfer_paged_t* paged) {
  if (!paged) return fail(VECINFER_ERR_INVALID_ARG, "encode_kv_paged: NULL paged descriptor");
  return encode_impl(k_bf16, v_bf16, B, T, H_kv, k_strides, v_strides, inv_lambda, ck_bf16, cv_bf16, ck_head_stride,
                     cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, write_pos, err_flags, workspace,
                     workspace_bytes, stream, paged);
}
