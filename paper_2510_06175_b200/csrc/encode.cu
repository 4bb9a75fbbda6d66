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
#include <type_traits>

#include "common.cuh"
#include "tc.cuh"

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
  int gen_mask;            // encode_generic_kernel: bit z = encode stream z (the filter does the others)
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


// ------------------------------------------------------------------ 16-bit: tensor-core filter
// Exact nearest-centroid search over a 65 536-entry book in two launches (decode append and bulk).
//
// Filter (nn16_filter_kernel, mma.sync bf16 -> fp32): with D_j = ||x - c_j||^2 = ||x||^2 + a_j,
// a_j = ||c_j||^2 - 2 x.c_j is a dense contraction over K = 16: A row (sub-vector x) =
// [-2x split into three bf16 parts (hi, mid, lo: exact, 24 bits) | 1, 1, 1 | 0], B column
// (centroid c, bf16-exact) = [c | c | c | ||c||^2 as three bf16 parts | 0].  Every product is
// exact; only the tensor core's fp32 accumulation rounds, by at most 17 * 2^-23 * S with
// S = sum |terms| <= 2.1 ||x||_1 max|c_i| + 1.01 max ||c||^2 (bounds per 512-centroid chunk).  For
// each (sub-vector, chunk) the filter stores lo = min_j~ a~_j - E and hi = min_j~ a~_j + E with
// E = 2^-17 S (4x the accumulation bound), so lo <= a_j for every j of the chunk and hi >= a_j of
// the chunk's approximate argmin.
//
// Selection (nn16_select_kernel): the pinned distance (fp32 RN, no FMA, reading R9) of any
// centroid is D_j (1 + delta), |delta| <= 7 * 2^-24.  U = min_k (||x||^2 + hi_k) (1 + 2^-19) + slack
// bounds the minimum pinned distance from above; a chunk can hold the pinned argmin only if
// (||x||^2 + lo_k) (1 - 2^-19) - slack <= U.  Every such chunk (usually one) is scanned with the
// exact pinned distance and the (dist_bits << 32 | index) minimum -- lowest index on ties -- is
// the code: bit-identical to the full scan, at ~1/100 of its ALU work.  The workspace entries are
// written by the filter and zeroed by the selection that consumes them.
constexpr int kNC16 = 128;          // chunks of the 65 536-entry book
constexpr int kCS16 = 512;          // centroids per chunk (64 n-tiles of 8)
constexpr int kFW16 = 8;            // warps per filter CTA: two m16 tiles (32 rows) each
constexpr int kRows16 = 32 * kFW16; // book rows per filter CTA

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}

__device__ __forceinline__ void mma_bf16_16816_acc(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                   uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bf16_bits_rn(float v) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));
}
// v = p0 + p1 + p2 exactly (three bf16 parts of an fp32 value)
__device__ __forceinline__ void split3_bf16(float v, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
  p0 = bf16_bits_rn(v);
  const float r1 = v - __uint_as_float(p0 << 16);
  p1 = bf16_bits_rn(r1);
  const float r2 = r1 - __uint_as_float(p1 << 16);
  p2 = bf16_bits_rn(r2);
}

// streams searched by the tensor-core filter: 65 536-entry d = 4 books and the d = 8 books of 4096 /
// 65 536 entries (NEXT-2 d8b12, d8b16)
__host__ __device__ __forceinline__ bool nn_filtered(int sub, int bits) {
  return (sub == 4 && bits == 16) || (sub == 8 && (bits == 12 || bits == 16));
}
// book z of the launch -> stream s (0 = K, 1 = V) and head hb (per-head books) / shared flag
__device__ __forceinline__ void nn16_book(const EncArgs& a, int z, int& s, int& hb, bool& shared) {
  const int nk = nn_filtered(a.ksub, a.kbits) ? (a.ck_hs ? a.H : 1) : 0;
  s = z < nk ? 0 : 1;
  hb = s == 0 ? z : z - nk;
  shared = (s == 0 ? a.ck_hs : a.cv_hs) == 0;
}

// workspace (float2 lo/hi) of sub-vector m, stream s, token-head (btl, h) of the pass
__device__ __forceinline__ int64_t nn16_ws_row(const EncArgs& a, int64_t btl, int h, int s, int m) {
  return (((btl * a.H + h) * 2 + s) * 32 + m) * kNC16;
}

// grid (max chunks / ncpb, row blocks, books); rows of book (s, hb): (token, [head,] sub-vector) of
// the pass.  A CTA filters its 256 rows against ncpb consecutive chunks: the rows' x and A fragments
// are built once, the chunks go through two shared fragment buffers (chunk c + 1 is staged -- its
// centroids prefetched into registers a chunk earlier -- while c is multiplied).
// DS = sub-vector dims: 4 (K = 16, one MMA per n-tile) or 8 (K = 32, two chained MMAs:
// [hi | mid] . [c | c] then [lo | 1 1 1 0 0 0 0 0] . [c | n0 n1 n2 0 0 0 0 0]).
template <int DS>
__global__ void __launch_bounds__(kFW16 * 32) nn16_filter_kernel(EncArgs a, int64_t bt0, int nbt_p, int ncpb) {
  extern __shared__ __align__(16) unsigned char fsm[];
  using Frag = typename std::conditional<DS == 4, uint2, uint4>::type;   // B fragment words of a lane
  Frag* sfrag = reinterpret_cast<Frag*>(fsm);                             // [2][64 n-tiles][32 lanes]
  float* sx = reinterpret_cast<float*>(fsm + 2 * (kCS16 / 8) * 32 * sizeof(Frag));   // [warps][32 rows][DS]
  float* sbnd = sx + kFW16 * 32 * DS;                                     // [2][warps][2]
  int s, hb;
  bool shared;
  nn16_book(a, blockIdx.z, s, hb, shared);
  const int nsub = a.D / DS;
  const int nch = (1 << (s ? a.vbits : a.kbits)) / kCS16;
  const int64_t rows = static_cast<int64_t>(nbt_p) * (shared ? a.H : 1) * nsub;
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * kRows16;
  const int chunk0 = blockIdx.x * ncpb;
  if (row0 >= rows || chunk0 >= nch) return;   // (per-head books: fewer rows; 4096-entry books: 8 chunks)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // centroids (static codebook) are loaded before the grid-dependency wait; column j of n-tile nt =
  // centroid chunk * 512 + 8 nt + j; lane (j, t) of the fragment holds k = 2t, 2t+1 | 2t+8, 2t+9
  const uint16_t* cbook = s == 0 ? a.ck + hb * a.ck_hs : a.cv + hb * a.cv_hs;
  constexpr int kPer = kCS16 / (kFW16 * 32);
  Frag cw[kPer];
  auto prefetch = [&](int chunk) {
#pragma unroll
    for (int q = 0; q < kPer; ++q)
      cw[q] = *reinterpret_cast<const Frag*>(cbook + (static_cast<int64_t>(chunk) * kCS16 + tid + kFW16 * 32 * q) * DS);
  };
  auto stage = [&](int buf) {
    float cmax = 0.f, nmax = 0.f;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = tid + kFW16 * 32 * q;
      uint32_t w[DS / 2];
      if constexpr (DS == 4) { w[0] = cw[q].x; w[1] = cw[q].y; }
      else { w[0] = cw[q].x; w[1] = cw[q].y; w[2] = cw[q].z; w[3] = cw[q].w; }
      float n = 0.f;
#pragma unroll
      for (int u = 0; u < DS / 2; ++u) {
        const float c0 = __uint_as_float(w[u] << 16), c1 = __uint_as_float(w[u] & 0xFFFF0000u);
        n = __fadd_rn(__fadd_rn(n, __fmul_rn(c0, c0)), __fmul_rn(c1, c1));
        cmax = fmaxf(cmax, fmaxf(fabsf(c0), fabsf(c1)));
      }
      uint32_t n0, n1, n2;
      split3_bf16(n, n0, n1, n2);
      nmax = fmaxf(nmax, n);
      Frag* f = sfrag + (buf * (kCS16 / 8) + (i >> 3)) * 32 + (i & 7) * 4;
      if constexpr (DS == 4) {
        f[0] = make_uint2(w[0], w[0]);                 // k 0,1 | 8,9   = c0 c1 | c0 c1
        f[1] = make_uint2(w[1], w[1]);                 // k 2,3 | 10,11 = c2 c3 | c2 c3
        f[2] = make_uint2(w[0], n0 | (n1 << 16));     // k 4,5 | 12,13 = c0 c1 | n0 n1
        f[3] = make_uint2(w[1], n2);                   // k 6,7 | 14,15 = c2 c3 | n2 0
      } else {   // lane t: first MMA (c pair t | c pair t), second MMA (c pair t | n parts)
        f[0] = make_uint4(w[0], w[0], w[0], n0 | (n1 << 16));
        f[1] = make_uint4(w[1], w[1], w[1], n2);
        f[2] = make_uint4(w[2], w[2], w[2], 0u);
        f[3] = make_uint4(w[3], w[3], w[3], 0u);
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
      nmax = fmaxf(nmax, __shfl_xor_sync(0xffffffffu, nmax, off));
    }
    if (lane == 0) { sbnd[(buf * kFW16 + warp) * 2] = cmax; sbnd[(buf * kFW16 + warp) * 2 + 1] = nmax; }
  };
  prefetch(chunk0);
  griddep_wait();   // k / v may come from the previous kernel; the workspace is reused across passes
  // x of the warp's 32 rows: the token-heads' transforms (lane l holds dims 4l..4l+3) -> sx rows
  const int64_t wr0 = row0 + 32 * warp;
  float* sxw = sx + warp * 32 * DS;
  for (int part = 0; part < 32 / nsub; ++part) {
    const int64_t rp = wr0 + part * nsub;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (rp < rows) {
      const int64_t th = rp / nsub;
      const int64_t btl = shared ? th / a.H : th;
      const int h = shared ? static_cast<int>(th % a.H) : hb;
      const int64_t bt = bt0 + btl;
      const int b = static_cast<int>(bt / a.T), tt = static_cast<int>(bt % a.T);
      if (s == 0) transform_key_lane(a, b, tt, h, lane, x);
      else load_value_lane(a, b, tt, h, lane, x);
    }
    if (lane < a.D / 4) {   // dims 4l.. of the token-head = row (4l) / DS, components (4l) % DS ..
      float* d = sxw + (part * nsub + (4 * lane) / DS) * DS + (4 * lane) % DS;
      d[0] = x[0]; d[1] = x[1]; d[2] = x[2]; d[3] = x[3];
    }
  }
  stage(0);
  if (ncpb > 1 && chunk0 + 1 < nch) prefetch(chunk0 + 1);
  __syncthreads();
  // A fragments of the two m16 tiles: row r0 = 16 mt + g, r1 = r0 + 8 (DS = 8: [mma][mt][4])
  constexpr int NM = DS == 4 ? 1 : 2;
  uint32_t af[NM][2][4];
  const uint32_t one = 0x3F80u;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const float* x0 = sxw + (16 * mt + g) * DS;
    const float* x1 = sxw + (16 * mt + g + 8) * DS;
    const int c = DS == 4 ? (t & 1) * 2 : 2 * t;   // components c, c + 1
    uint32_t h0[2], m0[2], l0[2], h1[2], m1[2], l1[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      split3_bf16(-2.f * x0[c + u], h0[u], m0[u], l0[u]);
      split3_bf16(-2.f * x1[c + u], h1[u], m1[u], l1[u]);
    }
    if constexpr (DS == 4) {
      if (t < 2) {   // k 2t, 2t+1 = hi parts; k 2t+8, 2t+9 = lo parts
        af[0][mt][0] = h0[0] | (h0[1] << 16); af[0][mt][1] = h1[0] | (h1[1] << 16);
        af[0][mt][2] = l0[0] | (l0[1] << 16); af[0][mt][3] = l1[0] | (l1[1] << 16);
      } else {       // k 2t = 4 + c: mid parts; k 12..15 = 1, 1, 1, 0
        af[0][mt][0] = m0[0] | (m0[1] << 16); af[0][mt][1] = m1[0] | (m1[1] << 16);
        af[0][mt][2] = t == 2 ? (one | (one << 16)) : one;
        af[0][mt][3] = af[0][mt][2];
      }
    } else {         // first MMA: k 2t.. = hi, k 2t+8.. = mid; second: k 2t.. = lo, k 8..15 = 1 1 1 0 ..
      af[0][mt][0] = h0[0] | (h0[1] << 16); af[0][mt][1] = h1[0] | (h1[1] << 16);
      af[0][mt][2] = m0[0] | (m0[1] << 16); af[0][mt][3] = m1[0] | (m1[1] << 16);
      af[NM - 1][mt][0] = l0[0] | (l0[1] << 16); af[NM - 1][mt][1] = l1[0] | (l1[1] << 16);
      af[NM - 1][mt][2] = t == 0 ? (one | (one << 16)) : t == 1 ? one : 0u;
      af[NM - 1][mt][3] = af[NM - 1][mt][2];
    }
  }
  const int nci = min(ncpb, nch - chunk0);
  for (int ci = 0; ci < nci; ++ci) {
    const int buf = ci & 1;
    float mn[2][2] = {{INFINITY, INFINITY}, {INFINITY, INFINITY}};
#pragma unroll 4
    for (int nt = 0; nt < kCS16 / 8; ++nt) {
      const Frag bf = sfrag[(buf * (kCS16 / 8) + nt) * 32 + lane];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        float d[4];
        if constexpr (DS == 4) {
          mma_bf16_16816(d, af[0][mt][0], af[0][mt][1], af[0][mt][2], af[0][mt][3], bf.x, bf.y);
        } else {
          mma_bf16_16816(d, af[0][mt][0], af[0][mt][1], af[0][mt][2], af[0][mt][3], bf.x, bf.y);
          mma_bf16_16816_acc(d, af[NM - 1][mt][0], af[NM - 1][mt][1], af[NM - 1][mt][2], af[NM - 1][mt][3], bf.z, bf.w);
        }
        mn[mt][0] = fminf(mn[mt][0], fminf(d[0], d[1]));
        mn[mt][1] = fminf(mn[mt][1], fminf(d[2], d[3]));
      }
    }
    float cm = 0.f, nm = 0.f;
#pragma unroll
    for (int w = 0; w < kFW16; ++w) { cm = fmaxf(cm, sbnd[(buf * kFW16 + w) * 2]); nm = fmaxf(nm, sbnd[(buf * kFW16 + w) * 2 + 1]); }
    const int chunk = chunk0 + ci;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float v = mn[mt][hf];
        v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 1));
        v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 2));
        const int rl = 16 * mt + g + 8 * hf;   // row of the warp
        const int64_t r = wr0 + rl;
        if (t != 0 || r >= rows) continue;
        const float* xx = sxw + rl * DS;
        float x1n = 0.f;
#pragma unroll
        for (int u = 0; u < DS; ++u) x1n += fabsf(xx[u]);
        // accumulation bound: DS = 4: 16 products, E = 4x; DS = 8: 32 chained, E = 4x (2^-16)
        const float E = (DS == 4 ? 0x1p-17f : 0x1p-16f) * (2.1f * x1n * cm + 1.01f * nm);
        const int m = static_cast<int>(r % nsub);
        const int64_t th = r / nsub;
        const int64_t btl = shared ? th / a.H : th;
        const int h = shared ? static_cast<int>(th % a.H) : hb;
        reinterpret_cast<float2*>(a.ws)[nn16_ws_row(a, btl, h, s, m) + chunk] = make_float2(v - E, v + E);
      }
    if (ci + 1 < nci) {   // stage chunk ci + 1 into the other buffer (last read in iteration ci - 1)
      stage(buf ^ 1);
      if (ci + 2 < nci) prefetch(chunk0 + ci + 2);
      __syncthreads();
    }
  }
}
template <int DS>
constexpr int nn_filter_smem() {
  return 2 * (kCS16 / 8) * 32 * (DS == 4 ? 8 : 16) + kFW16 * 32 * DS * 4 + 2 * kFW16 * 2 * 4;
}

// tcgen05 helpers of the warp-specialised filter variant below (M = 128 rows, K = 16, bf16 in, fp32 out)
constexpr int kTcRows = 128;                      // M
constexpr int kTcTile = kTcRows * 32;             // A tile bytes (128 x 16 bf16)
__device__ __forceinline__ void tc_mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(0u) : "memory");   // D = A.B^T (no accumulate)
}
__device__ __forceinline__ void sts_u128(uint32_t saddr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(saddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void tc_ld_32x32b_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
      "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr) : "memory");
}
// byte offset of (row r, 16-byte K group kg) in a K-major no-swizzle 128 x 16 tile: core matrices of
// 8 rows x 16 B, next 8 rows at +128 B (SBO), next K group at +2048 B (LBO)
__device__ __forceinline__ uint32_t tc_tile_off(int r, int kg) { return kg * 2048 + (r >> 3) * 128 + (r & 7) * 16; }

// Warp-specialised tcgen05 filter (opt-in VECINFER_NN16_TC=1; same arithmetic, error bound and
// workspace contract as nn16_filter_kernel): one CTA per SM (all 512 TMEM columns), 128 book rows as
// the A tile in shared memory (K-major, no swizzle, K = 16: [-2x hi | mid | lo | 1 1 1 0]); warp 0
// issues tcgen05.mma kind::f16 (bf16 in, fp32 out, N = 256 centroids [c | c | c | ||c||^2 parts | 0]
// per unit) into one of two 256-column TMEM accumulators, warps 1-3 stage B tiles into a 4-deep
// ring, warps 4-11 read D (TMEM lane quadrant w % 4 = their 32 rows, one half of the columns each,
// tcgen05.ld.32x32b.x64) and fold the minima with 3-input FMNMX.  Hand-offs are mbarriers only:
// bfull / bempty per B stage, dfull / dempty per accumulator.  Measured ~1.15x SLOWER than the
// mma.sync filter: reading the fp32 accumulator back out of TMEM (128 x 256 x 4 B per unit) caps the
// min-reduction near the mma.sync pipe's own rate (0.465 HMMA x 128 results per clk and SM), so the
// tensor-core speed-up has nothing to feed (profiles/r02/exp_nn16_filter.txt).
constexpr int kWsN = 256, kWsStages = 4;
constexpr int kWsBT = kWsN * 32;                           // B tile bytes (256 x 16 bf16)
constexpr int kWsSmem = 120 * 1024;                        // > 114 KiB: one CTA per SM
__device__ __forceinline__ uint32_t ws_btile_off(int r, int kg) { return kg * (kWsN * 16) + (r >> 3) * 128 + (r & 7) * 16; }
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
}

constexpr int kWsThreads = 384;   // warp 0 MMA, 1-3 stagers, 4-11 reducers (two per TMEM lane quadrant)
__global__ void __launch_bounds__(kWsThreads, 1) nn16_filter_ws_kernel(EncArgs a, int64_t bt0, int nbt_p, int ncpb) {
  extern __shared__ __align__(1024) unsigned char wsm[];
  // [0, 4K) A | [4K, 4K + 4 x 8K) B ring | barriers | TMEM slot | chunk bounds [ncpb][2]
  const uint32_t sA = smem_u32(wsm), sB = sA + kTcTile;
  unsigned char* misc = wsm + kTcTile + kWsStages * kWsBT;
  uint64_t* bfull = reinterpret_cast<uint64_t*>(misc);
  uint64_t* bempty = bfull + kWsStages;
  uint64_t* dfull = bempty + kWsStages;
  uint64_t* dempty = dfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);
  float* cbnd = reinterpret_cast<float*>(misc + 256);   // [ncpb][2]: max |c_i|, max ||c||^2 per chunk
  float* smin = cbnd + 64;                              // [128 rows]: column-half minima of a chunk
  int s, hb;
  bool shared;
  nn16_book(a, blockIdx.z, s, hb, shared);
  const int nsub = a.nsub;
  const int64_t rows = static_cast<int64_t>(nbt_p) * (shared ? a.H : 1) * nsub;
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * kTcRows;
  if (row0 >= rows) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk0 = blockIdx.x * ncpb, nunits = ncpb * (kCS16 / kWsN);
  const uint16_t* cbook = s == 0 ? a.ck + hb * a.ck_hs : a.cv + hb * a.cv_hs;
  const uint16_t* crange = cbook + static_cast<int64_t>(chunk0) * kCS16 * 4;
  if (warp == 0) tc::alloc(smem_u32(tmem_slot), 512);
  if (tid == 0) {
    for (int i = 0; i < kWsStages; ++i) { tc::mbar_init(smem_u32(bfull + i), 96); tc::mbar_init(smem_u32(bempty + i), 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(smem_u32(dfull + i), 1); tc::mbar_init(smem_u32(dempty + i), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // chunk bounds (static codebook), all threads, before the grid-dependency wait
  for (int ci = warp; ci < ncpb; ci += kWsThreads / 32) {
    float cm = 0.f, nm = 0.f;
    for (int j = lane; j < kCS16; j += 32) {
      const uint2 w = *reinterpret_cast<const uint2*>(crange + (static_cast<int64_t>(ci) * kCS16 + j) * 4);
      const float c0 = __uint_as_float(w.x << 16), c1 = __uint_as_float(w.x & 0xFFFF0000u);
      const float c2 = __uint_as_float(w.y << 16), c3 = __uint_as_float(w.y & 0xFFFF0000u);
      cm = fmaxf(cm, fmaxf(fmaxf(fabsf(c0), fabsf(c1)), fmaxf(fabsf(c2), fabsf(c3))));
      nm = fmaxf(nm, __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c0, c0), __fmul_rn(c1, c1)), __fmul_rn(c2, c2)), __fmul_rn(c3, c3)));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
      nm = fmaxf(nm, __shfl_xor_sync(0xffffffffu, nm, off));
    }
    if (lane == 0) { cbnd[2 * ci] = cm; cbnd[2 * ci + 1] = nm; }
  }
  griddep_wait();
  float x1n = 0.f;
  if (warp >= 4 && warp < 8) {   // first-half reducers: the row's x -> A row (row rt = 32 (warp - 4) + lane = TMEM lane)
    const int rw = warp - 4;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    const int64_t wr0 = row0 + 32 * rw;
    for (int part = 0; part < 32 / nsub; ++part) {
      if (wr0 + part * nsub >= rows) break;
      const int64_t th = (wr0 + part * nsub) / nsub;
      const int64_t btl = shared ? th / a.H : th;
      const int h = shared ? static_cast<int>(th % a.H) : hb;
      const int64_t bt = bt0 + btl;
      const int b = static_cast<int>(bt / a.T), tt = static_cast<int>(bt % a.T);
      float xx[4];
      if (s == 0) transform_key_lane(a, b, tt, h, lane, xx);
      else load_value_lane(a, b, tt, h, lane, xx);
      if ((lane >= part * nsub && lane < (part + 1) * nsub) || nsub == 32) {
        x[0] = xx[0]; x[1] = xx[1]; x[2] = xx[2]; x[3] = xx[3];
      }
    }
    uint32_t hi[4], mi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split3_bf16(-2.f * x[i], hi[i], mi[i], lo[i]);
    const int rt = 32 * rw + lane;
    sts_u128(sA + tc_tile_off(rt, 0), make_uint4(hi[0] | (hi[1] << 16), hi[2] | (hi[3] << 16),
                                                mi[0] | (mi[1] << 16), mi[2] | (mi[3] << 16)));
    sts_u128(sA + tc_tile_off(rt, 1), make_uint4(lo[0] | (lo[1] << 16), lo[2] | (lo[3] << 16), 0x3F803F80u, 0x00003F80u));
    x1n = fabsf(x[0]) + fabsf(x[1]) + fabsf(x[2]) + fabsf(x[3]);
    tc::fence_proxy_async_smem();
  }
  tc::fence_before();
  __syncthreads();   // A tile, chunk bounds, barriers and the TMEM address are ready
  tc::fence_after();
  const uint32_t tbase = *tmem_slot;
  if (warp == 0) {   // MMA issuer: the whole warp waits, lane 0 issues
    constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kWsN >> 3) << 17) |
                                (static_cast<uint32_t>(kTcRows >> 4) << 24);
    const uint64_t adesc = tc::smem_desc_kmajor(sA, 2048, 128);
    for (int u = 0; u < nunits; ++u) {
      const int st = u % kWsStages, d = u & 1;
      tc::mbar_wait(smem_u32(bfull + st), (u / kWsStages) & 1);
      tc::mbar_wait(smem_u32(dempty + d), ((u >> 1) & 1) ^ 1);
      tc::fence_after();
      if (lane == 0) {
        tc_mma_ss(tbase + d * kWsN, adesc, tc::smem_desc_kmajor(sB + st * kWsBT, kWsBT / 2, 128), kIdesc);
        tc::commit(smem_u32(bempty + st));
        tc::commit(smem_u32(dfull + d));
      }
      __syncwarp();
    }
  } else if (warp < 4) {   // stagers: centroid i = t, t + 96, t + 192 of each unit
    const int t = tid - 32;
    constexpr int kPer = (kWsN + 95) / 96;
    uint2 cw[kPer];
    auto fetch = [&](int u) {
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int i = t + 96 * q;
        cw[q] = (i < kWsN && u < nunits) ? *reinterpret_cast<const uint2*>(crange + (static_cast<int64_t>(u) * kWsN + i) * 4)
                                         : make_uint2(0u, 0u);
      }
    };
    fetch(0);
    for (int u = 0; u < nunits; ++u) {
      const int st = u % kWsStages;
      tc::mbar_wait(smem_u32(bempty + st), ((u / kWsStages) & 1) ^ 1);
      const uint32_t b = sB + st * kWsBT;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int i = t + 96 * q;
        if (i >= kWsN) continue;
        const uint2 w = cw[q];
        const float c0 = __uint_as_float(w.x << 16), c1 = __uint_as_float(w.x & 0xFFFF0000u);
        const float c2 = __uint_as_float(w.y << 16), c3 = __uint_as_float(w.y & 0xFFFF0000u);
        const float n = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c0, c0), __fmul_rn(c1, c1)), __fmul_rn(c2, c2)), __fmul_rn(c3, c3));
        uint32_t n0, n1, n2;
        split3_bf16(n, n0, n1, n2);
        sts_u128(b + ws_btile_off(i, 0), make_uint4(w.x, w.y, w.x, w.y));
        sts_u128(b + ws_btile_off(i, 1), make_uint4(w.x, w.y, n0 | (n1 << 16), n2));
      }
      fetch(u + 1);
      tc::fence_proxy_async_smem();
      mbar_arrive(smem_u32(bfull + st));
    }
  } else {   // reducers: warp w reads rows 32 ((w - 4) % 4) + lane (its TMEM lane quadrant), columns half (w - 4) / 4
    const int rw = (warp - 4) & 3, half = (warp - 4) >> 2, rt = 32 * rw + lane;
    const uint32_t tl = (static_cast<uint32_t>(32 * rw) << 16) + half * (kWsN / 2);
    // the first-half warp holds the row's ||x||_1 (x1n); the pair meets on named barrier 1 + rw
    float mn = INFINITY;
    for (int u = 0; u < nunits; ++u) {
      const int d = u & 1;
      tc::mbar_wait(smem_u32(dfull + d), (u >> 1) & 1);
      tc::fence_after();
      float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
      for (int hq = 0; hq < kWsN / 128; ++hq) {
        uint32_t v[64];
        tc_ld_32x32b_x64(tbase + tl + d * kWsN + 64 * hq, v);
        tc::wait_ld();
#pragma unroll
        for (int i = 0; i < 64; i += 8) {
          m4[0] = fminf(m4[0], fminf(__uint_as_float(v[i]), __uint_as_float(v[i + 1])));
          m4[1] = fminf(m4[1], fminf(__uint_as_float(v[i + 2]), __uint_as_float(v[i + 3])));
          m4[2] = fminf(m4[2], fminf(__uint_as_float(v[i + 4]), __uint_as_float(v[i + 5])));
          m4[3] = fminf(m4[3], fminf(__uint_as_float(v[i + 6]), __uint_as_float(v[i + 7])));
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(dempty + d));   // D[d] free for unit u + 2
      mn = fminf(mn, fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3])));
      if ((u & 1) == 1) {   // chunk u / 2 done: the second-half warp hands its minima to the first
        const int ci = u >> 1;
        if (half) smin[rt] = mn;
        tc::bar_sync(1 + rw, 64);
        if (!half) {
          const float v = fminf(mn, smin[rt]);
          const int64_t r = row0 + rt;
          if (r < rows) {
            const float E = 0x1p-17f * (2.1f * x1n * cbnd[2 * ci] + 1.01f * cbnd[2 * ci + 1]);
            const int m = static_cast<int>(r % nsub);
            const int64_t th = r / nsub;
            const int64_t btl = shared ? th / a.H : th;
            const int h = shared ? static_cast<int>(th % a.H) : hb;
            reinterpret_cast<float2*>(a.ws)[nn16_ws_row(a, btl, h, s, m) + chunk0 + ci] = make_float2(v - E, v + E);
          }
        }
        tc::bar_sync(1 + rw, 64);   // smin[rt] is read before the next chunk overwrites it
        mn = INFINITY;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tbase, 512);
}

// grid (pass token rows, H, 2 streams x 4 row groups), 8 warps: warp w of row group z selects and
// stores the 16-bit code of sub-vector m = 8 z + w (one memory round trip for the chunk bounds,
// one per scanned chunk: the chunk is copied into the warp's shared buffer with every cp.async of a
// lane in flight).  A 4/8-bit stream is encoded by warp 0 of its row group 0.
constexpr int kSelWarps = 8;
constexpr int kSelSmem = kSelWarps * kCS16 * 8;   // one 4 KiB chunk buffer per warp
__global__ void __launch_bounds__(kSelWarps * 32) nn16_select_kernel(EncArgs a, int64_t bt0) {
  __shared__ __align__(16) unsigned char sel_smem[kSelSmem];
  griddep_wait();
  const int64_t btl = blockIdx.x, bt = bt0 + btl;
  const int h = blockIdx.y, s = blockIdx.z >> 2, grp = blockIdx.z & 3;
  const int b = static_cast<int>(bt / a.T), t = static_cast<int>(bt % a.T);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsub = a.nsub;
  const int bits = s ? a.vbits : a.kbits;
  const uint16_t* cb = s ? a.cv + h * a.cv_hs : a.ck + h * a.ck_hs;
  const int m = kSelWarps * grp + warp;
  if (bits == 16 ? m >= nsub : (grp != 0 || warp != 0)) return;
  float x[4];
  if (s == 0) transform_key_lane(a, b, t, h, lane, x);
  else load_value_lane(a, b, t, h, lane, x);
  if (bits != 16) {   // 4/8-bit stream next to a 16-bit one: the shared-nothing small scan
    int64_t row;
    if (!cache_row(a, b, t, h, lane, row)) return;
    uint32_t code;
    if (bits == 8) small_nn_global<8>(cb, x, code);
    else small_nn_global<4>(cb, x, code);
    store_code(s ? a.vcodes : a.kcodes, bits, row, lane, code, nsub);
    return;
  }
  const uint32_t sbuf = smem_u32(sel_smem) + static_cast<uint32_t>(warp * kCS16 * 8);
  float xm[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) xm[i] = __shfl_sync(0xffffffffu, x[i], m);
  const float X2 = xm[0] * xm[0] + xm[1] * xm[1] + xm[2] * xm[2] + xm[3] * xm[3];
  const float slack = 0x1p-20f * X2;
  float2* pm = reinterpret_cast<float2*>(a.ws) + nn16_ws_row(a, btl, h, s, m);
  float2 lh[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) lh[i] = __ldcg(pm + lane + 32 * i);
#pragma unroll
  for (int i = 0; i < 4; ++i) __stcg(pm + lane + 32 * i, make_float2(0.f, 0.f));   // consumed
  float U = INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) U = fminf(U, (X2 + lh[i].y + slack) * (1.f + 0x1p-19f));
#pragma unroll
  for (int off = 16; off; off >>= 1) U = fminf(U, __shfl_xor_sync(0xffffffffu, U, off));
  unsigned selm[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) selm[i] = __ballot_sync(0xffffffffu, (X2 + lh[i].x - slack) * (1.f - 0x1p-19f) <= U);
  unsigned long long best = ~0ull;
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    unsigned sel = i == 0 ? selm[0] : i == 1 ? selm[1] : i == 2 ? selm[2] : selm[3];
    while (sel) {
      const int k = __ffs(sel) - 1 + 32 * i;
      sel &= sel - 1;
      const unsigned char* src = reinterpret_cast<const unsigned char*>(cb + static_cast<int64_t>(k) * kCS16 * 4);
#pragma unroll
      for (int q = 0; q < kCS16 * 8 / 16 / 32; ++q)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbuf + 16 * (lane + 32 * q)),
                     "l"(src + 16 * (lane + 32 * q)) : "memory");
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      __syncwarp();
#pragma unroll 4
      for (int q = 0; q < kCS16 / 32; ++q) {
        const float4 c = bf16x4_to_float4(lds_u64(sbuf + 8 * (32 * q + lane)));
        const float dd = pinned_dist4(xm[0], xm[1], xm[2], xm[3], c.x, c.y, c.z, c.w);
        const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(dd)) << 32) |
                                       static_cast<uint32_t>(k * kCS16 + 32 * q + lane);
        best = key < best ? key : best;
      }
      __syncwarp();   // the buffer is read before the next chunk's copies overwrite it
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
    best = o < best ? o : best;
  }
  int64_t row;
  if (!cache_row(a, b, t, h, lane, row)) return;
  if (lane == 0)   // 16-bit codes: sub-vector m is the little-endian u16 at byte 2m of the row
    reinterpret_cast<uint16_t*>((s ? a.vcodes : a.kcodes) + row * (nsub * 2))[m] = static_cast<uint16_t>(best & 0xFFFFull);
}

// d = 8 books (NEXT-2 d8b12 / d8b16): grid (pass token rows, H, 2 streams), 8 warps; warp w selects
// sub-vectors w and w + 8 (chunks of 512 x 16 B copied to the warp's 8 KiB buffer with cp.async),
// then the row's 16 codes are packed into its little-endian bit string (reading R11) and stored.
constexpr int kSel8Smem = 8 * kCS16 * 16;
__global__ void __launch_bounds__(256) nn_select8_kernel(EncArgs a, int64_t bt0) {
  extern __shared__ __align__(16) unsigned char s8m[];
  __shared__ uint32_t scode[16];
  griddep_wait();
  const int64_t btl = blockIdx.x, bt = bt0 + btl;
  const int h = blockIdx.y, s = blockIdx.z;
  const int sub = s ? a.vsub : a.ksub, bits = s ? a.vbits : a.kbits;
  if (!nn_filtered(sub, bits)) return;
  const int b = static_cast<int>(bt / a.T), t = static_cast<int>(bt % a.T);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint16_t* cb = s ? a.cv + h * a.cv_hs : a.ck + h * a.ck_hs;
  float x[4];
  if (s == 0) transform_key_lane(a, b, t, h, lane, x);
  else load_value_lane(a, b, t, h, lane, x);
  const uint32_t sbuf = smem_u32(s8m) + static_cast<uint32_t>(warp * kCS16 * 16);
  for (int m = warp; m < 16; m += 8) {
    float xm[8];   // dims 8m .. 8m + 7 = lanes 2m, 2m + 1
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      xm[i] = __shfl_sync(0xffffffffu, x[i], 2 * m);
      xm[4 + i] = __shfl_sync(0xffffffffu, x[i], 2 * m + 1);
    }
    float X2 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) X2 += xm[i] * xm[i];
    const float slack = 0x1p-20f * X2;
    float2* pm = reinterpret_cast<float2*>(a.ws) + nn16_ws_row(a, btl, h, s, m);
    const int nch = (1 << bits) / kCS16;
    float2 lh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) lh[i] = lane + 32 * i < nch ? __ldcg(pm + lane + 32 * i) : make_float2(INFINITY, INFINITY);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < nch) __stcg(pm + lane + 32 * i, make_float2(0.f, 0.f));   // consumed
    // pinned distance of d = 8: relative error <= 10 * 2^-24 -> (1 +- 2^-18) factors
    float U = INFINITY;
#pragma unroll
    for (int i = 0; i < 4; ++i) U = fminf(U, (X2 + lh[i].y + slack) * (1.f + 0x1p-18f));
#pragma unroll
    for (int off = 16; off; off >>= 1) U = fminf(U, __shfl_xor_sync(0xffffffffu, U, off));
    unsigned selm[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) selm[i] = __ballot_sync(0xffffffffu, (X2 + lh[i].x - slack) * (1.f - 0x1p-18f) <= U);
    unsigned long long best = ~0ull;
#pragma unroll 1
    for (int i = 0; i < 4; ++i) {
      unsigned sel = i == 0 ? selm[0] : i == 1 ? selm[1] : i == 2 ? selm[2] : selm[3];
      while (sel) {
        const int k = __ffs(sel) - 1 + 32 * i;
        sel &= sel - 1;
        const unsigned char* src = reinterpret_cast<const unsigned char*>(cb + static_cast<int64_t>(k) * kCS16 * 8);
#pragma unroll
        for (int q = 0; q < kCS16 * 16 / 16 / 32; ++q)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbuf + 16 * (lane + 32 * q)),
                       "l"(src + 16 * (lane + 32 * q)) : "memory");
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncwarp();
#pragma unroll 2
        for (int q = 0; q < kCS16 / 32; ++q) {
          const uint4 w = lds_u128(sbuf + 16 * (32 * q + lane));
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
          float dsum = 0.f;
#pragma unroll
          for (int u = 0; u < 4; ++u) {   // left to right over the 8 dims, fp32 RN, no FMA (R9)
            const float e0 = __fsub_rn(xm[2 * u], __uint_as_float(ww[u] << 16));
            const float e1 = __fsub_rn(xm[2 * u + 1], __uint_as_float(ww[u] & 0xFFFF0000u));
            dsum = u == 0 ? __fmul_rn(e0, e0) : __fadd_rn(dsum, __fmul_rn(e0, e0));
            dsum = __fadd_rn(dsum, __fmul_rn(e1, e1));
          }
          const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(dsum)) << 32) |
                                         static_cast<uint32_t>(k * kCS16 + 32 * q + lane);
          best = key < best ? key : best;
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
      best = o < best ? o : best;
    }
    if (lane == 0) scode[m] = static_cast<uint32_t>(best & 0xFFFFFFFFull);
  }
  __syncthreads();
  if (warp != 0) return;
  int64_t row;
  if (!cache_row(a, b, t, h, lane, row)) return;
  const int rb = 16 * bits / 8;
  uint8_t* dst = (s ? a.vcodes : a.kcodes) + row * rb;
  for (int i = lane; i < rb; i += 32) {   // byte i = row bits [8i, 8i + 8): <= 2 codes (b >= 8)
    const int p = 8 * i, c0 = p / bits, off = p - c0 * bits;
    uint32_t w = scode[c0];
    if (c0 + 1 < 16) w |= scode[c0 + 1] << bits;
    dst[i] = static_cast<uint8_t>(w >> off);
  }
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
constexpr int kGenGroups = 4;   // sub-vector groups per (token-head, stream): 16 / 32 / 64 sub-vectors -> 4 / 8 / 16 per CTA

__global__ void __launch_bounds__(kGenThreads) encode_generic_kernel(EncArgs a) {
  __shared__ __align__(16) float xs[128];
  __shared__ unsigned long long best[64];
  __shared__ uint4 sbook[512];
  griddep_launch_dependents();
  // grid z = stream x kGenGroups row groups: group g encodes sub-vectors [g M / G, (g + 1) M / G), a
  // whole number of bytes of the row's bit string for every format served here (8 x 10 bits = 10 B)
  const int which = blockIdx.z / kGenGroups, grp = blockIdx.z % kGenGroups, h = blockIdx.y;
  if (!((a.gen_mask >> which) & 1)) return;   // this stream goes through the tensor-core filter
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
  // books of <= 8 KiB (d8b8, d4b10, d2b8: the formats this kernel serves) are staged in shared memory
  const bool staged = n_ent * sub * 2 <= static_cast<int>(sizeof(sbook));
  if (staged)
    for (int i = tid; i < n_ent * sub / 8; i += kGenThreads) sbook[i] = reinterpret_cast<const uint4*>(cb)[i];
  __syncthreads();
  const uint16_t* book = staged ? reinterpret_cast<const uint16_t*>(sbook) : cb;
  // warp w owns sub-vectors m = w, w + 8, ...: its lanes scan centroids j = lane, lane + 32, ... and a
  // shuffle tree keeps the (dist_bits << 32 | j) minimum -- no cross-warp reduction per sub-vector
  const int mg0 = grp * M / kGenGroups, mg1 = (grp + 1) * M / kGenGroups;
  for (int m = mg0 + warp; m < mg1; m += kGenThreads / 32) {
    const float* xm = xs + m * sub;
    unsigned long long key = ~0ull;
    for (int j = lane; j < n_ent; j += 32) {
      const uint16_t* c = book + static_cast<int64_t>(j) * sub;
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
    if (lane == 0) best[m] = key;
  }
  __syncthreads();
  const int rb = M * bits / 8;
  uint8_t* dst = (which ? a.vcodes : a.kcodes) + row * rb;
  for (int i = mg0 * bits / 8 + tid; i < mg1 * bits / 8; i += kGenThreads) {   // byte i = row bits [8i, 8i + 8): <= 2 codes (b >= 8)
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

// token rows (b, t) per filter + selection pass: about 512 token-heads (32 MiB of workspace)
static int64_t nn16_pass_rows(int64_t nbt, int H) {
  int64_t p = 512 / (H > 0 ? H : 1);
  if (p < 1) p = 1;
  return nbt < p ? nbt : p;
}

static bool nn16_scan_from_env();
namespace vecinfer {
// kernel launches of one vecinfer_encode_kv call of B*T token rows (vecinfer_decode_step_launches)
int encode_launch_count(int64_t nbt, int H, const vecinfer_vq_t& k, const vecinfer_vq_t& v) {
  if (nbt <= 0) return 0;
  const bool kf = nn_filtered(k.sub_dim, k.code_bits), vf = nn_filtered(v.sub_dim, v.code_bits);
  const bool next2 = vq_next2(k) || vq_next2(v);
  if ((kf || vf) && !(!next2 && nn16_scan_from_env())) {
    const int64_t np = nn16_pass_rows(nbt, H);
    return static_cast<int>(2 * ((nbt + np - 1) / np)) + (next2 && !(kf && vf) ? 1 : 0);
  }
  if (k.code_bits == 16 || v.code_bits == 16) return nbt * H <= 4096 ? 1 : 2;   // (full-scan experiment)
  return 1;
}
}  // namespace vecinfer

extern "C" size_t vecinfer_encode_workspace_bytes(int32_t B, int32_t T, int32_t H_kv, vecinfer_vq_t kcfg,
                                                  vecinfer_vq_t vcfg) {
  if (B <= 0 || T <= 0 || H_kv <= 0) return 0;
  if (!nn_filtered(kcfg.sub_dim, kcfg.code_bits) && !nn_filtered(vcfg.sub_dim, vcfg.code_bits)) return 0;
  // tensor-core filter: (lo, hi) per (token-head, stream, sub-vector, 512-centroid chunk) of one
  // pass of nn16_pass_rows(...) token rows (fp32 pairs: 64 KiB per token-head)
  // (the full-scan experiment behind VECINFER_NN16_SCAN=1 needs B*T*H_kv*516 bytes: packed minima +
  // one arrival counter per token-head; it fails with VECINFER_ERR_WORKSPACE if this is smaller)
  return static_cast<size_t>(nn16_pass_rows(static_cast<int64_t>(B) * T, H_kv)) * H_kv * 2 * 32 * kNC16 * 2 * sizeof(float);
}

// VECINFER_NN16_SCAN=1: 16-bit codes by the full pinned scan (centroid-split CTAs) instead of the
// tensor-core filter (A/B experiments; same codes)
static bool nn16_scan_from_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VECINFER_NN16_SCAN");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// VECINFER_NN16_TC=1: the tcgen05 filter instead of the mma.sync one (A/B; same codes).  Measured
// slower (N2): mma.sync stays the default.
static bool nn16_hmma_from_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VECINFER_NN16_TC");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
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
  a.gen_mask = 3;
  const bool kfilt = nn_filtered(kcfg.sub_dim, kcfg.code_bits), vfilt = nn_filtered(vcfg.sub_dim, vcfg.code_bits);
  const bool next2 = vq_next2(kcfg) || vq_next2(vcfg);
  // 65 536-entry d = 4 books and the 4096 / 65 536-entry d = 8 books: tensor-core filter + exact
  // selection (two PDL launches per pass of ~512 token-heads); a NEXT-2 stream outside that set is
  // encoded by the generic scan (gen_mask), in its own launch
  const bool use_filter = (kfilt || vfilt) && !(!next2 && nn16_scan_from_env());
  if (use_filter) {
    const size_t need = vecinfer_encode_workspace_bytes(B, T, H_kv, kcfg, vcfg);
    if (!workspace || workspace_bytes < need || !aligned(workspace, 16))
      return fail(VECINFER_ERR_WORKSPACE, "encode_kv: 16-bit / d8 codebooks need %zu bytes of workspace", need);
    if (kcfg.head_dim != 128 && kcfg.head_dim != 64) return fail(VECINFER_ERR_UNSUPPORTED, "encode_kv: 16-bit head_dim");
    const int ds = kfilt ? kcfg.sub_dim : vcfg.sub_dim;   // (the filtered streams of a pair share d)
    static bool attr_done = false;   // benign race: idempotent attributes
    if (!attr_done) {
      cudaFuncSetAttribute(nn16_filter_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem);
      cudaFuncSetAttribute(nn16_filter_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, nn_filter_smem<4>());
      cudaFuncSetAttribute(nn16_filter_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, nn_filter_smem<8>());
      cudaFuncSetAttribute(nn_select8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSel8Smem);
      attr_done = true;
    }
    if (next2 && !(kfilt && vfilt)) {   // the other stream: the generic scan, one CTA per (token-head)
      a.gen_mask = kfilt ? 2 : 1;
      if (nbt > 2147483647) return fail(VECINFER_ERR_SHAPE, "encode_kv: too many tokens");
      const cudaError_t e = launch_pdl(encode_generic_kernel, dim3(static_cast<unsigned>(nbt), H_kv, 2 * kGenGroups),
                                       dim3(kGenThreads), 0, st, a);
      if (e != cudaSuccess) { cudaGetLastError(); return fail(VECINFER_ERR_CUDA, "encode_generic_kernel: %s", cudaGetErrorString(e)); }
    }
    const bool hmma = nn16_hmma_from_env() || ds == 8;   // (the tcgen05 variant covers d = 4)
    const int64_t np = nn16_pass_rows(nbt, H_kv);
    const int nbk = (kfilt ? (ck_head_stride ? H_kv : 1) : 0) + (vfilt ? (cv_head_stride ? H_kv : 1) : 0);
    const int maxch = (1 << ((kfilt ? kcfg.code_bits : 0) > (vfilt ? vcfg.code_bits : 0) ? kcfg.code_bits : vcfg.code_bits)) / kCS16;
    for (int64_t b0 = 0; b0 < nbt; b0 += np) {
      const int nb = static_cast<int>(nbt - b0 < np ? nbt - b0 : np);
      // rows of the largest book (shared books hold every head's rows)
      const int64_t rows = static_cast<int64_t>(nb) * H_kv * (kcfg.head_dim / ds);
      cudaError_t e;
      if (!hmma) {   // warp-specialised tcgen05 filter (VECINFER_NN16_TC=1): one CTA per SM
        const int64_t rblk = (rows + kTcRows - 1) / kTcRows;
        int ncpb = 16;
        while (ncpb > 1 && (kNC16 / ncpb) * rblk * nbk < device_sm_count()) ncpb >>= 1;
        const dim3 g1(kNC16 / ncpb, static_cast<unsigned>(rblk), static_cast<unsigned>(nbk));
        e = launch_pdl(nn16_filter_ws_kernel, g1, dim3(kWsThreads), kWsSmem, st, a, b0, nb, ncpb);
      } else {       // mma.sync filter (default)
        const int64_t rblk = (rows + kRows16 - 1) / kRows16;
        // chunks per CTA: amortise the rows' transform over up to 8 chunks while keeping >= ~4 CTAs per SM
        int ncpb = 8;
        while (ncpb > 1 && ((maxch + ncpb - 1) / ncpb) * rblk * nbk < 4 * device_sm_count()) ncpb >>= 1;
        const dim3 g1((maxch + ncpb - 1) / ncpb, static_cast<unsigned>(rblk), static_cast<unsigned>(nbk));
        e = ds == 4 ? launch_pdl(nn16_filter_kernel<4>, g1, dim3(kFW16 * 32), nn_filter_smem<4>(), st, a, b0, nb, ncpb)
                    : launch_pdl(nn16_filter_kernel<8>, g1, dim3(kFW16 * 32), nn_filter_smem<8>(), st, a, b0, nb, ncpb);
      }
      if (e == cudaSuccess)
        e = ds == 4 ? launch_pdl(nn16_select_kernel, dim3(static_cast<unsigned>(nb), H_kv, 8), dim3(kSelWarps * 32), 0, st, a, b0)
                    : launch_pdl(nn_select8_kernel, dim3(static_cast<unsigned>(nb), H_kv, 2), dim3(256), kSel8Smem, st, a, b0);
      if (e != cudaSuccess) { cudaGetLastError(); return fail(VECINFER_ERR_CUDA, "encode_kv (filter): %s", cudaGetErrorString(e)); }
    }
    return check_launch("encode_kv (filter)");
  }
  if (next2) {   // one generic launch encodes both streams
    if (nbt > 2147483647) return fail(VECINFER_ERR_SHAPE, "encode_kv: too many tokens");
    const cudaError_t e = launch_pdl(encode_generic_kernel, dim3(static_cast<unsigned>(nbt), H_kv, 2 * kGenGroups),
                                     dim3(kGenThreads), 0, st, a);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(VECINFER_ERR_CUDA, "encode_generic_kernel: %s", cudaGetErrorString(e)); }
    return check_launch("encode_generic_kernel");
  }
  if (kcfg.code_bits == 16 || vcfg.code_bits == 16) {   // VECINFER_NN16_SCAN=1: the full pinned scan
    const size_t need = static_cast<size_t>(B) * T * H_kv * (2 * 32 * sizeof(unsigned long long) + sizeof(uint32_t));
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
