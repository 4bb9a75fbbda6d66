// Shared pieces of the DEQUANT_MMA attention kernels (split kernel attn_mma.cu, stream kernel
// attn_stream.cu): code-width traits, codebook table fill, code-tile loads, and the centroid
// gathers that feed mma.sync directly.  See attn_mma.cu for the data layout.
#pragma once
#include "attn_common.cuh"

namespace vecinfer {

constexpr int kNW = 16;            // warps per CTA (1 CTA per SM)
constexpr int kThreads = kNW * 32;
constexpr float kTau = 8.0f;       // lazy-rescale threshold (log2 units): p <= 2^8
constexpr int kTab = 65536;        // [256 centroids][256 B] codebook table, 64 KiB-aligned

// bf16x4 centroid (global) -> fp16x4 MMA operand pair (exact for |c| in the fp16 normal range)
__device__ __forceinline__ uint2 bf16x4_to_f16x4(uint2 w) {
  uint2 e;
  e.x = pack_half2(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u));
  e.y = pack_half2(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
  return e;
}

// ---- code-width traits.  Per lane and token: the K chunk holds sub-vectors 8j..8j+7 (score MMA
// k-steps), the V chunk sub-vectors 4r..4r+3 (P.V m-tiles).  4/8-bit codebooks are gathered from the
// shared table (rows of 256 B: [16 K replicas | 16 V replicas]); 16-bit codebooks (65536 x 4 bf16 =
// 512 KiB) do not fit shared memory and are gathered from global memory (L2/L1 resident).
template <int BITS> struct Fmt;
// kSep: the format has its own shared table (1024 / 4096-entry NEXT-2 books) instead of a half
// of the classic 256-row [K | V] table
template <> struct Fmt<8> {
  static constexpr int kRow = 32, kOffK = 8, kOffV = 4;
  static constexpr bool kSmem = true, kGeneric = false, kWide = false, kSep = false;
  static __device__ __forceinline__ uint32_t lane_off(int lane) { return (lane & 15) * 8; }   // copy lane % 16
  using K = uint2;
  using V = uint32_t;
  static __device__ __forceinline__ K ldk(const uint8_t* p) { return ldg_nc_u64(p); }
  static __device__ __forceinline__ V ldv(const uint8_t* p) { return ldg_nc_u32(p); }
  static __device__ __forceinline__ K zk() { return make_uint2(0u, 0u); }
  // shared address of the centroid of code T of the chunk: code byte -> address bits 8..15 (PRMT)
  template <int T> static __device__ __forceinline__ uint32_t kaddr(const K& c, uint32_t base) {
    return prmt(T < 4 ? c.x : c.y, base, 0x7604u | ((T & 3) << 4));
  }
  template <int U> static __device__ __forceinline__ uint32_t vaddr(V c, uint32_t base) {
    return prmt(c, base, 0x7604u | (U << 4));
  }
};
template <> struct Fmt<4> {
  static constexpr int kRow = 16, kOffK = 4, kOffV = 2;
  static constexpr bool kSmem = true, kGeneric = false, kWide = false, kSep = false;
  static __device__ __forceinline__ uint32_t lane_off(int lane) { return (lane & 15) * 8; }
  using K = uint32_t;
  using V = uint32_t;   // low 16 bits
  static __device__ __forceinline__ K ldk(const uint8_t* p) { return ldg_nc_u32(p); }
  static __device__ __forceinline__ V ldv(const uint8_t* p) { return ldg_nc_u16(p); }
  static __device__ __forceinline__ K zk() { return 0u; }
  template <int T> static __device__ __forceinline__ uint32_t nib8(uint32_t w) {   // nibble T -> bits 8..11
    return T >= 2 ? ((w >> (4 * T - 8)) & 0xF00u) : ((w << (8 - 4 * T)) & 0xF00u);
  }
  template <int T> static __device__ __forceinline__ uint32_t kaddr(K c, uint32_t base) { return nib8<T>(c) | base; }
  template <int U> static __device__ __forceinline__ uint32_t vaddr(V c, uint32_t base) { return nib8<U>(c) | base; }
};
template <> struct Fmt<16> {
  static constexpr int kRow = 64, kOffK = 16, kOffV = 8;
  static constexpr bool kSmem = false, kGeneric = false, kWide = false, kSep = false;
  using K = uint4;
  using V = uint2;
  static __device__ __forceinline__ K ldk(const uint8_t* p) { return ldg_nc_u128(p); }
  static __device__ __forceinline__ V ldv(const uint8_t* p) { return ldg_nc_u64(p); }
  static __device__ __forceinline__ K zk() { return make_uint4(0u, 0u, 0u, 0u); }
  template <int T> static __device__ __forceinline__ uint32_t kidx(const K& c) {
    const uint32_t w = T < 2 ? c.x : T < 4 ? c.y : T < 6 ? c.z : c.w;
    return (T & 1) ? (w >> 16) : (w & 0xFFFFu);
  }
  template <int U> static __device__ __forceinline__ uint32_t vidx(const V& c) {
    const uint32_t w = U < 2 ? c.x : c.y;
    return (U & 1) ? (w >> 16) : (w & 0xFFFFu);
  }
};

// ---- the paper's other configurations (NEXT-2), D = 128: d-dim
// sub-vectors with b-bit codes, rows = one little-endian bit string (code m in bits [mb, mb+b),
// reading R11).  The kernels keep their 4-dim "virtual sub-vector" view (one gather = one MMA
// fragment pair): lane j's K chunk is dims 32j..32j+31 (32b/d bits at byte 4jb/d), lane r's V
// chunk dims 16r..16r+15.  Virtual sub-vector T of a chunk is half T&1 of code T/2 (d = 8), code T
// (d = 4) or codes 2T, 2T+1 (d = 2).  Codebooks (bf16, <= 64 KiB) are gathered from global memory
// through L1 like the 16-bit ones.  Format ids: d = 4 keeps id = b (4, 8, 16); else 100d + b.
template <int NB, int AL>
__device__ __forceinline__ void load_chunk(const uint8_t* p, uint32_t* w) {
  // NB bytes at an AL-aligned address -> little-endian words w[0..(NB+3)/4)
  if constexpr (AL >= 16 && NB == 16) {
    const uint4 v = ldg_nc_u128(p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else if constexpr (AL >= 8 && NB == 8) {
    const uint2 v = ldg_nc_u64(p);
    w[0] = v.x; w[1] = v.y;
  } else if constexpr (AL >= 4 && NB % 4 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 4; ++i) w[i] = ldg_ro_u32(p + 4 * i);
  } else if constexpr (AL >= 2 && NB % 2 == 0) {
#pragma unroll
    for (int i = 0; i < (NB + 3) / 4; ++i) w[i] = 0u;
#pragma unroll
    for (int i = 0; i < NB / 2; ++i) w[i >> 1] |= ldg_ro_u16(p + 2 * i) << (16 * (i & 1));
  } else {
#pragma unroll
    for (int i = 0; i < (NB + 3) / 4; ++i) w[i] = 0u;
#pragma unroll
    for (int i = 0; i < NB; ++i) w[i >> 2] |= ldg_ro_u8(p + i) << (8 * (i & 3));
  }
}

template <int SUB, int BITS>
struct FmtG {
  static constexpr int kRow = 128 / SUB * BITS / 8;        // bytes per cached row
  static constexpr int kOffK = 32 / SUB * BITS / 8;        // K chunk bytes (= lane stride)
  static constexpr int kOffV = 16 / SUB * BITS / 8;        // V chunk bytes
  static constexpr bool kSmem = false, kGeneric = true, kWide = false, kSep = false;
  static_assert(kOffV * 8 == 16 / SUB * BITS, "V chunk must be whole bytes");
  static constexpr int kRowAl = (kRow % 16 == 0) ? 16 : (kRow % 8 == 0) ? 8 : 4;
  static constexpr int gcd(int x, int y) { return y == 0 ? x : gcd(y, x % y); }
  struct K { uint32_t w[(kOffK + 3) / 4]; };
  struct V { uint32_t w[(kOffV + 3) / 4]; };
  static __device__ __forceinline__ K ldk(const uint8_t* p) {
    K c;
    load_chunk<kOffK, gcd(kOffK, kRowAl)>(p, c.w);
    return c;
  }
  static __device__ __forceinline__ V ldv(const uint8_t* p) {
    V c;
    load_chunk<kOffV, gcd(kOffV, kRowAl)>(p, c.w);
    return c;
  }
  static __device__ __forceinline__ K zk() { return K{}; }
  template <int I, int NW> static __device__ __forceinline__ uint32_t code(const uint32_t (&w)[NW]) {
    constexpr int p = I * BITS, wi = p / 32, sh = p % 32;
    uint32_t x = w[wi] >> sh;
    if constexpr (sh + BITS > 32) x |= w[wi + 1] << (32 - sh);
    return x & ((1u << BITS) - 1u);
  }
  // fp16x4 operand pair of virtual sub-vector T of a chunk (codebook cb: bf16 [2^b][SUB])
  template <int T, int NW> static __device__ __forceinline__ uint2 gather(const uint32_t (&w)[NW], const uint16_t* cb) {
    if constexpr (SUB == 8) {
      return bf16x4_to_f16x4(ldg_ro_u64(cb + 8 * code<T / 2>(w) + 4 * (T & 1)));
    } else if constexpr (SUB == 4) {
      return bf16x4_to_f16x4(ldg_ro_u64(cb + 4 * code<T>(w)));
    } else {
      return bf16x4_to_f16x4(make_uint2(ldg_ro_u32(cb + 2 * code<2 * T>(w)), ldg_ro_u32(cb + 2 * code<2 * T + 1>(w))));
    }
  }
};
constexpr int kFmtD8B8 = 808, kFmtD8B12 = 812, kFmtD4B10 = 410, kFmtD2B8 = 208, kFmtD8B16 = 816;
// d8b12 and d4b10 read their books from their own shared tables (one per stream, 64 KiB each), not
// through L1: d8b12 = 4096 x 16-byte fp16 centroids, unreplicated, one LDS.128 per code = two
// virtual sub-vectors ("wide", as d8b8); d4b10 = 1024 x 8-byte centroids in 8 replicas (rows of
// 64 B, lane l reads replica l % 8).  kSepShift = log2 row pitch, kSepReps = replicas.
template <> struct Fmt<kFmtD8B12> : FmtG<8, 12> {
  static constexpr bool kSmem = true, kGeneric = false, kWide = true, kSep = true;
  static constexpr int kSepShift = 4, kSepReps = 1, kSepEnt = 4096, kSepCent = 16;
  static __device__ __forceinline__ uint32_t sep_lane_off(int) { return 0u; }
  template <int I> static __device__ __forceinline__ uint32_t kaddr(const K& c, uint32_t base) {
    return base + (code<I>(c.w) << 4);
  }
  template <int I> static __device__ __forceinline__ uint32_t vaddr(const V& c, uint32_t base) {
    return base + (code<I>(c.w) << 4);
  }
};
template <> struct Fmt<kFmtD4B10> : FmtG<4, 10> {
  static constexpr bool kSmem = true, kGeneric = false, kWide = false, kSep = true;
  static constexpr int kSepShift = 6, kSepReps = 8, kSepEnt = 1024, kSepCent = 8;
  static __device__ __forceinline__ uint32_t sep_lane_off(int lane) { return (lane & 7) * 8; }
  template <int T> static __device__ __forceinline__ uint32_t kaddr(const K& c, uint32_t base) {
    return base + (code<T>(c.w) << 6);
  }
  template <int U> static __device__ __forceinline__ uint32_t vaddr(const V& c, uint32_t base) {
    return base + (code<U>(c.w) << 6);
  }
};
// d8b16 (Table 5's 2-bit row): 65 536 eight-dim centroids = 1 MiB bf16 per book, far
// beyond shared memory, gathered through L1/L2 like b4d4 (larger books cost efficiency)
template <> struct Fmt<kFmtD8B16> : FmtG<8, 16> {};
// 256-entry books live in the shared table like b2d4 (code byte -> address bits 8..15, rows of
// 256 B = [K half | V half]).  d8b8: the 16-byte centroid in 8 copies per half (lane l reads copy
// l % 8: one LDS.128 per quarter-warp phase hits 8 distinct 16-byte bank groups) and one 16-byte
// gather feeds two virtual sub-vectors ("wide").  d2b8: the 4-byte centroid in 32 copies per half
// (one LDS.32 per lane, all 32 banks); a virtual sub-vector is two gathers.
template <> struct Fmt<kFmtD8B8> {
  static constexpr int kRow = 16, kOffK = 4, kOffV = 2;   // K chunk: codes 4j..4j+3, V: 2r, 2r+1
  static constexpr bool kSmem = true, kGeneric = false, kWide = true, kSep = false;
  static __device__ __forceinline__ uint32_t lane_off(int lane) { return (lane & 7) * 16; }
  using K = uint32_t;
  using V = uint32_t;   // low 16 bits
  static __device__ __forceinline__ K ldk(const uint8_t* p) { return ldg_nc_u32(p); }
  static __device__ __forceinline__ V ldv(const uint8_t* p) { return ldg_nc_u16(p); }
  static __device__ __forceinline__ K zk() { return 0u; }
  template <int I> static __device__ __forceinline__ uint32_t kaddr(K c, uint32_t base) {
    return prmt(c, base, 0x7604u | (I << 4));
  }
  template <int I> static __device__ __forceinline__ uint32_t vaddr(V c, uint32_t base) {
    return prmt(c, base, 0x7604u | (I << 4));
  }
};
template <> struct Fmt<kFmtD2B8> {
  static constexpr int kRow = 64, kOffK = 16, kOffV = 8;  // K chunk: codes 16j..16j+15, V: 8r..8r+7
  static constexpr bool kSmem = true, kGeneric = false, kWide = false, kSep = false;
  static __device__ __forceinline__ uint32_t lane_off(int lane) { return lane * 4; }
  using K = uint4;
  using V = uint2;
  static __device__ __forceinline__ K ldk(const uint8_t* p) { return ldg_nc_u128(p); }
  static __device__ __forceinline__ V ldv(const uint8_t* p) { return ldg_nc_u64(p); }
  static __device__ __forceinline__ K zk() { return make_uint4(0u, 0u, 0u, 0u); }
  template <int I> static __device__ __forceinline__ uint32_t byte_addr(uint32_t w, uint32_t base) {
    return prmt(w, base, 0x7604u | ((I & 3) << 4));
  }
  template <int T> static __device__ __forceinline__ uint2 gk(const K& c, uint32_t base) {
    const uint32_t w = T < 2 ? c.x : T < 4 ? c.y : T < 6 ? c.z : c.w;   // codes 2T, 2T+1
    return make_uint2(lds_u32(byte_addr<2 * T>(w, base)), lds_u32(byte_addr<2 * T + 1>(w, base)));
  }
  template <int U> static __device__ __forceinline__ uint2 gv(const V& c, uint32_t base) {
    const uint32_t w = U < 2 ? c.x : c.y;
    return make_uint2(lds_u32(byte_addr<2 * U>(w, base)), lds_u32(byte_addr<2 * U + 1>(w, base)));
  }
};

template <int BITS> using KCode = typename Fmt<BITS>::K;
template <int BITS> using VCode = typename Fmt<BITS>::V;

// head-dim variants of the traits: D = 128 is Fmt<BITS>; D = 64 (16 sub-vectors, NEXT-4) keeps the
// register types and gather selectors but halves the row and the per-lane chunks: lane j's K chunk
// is sub-vectors 4j..4j+3 (4 score k-steps), lane r's V chunk sub-vectors 2r, 2r+1 (4 m-tiles).
template <int BITS, int DH> struct FmtD : Fmt<BITS> {};
template <> struct FmtD<8, 64> : Fmt<8> {
  static constexpr int kRow = 16, kOffK = 4, kOffV = 2;
  static __device__ __forceinline__ uint2 ldk(const uint8_t* p) { return make_uint2(ldg_nc_u32(p), 0u); }
  static __device__ __forceinline__ uint32_t ldv(const uint8_t* p) { return ldg_nc_u16(p); }
};
template <> struct FmtD<4, 64> : Fmt<4> {
  static constexpr int kRow = 8, kOffK = 2, kOffV = 1;
  static __device__ __forceinline__ uint32_t ldk(const uint8_t* p) { return ldg_nc_u16(p); }
  static __device__ __forceinline__ uint32_t ldv(const uint8_t* p) { return ldg_nc_u8(p); }
};
template <> struct FmtD<16, 64> : Fmt<16> {
  static constexpr int kRow = 32, kOffK = 8, kOffV = 4;
  static __device__ __forceinline__ uint4 ldk(const uint8_t* p) {
    const uint2 w = ldg_nc_u64(p);
    return make_uint4(w.x, w.y, 0u, 0u);
  }
  static __device__ __forceinline__ uint2 ldv(const uint8_t* p) { return make_uint2(ldg_nc_u32(p), 0u); }
};


template <int KB, int T>
__device__ __forceinline__ uint2 gather_k(const KCode<KB>& c, uint32_t kbase, const uint16_t* cbk) {
  if constexpr (KB == kFmtD2B8) return Fmt<KB>::template gk<T>(c, kbase);
  else if constexpr (Fmt<KB>::kSmem) return lds_u64(Fmt<KB>::template kaddr<T>(c, kbase));
  else if constexpr (Fmt<KB>::kGeneric) return Fmt<KB>::template gather<T>(c.w, cbk);
  else return bf16x4_to_f16x4(ldg_ro_u64(cbk + 4 * Fmt<KB>::template kidx<T>(c)));
}
template <int VB, int U>
__device__ __forceinline__ uint2 gather_v(const VCode<VB>& c, uint32_t vbase, const uint16_t* cbv) {
  if constexpr (VB == kFmtD2B8) return Fmt<VB>::template gv<U>(c, vbase);
  else if constexpr (Fmt<VB>::kSmem) return lds_u64(Fmt<VB>::template vaddr<U>(c, vbase));
  else if constexpr (Fmt<VB>::kGeneric) return Fmt<VB>::template gather<U>(c.w, cbv);
  else return bf16x4_to_f16x4(ldg_ro_u64(cbv + 4 * Fmt<VB>::template vidx<U>(c)));
}

// entries of a format's shared-table half (0: no shared table) and the 16-byte store pattern of
// centroid j (fp16): d = 4 -> the 8-byte centroid twice, d8b8 -> the 16-byte centroid, d2b8 -> the
// 4-byte centroid four times; 8 such stores fill the 128-byte half-row
template <int F> constexpr int smem_entries() {
  return F == 4 ? 16 : (F == 8 || F == kFmtD8B8 || F == kFmtD2B8) ? 256 : 0;
}
template <int F>
__device__ __forceinline__ uint4 table_pattern(const uint16_t* cb, int j) {
  if constexpr (F == kFmtD8B8) {
    const uint2 lo = bf16x4_to_f16x4(*reinterpret_cast<const uint2*>(cb + 8 * j));
    const uint2 hi = bf16x4_to_f16x4(*reinterpret_cast<const uint2*>(cb + 8 * j + 4));
    return make_uint4(lo.x, lo.y, hi.x, hi.y);
  } else if constexpr (F == kFmtD2B8) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(cb + 2 * j);
    const uint32_t h = pack_half2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
    return make_uint4(h, h, h, h);
  } else {
    const uint2 e = bf16x4_to_f16x4(*reinterpret_cast<const uint2*>(cb + 4 * j));
    return make_uint4(e.x, e.y, e.x, e.y);
  }
}

template <int F>
__device__ __forceinline__ uint32_t table_lane_off(int lane) {
  if constexpr (Fmt<F>::kSep) return Fmt<F>::sep_lane_off(lane);
  else if constexpr (Fmt<F>::kSmem) return Fmt<F>::lane_off(lane);
  else return 0u;
}

// fill of a separate (NEXT-2) table: centroid j (bf16, kSepCent / 2 dims) -> fp16 at row j, in
// kSepReps replicas; 16-byte stores, all threads of the CTA
template <int F>
__device__ __forceinline__ void sep_fill(unsigned char* tab, const uint16_t* cb, int tid, int nthreads) {
  if constexpr (Fmt<F>::kSep) {
    constexpr int kEnt = Fmt<F>::kSepEnt, kReps = Fmt<F>::kSepReps, kPitch = 1 << Fmt<F>::kSepShift;
    if constexpr (Fmt<F>::kSepCent == 16) {
      for (int j = tid; j < kEnt; j += nthreads) {
        const uint2 lo = bf16x4_to_f16x4(*reinterpret_cast<const uint2*>(cb + 8 * j));
        const uint2 hi = bf16x4_to_f16x4(*reinterpret_cast<const uint2*>(cb + 8 * j + 4));
        *reinterpret_cast<uint4*>(tab + j * kPitch) = make_uint4(lo.x, lo.y, hi.x, hi.y);
      }
    } else {   // 8-byte centroids, kReps replicas = kReps / 2 stores of the centroid pair
      for (int i = tid; i < kEnt * (kReps / 2); i += nthreads) {
        const int j = i / (kReps / 2), u = i % (kReps / 2);
        const uint2 e = bf16x4_to_f16x4(*reinterpret_cast<const uint2*>(cb + 4 * j));
        *reinterpret_cast<uint4*>(tab + j * kPitch + 16 * u) = make_uint4(e.x, e.y, e.x, e.y);
      }
    }
  }
}

// codebook table fill in two halves, so the codebook loads can be issued first (raw bf16 words,
// before the grid-dependency wait) and converted + stored to shared memory later: thread t owns
// centroid j = t/2 of C_k (t even) or C_v (t odd)
template <int F>
__device__ __forceinline__ uint4 table_raw(const uint16_t* cb, int j) {
  if constexpr (F == kFmtD8B8) {
    const uint2 lo = *reinterpret_cast<const uint2*>(cb + 8 * j), hi = *reinterpret_cast<const uint2*>(cb + 8 * j + 4);
    return make_uint4(lo.x, lo.y, hi.x, hi.y);
  } else if constexpr (F == kFmtD2B8) {
    return make_uint4(*reinterpret_cast<const uint32_t*>(cb + 2 * j), 0u, 0u, 0u);
  } else {
    const uint2 w = *reinterpret_cast<const uint2*>(cb + 4 * j);
    return make_uint4(w.x, w.y, 0u, 0u);
  }
}
template <int F>
__device__ __forceinline__ uint4 table_cvt(const uint4 raw) {   // raw bf16 words -> the store pattern
  if constexpr (F == kFmtD8B8) {
    const uint2 lo = bf16x4_to_f16x4(make_uint2(raw.x, raw.y)), hi = bf16x4_to_f16x4(make_uint2(raw.z, raw.w));
    return make_uint4(lo.x, lo.y, hi.x, hi.y);
  } else if constexpr (F == kFmtD2B8) {
    const uint32_t h = pack_half2(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u));
    return make_uint4(h, h, h, h);
  } else {
    const uint2 e = bf16x4_to_f16x4(make_uint2(raw.x, raw.y));
    return make_uint4(e.x, e.y, e.x, e.y);
  }
}
template <int KB, int VB>
__device__ __forceinline__ uint4 table_load(const uint16_t* ck, const uint16_t* cv, int tid) {
  const int j = tid >> 1, which = tid & 1;
  const int n = which ? smem_entries<VB>() : smem_entries<KB>();
  if (j >= n) return make_uint4(0u, 0u, 0u, 0u);
  return which ? table_raw<VB>(cv, j) : table_raw<KB>(ck, j);
}
template <int KB, int VB>
__device__ __forceinline__ void table_store(unsigned char* tab, uint4 raw, int tid) {
  // 8 x 16-byte stores per half-row, rotated so that the 8 threads of a quarter-warp hit 8
  // different bank groups.  The empty asm pins the conversion after this point (the compiler would
  // otherwise hoist it -- and the wait for the codebook loads -- above the grid-dependency wait).
  asm volatile("" : "+r"(raw.x), "+r"(raw.y), "+r"(raw.z), "+r"(raw.w));
  const int j = tid >> 1, which = tid & 1;
  const int n = which ? smem_entries<VB>() : smem_entries<KB>();
  if (j >= n) return;
  const uint4 v = which ? table_cvt<VB>(raw) : table_cvt<KB>(raw);
  unsigned char* row = tab + j * 256 + which * 128;
#pragma unroll
  for (int u0 = 0; u0 < 8; ++u0) {
    const int u = (u0 + tid) & 7;
    *reinterpret_cast<uint4*>(row + 16 * u) = v;
  }
}
template <int KB, int VB>
__device__ __forceinline__ void fill_tables(unsigned char* tab, const uint16_t* ck, const uint16_t* cv, int tid) {
  table_store<KB, VB>(tab, table_load<KB, VB>(ck, cv, tid), tid);
}

template <int KB, int VB>
struct TileCodes {
  KCode<KB> k[2][2];  // [sub-tile][row r / r+8]
  VCode<VB> v[2][4];  // [sub-tile][token 2j, 2j+1, 2j+8, 2j+9]
};

// kp/vp point at this lane's bytes of token (tile start + r) / (tile start + 2j) respectively
template <int KB, int VB, int DH = 128>
__device__ __forceinline__ void load_tile_full(TileCodes<KB, VB>& tc, const uint8_t* kp, const uint8_t* vp) {
  using FK = FmtD<KB, DH>;
  using FV = FmtD<VB, DH>;
  constexpr int KR = FK::kRow, VR = FV::kRow;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    tc.k[q][0] = FK::ldk(kp + (16 * q) * KR);
    tc.k[q][1] = FK::ldk(kp + (16 * q + 8) * KR);
    tc.v[q][0] = FV::ldv(vp + (16 * q) * VR);
    tc.v[q][1] = FV::ldv(vp + (16 * q + 1) * VR);
    tc.v[q][2] = FV::ldv(vp + (16 * q + 8) * VR);
    tc.v[q][3] = FV::ldv(vp + (16 * q + 9) * VR);
  }
}

// ragged last tile: rem = tokens left in the split (1..31), rows beyond it read as code 0
template <int KB, int VB, int DH = 128>
__device__ __forceinline__ void load_tile_tail(TileCodes<KB, VB>& tc, const uint8_t* kp, const uint8_t* vp, int rem,
                                               int r, int j) {
  using FK = FmtD<KB, DH>;
  using FV = FmtD<VB, DH>;
  constexpr int KR = FK::kRow, VR = FV::kRow;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    tc.k[q][0] = (16 * q + r < rem) ? FK::ldk(kp + (16 * q) * KR) : Fmt<KB>::zk();
    tc.k[q][1] = (16 * q + r + 8 < rem) ? FK::ldk(kp + (16 * q + 8) * KR) : Fmt<KB>::zk();
    const int t0 = 16 * q + 2 * j;
    tc.v[q][0] = (t0 < rem) ? FV::ldv(vp + (16 * q) * VR) : VCode<VB>{};
    tc.v[q][1] = (t0 + 1 < rem) ? FV::ldv(vp + (16 * q + 1) * VR) : VCode<VB>{};
    tc.v[q][2] = (t0 + 8 < rem) ? FV::ldv(vp + (16 * q + 8) * VR) : VCode<VB>{};
    tc.v[q][3] = (t0 + 9 < rem) ? FV::ldv(vp + (16 * q + 9) * VR) : VCode<VB>{};
  }
}

// one 16-token sub-tile Q of a tile from its own row base (paged caches: the two sub-tiles of a
// tile may lie in different pages).  kq points at this lane's K bytes of the sub-tile's row r, vq at
// its V bytes of row 2j; rem = tokens left from the sub-tile start (rows beyond read as code 0)
template <int KB, int VB, int Q>
__device__ __forceinline__ void load_subtile(TileCodes<KB, VB>& tc, const uint8_t* kq, const uint8_t* vq, int rem,
                                             int r, int j) {
  constexpr int KR = Fmt<KB>::kRow, VR = Fmt<VB>::kRow;
  if (rem >= 16) {   // full sub-tile: unpredicated loads
    tc.k[Q][0] = Fmt<KB>::ldk(kq);
    tc.k[Q][1] = Fmt<KB>::ldk(kq + 8 * KR);
    tc.v[Q][0] = Fmt<VB>::ldv(vq);
    tc.v[Q][1] = Fmt<VB>::ldv(vq + VR);
    tc.v[Q][2] = Fmt<VB>::ldv(vq + 8 * VR);
    tc.v[Q][3] = Fmt<VB>::ldv(vq + 9 * VR);
    return;
  }
  tc.k[Q][0] = r < rem ? Fmt<KB>::ldk(kq) : Fmt<KB>::zk();
  tc.k[Q][1] = r + 8 < rem ? Fmt<KB>::ldk(kq + 8 * KR) : Fmt<KB>::zk();
  tc.v[Q][0] = 2 * j < rem ? Fmt<VB>::ldv(vq) : VCode<VB>{};
  tc.v[Q][1] = 2 * j + 1 < rem ? Fmt<VB>::ldv(vq + VR) : VCode<VB>{};
  tc.v[Q][2] = 2 * j + 8 < rem ? Fmt<VB>::ldv(vq + 8 * VR) : VCode<VB>{};
  tc.v[Q][3] = 2 * j + 9 < rem ? Fmt<VB>::ldv(vq + 9 * VR) : VCode<VB>{};
}

// store the packed code of sub-vector `lane` (4/8-bit) for the fused append
// (all 32 lanes call it; lanes >= nsub -- D = 64: 16 sub-vectors -- hold duplicates and do not store)
template <int BITS>
__device__ __forceinline__ void put_code(unsigned char* row, int lane, uint32_t code, int nsub = 32) {
  if constexpr (BITS == 8) {
    if (lane < nsub) row[lane] = static_cast<uint8_t>(code);
  } else {
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, code, 1);
    if ((lane & 1) == 0 && lane < nsub) row[lane >> 1] = static_cast<uint8_t>(code | (hi << 4));
  }
}

// the appended row's code chunks (just encoded into shared memory) in the per-lane register layout
// of FmtD<BITS, DH>: K chunk of lane j, V chunk of lane r
// NEXT-2 formats: d8b8 / d2b8 chunks are aligned words; the bit-string formats (d4b10, ...) are
// assembled byte by byte (little-endian, reading R11)
template <int NB, int NW>
__device__ __forceinline__ void bytes_to_words(const unsigned char* p, uint32_t (&w)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = 0u;
#pragma unroll
  for (int i = 0; i < NB; ++i) w[i >> 2] |= static_cast<uint32_t>(p[i]) << (8 * (i & 3));
}
template <int BITS, int DH>
__device__ __forceinline__ KCode<BITS> new_kchunk(const unsigned char* nc, int j) {
  if constexpr (BITS == 8 && DH == 128) return *reinterpret_cast<const uint2*>(nc + 8 * j);
  else if constexpr (BITS == 8) return make_uint2(*reinterpret_cast<const uint32_t*>(nc + 4 * j), 0u);
  else if constexpr (BITS == 4 && DH == 128) return *reinterpret_cast<const uint32_t*>(nc + 4 * j);
  else if constexpr (BITS == 4) return *reinterpret_cast<const uint16_t*>(nc + 2 * j);
  else if constexpr (BITS == kFmtD8B8) return *reinterpret_cast<const uint32_t*>(nc + 4 * j);
  else if constexpr (BITS == kFmtD2B8) return *reinterpret_cast<const uint4*>(nc + 16 * j);
  else {
    KCode<BITS> c;
    bytes_to_words<Fmt<BITS>::kOffK>(nc + Fmt<BITS>::kOffK * j, c.w);
    return c;
  }
}
template <int BITS, int DH>
__device__ __forceinline__ VCode<BITS> new_vchunk(const unsigned char* nc, int r) {
  if constexpr (BITS == 8 && DH == 128) return *reinterpret_cast<const uint32_t*>(nc + 4 * r);
  else if constexpr (BITS == 8) return *reinterpret_cast<const uint16_t*>(nc + 2 * r);
  else if constexpr (BITS == 4 && DH == 128) return *reinterpret_cast<const uint16_t*>(nc + 2 * r);
  else if constexpr (BITS == 4) return nc[r];
  else if constexpr (BITS == kFmtD8B8) return *reinterpret_cast<const uint16_t*>(nc + 2 * r);
  else if constexpr (BITS == kFmtD2B8) return *reinterpret_cast<const uint2*>(nc + 8 * r);
  else {
    VCode<BITS> c;
    bytes_to_words<Fmt<BITS>::kOffV>(nc + Fmt<BITS>::kOffV * r, c.w);
    return c;
  }
}
// sub-vector size and code width of a format id (b for d = 4, else 100 d + b)
constexpr int fmt_sub(int f) { return f < 100 ? 4 : f / 100; }
constexpr int fmt_bits(int f) { return f < 100 ? f : f % 100; }

// Query transform of Eq. 7 for one head (one warp): ((q * lambda) H_pm) * qscale, fp32 FWHT
// (2 register + 5 shuffle stages); q (4 bf16) and lambda (float4) are this lane's 4 channels;
// dst = this lane's 4 outputs (sub-vector `lane`).
__device__ __forceinline__ void qtransform_lane(uint2 w, float4 l, float qscale, int lane, float* dst,
                                                int nlanes = 32) {
  float x[4];
  x[0] = __uint_as_float(w.x << 16) * l.x;
  x[1] = __uint_as_float(w.x & 0xFFFF0000u) * l.y;
  x[2] = __uint_as_float(w.y << 16) * l.z;
  x[3] = __uint_as_float(w.y & 0xFFFF0000u) * l.w;
  float s0 = x[0] + x[1], s1 = x[0] - x[1], s2 = x[2] + x[3], s3 = x[2] - x[3];
  x[0] = s0 + s2; x[2] = s0 - s2; x[1] = s1 + s3; x[3] = s1 - s3;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    if (m >= nlanes) break;   // D = 64: 4 shuffle stages inside each half-warp
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float o = __shfl_xor_sync(0xffffffffu, x[i], m);
      x[i] = upper ? (o - x[i]) : (x[i] + o);
    }
  }
  if (lane < nlanes)
    *reinterpret_cast<float4*>(dst) = make_float4(x[0] * qscale, x[1] * qscale, x[2] * qscale, x[3] * qscale);
}

}  // namespace vecinfer
