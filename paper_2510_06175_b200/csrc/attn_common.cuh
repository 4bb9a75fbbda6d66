// Internal declarations shared by the attention kernels and their host dispatch.
#pragma once
#ifndef VECINFER_SPIN_NS
#define VECINFER_SPIN_NS 0    // back-off between polls of an unpublished split partial (ns; measured: 0 >= 20 > 100)
#endif
#include "common.cuh"

namespace vecinfer {

struct AttnArgs {
  const uint16_t* q;  // bf16 [B, Hq, D]
  int64_t q_sb, q_sh;
  int B, Hq, Hkv, G;   // Hkv: VIRTUAL KV heads (= Hc * hsplit); G: query heads per virtual head (<= 4)
  int Hc, hsplit, Gfull;   // code/cache KV heads, virtual heads per KV head (GQA group > 4), full group
  int D;                   // head dim: 128, or 64 (split kernel only)
  const float* lambda;  // [Hkv, 128]
  const uint16_t* ck;   // bf16 codebooks
  const uint16_t* cv;
  int64_t ck_hs, cv_hs;
  const uint8_t* kcodes;  // [B, Hkv, n_cap, row]
  const uint8_t* vcodes;
  int64_t n_cap;
  const int32_t* bt;           // paged code cache (split kernel): block table, NULL = contiguous
  int64_t bt_stride;
  int page_shift, n_pages;
  const int32_t* seq_lens;
  int64_t tok_begin, tok_end;  // tok_end < 0: to seq_len
  float qscale;                // (1/sqrt(D)) * softmax_scale * log2(e): folded into q~
  int S;                       // splits per (b, h_kv)
  int n_items;                 // B * H_kv * S work items
  int cluster;                 // 1: the S splits of a (b, h_kv) form one cluster, merged over DSMEM
  int tc;                      // 1: split kernel with the tcgen05 score contraction (VECINFER_ATTN_DEQUANT_TC)
  int merge_kernel;            // 1: split partials are merged by a separate PDL-launched kernel
  int merge_spin;              // 1: single-wave grid, every CTA merges a slice after an arrival barrier
  int early;                   // 1: seq_lens / write_pos / codes read before the grid-dependency wait
  // stream kernel (attn_stream.cu): U = B*H_kv units and V virtual CTAs tile one line of U*V ticks
  // (unit u = [u*V, (u+1)*V), CTA c = [c*U, (c+1)*U))
  int U, V;
  double rcpU, rcpV;           // 1/U, 1/V (host, double): division-free tick arithmetic
  int seg_cost;                // stream partition: virtual tokens per split-unit start (segment setup cost)
  int merge;                   // kMergeNone / kMergeSpin / kMergeLast
  unsigned long long* part_elem;   // [U + V][4][128] published (o, L) elements (zero = empty)
  void* o;
  int o_f32;
  float* lse;
  float* part_o;     // [B*Hkv*S][4][128]
  float* part_l;     // [B*Hkv*S][4]   (log2 domain)
  uint32_t* counter; // [B*Hkv] 64-bit words: last-arriver counts (low half), zero on exit
  unsigned long long* phase;  // profiling builds: per-CTA phase stamps (else null)
  // fused decode append (vecinfer_decode_step): encode the new token's k, v of each (b, h_kv)
  // into cache row write_pos[b] inside the attention launch (append == 0: plain attention)
  int append;
  const uint16_t* knew;  // bf16 [B, H_kv, 128] (strides kn_sb, kn_sh)
  const uint16_t* vnew;
  int64_t kn_sb, kn_sh, vn_sb, vn_sh;
  const float* inv_lambda;  // [H_kv, 128]
  const int32_t* write_pos; // [B]
  uint32_t* err;            // optional VECINFER_FLAG_* word
  uint8_t* kcodes_w;        // writable views of the code caches
  uint8_t* vcodes_w;
  float inv_sqrt_d;
  // full-precision residual window (NEXT-1): row t is attended by split t % S, warp (t / S) % 16;
  // res_append: the new token goes to residual row res_lens[b]-1 (raw bf16 copy), not the codes
  int res;
  const uint16_t* kres;  // bf16 [B, H_kv, r_cap, 128]
  const uint16_t* vres;
  int64_t res_sb, res_sh, r_cap;
  const int32_t* res_lens;
  int res_append;
  float qscale_raw;      // softmax_scale * log2(e): raw-query scale for the residual scores
  // cross-GPU merge fused into the launch (vecinfer_attn_decode_xr): xr_P ranks, 0 = off; windows
  // [xr_P] of 64-bit words: a 256-byte header (epoch, arrival counter), then [2][xr_P][xr_rows][D]
  int xr_P, xr_rank;
  void* const* xr_win;
  int64_t xr_rows;
  uint32_t* xr_err;
};

constexpr unsigned long long kXrTimeoutNs = 5000000000ull;   // a missing peer flags instead of hanging
constexpr int kXrHeaderWords = 32;                          // 256-byte window header
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long xr_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Fused cross-rank step of one output element (o row `row`, dimension `dim`), called by every lane
// of an L-lane merge group after the rank-local merge (m, wsum, osum; log2 domain, identical in
// all L lanes).  The rank partial (o_r, L_r) is published as ~(L_r << 32 | o_r) (zero = not yet
// written) into slot [par][rank][row][dim] of every rank's window (lane ll stores to ranks ll,
// ll + L, ...); then the lanes poll the P slots [par][p][row][dim] of the own window, consume them
// (store zero back: slots of a parity are reused two calls later, after every rank has passed this
// call), and merge the P partials with a fixed butterfly -- the same arithmetic and order on every
// rank, so all ranks hold bitwise the same o.  Alg. 1 l.729-730 / S:314-322 over ranks.
template <int DH>
__device__ __forceinline__ void xr_merge(const AttnArgs& a, int64_t row, int dim, bool act, int ll, int L,
                                         float m, float wsum, float osum, uint32_t par, int64_t row_lse) {
  const int P = a.xr_P;
  const bool empty = !(wsum > 0.f);
  const float ov = empty ? 0.f : osum * __frcp_rn(wsum);
  const float lr = empty ? -INFINITY : m + __log2f(wsum);
  const unsigned long long word =
      ~((static_cast<unsigned long long>(__float_as_uint(lr)) << 32) | __float_as_uint(ov));
  const int64_t blk = a.xr_rows * DH;                  // one rank's slot block
  const int64_t slot = row * DH + dim;
  if (act) {
    for (int p = ll; p < P; p += L) {
      unsigned long long* w = static_cast<unsigned long long*>(a.xr_win[p]) + kXrHeaderWords +
                              (static_cast<int64_t>(par) * P + a.xr_rank) * blk + slot;
      st_relaxed_sys_u64(w, word);
    }
  }
  unsigned long long* own = static_cast<unsigned long long*>(a.xr_win[a.xr_rank]) + kXrHeaderWords +
                            static_cast<int64_t>(par) * P * blk + slot;
  constexpr int kPer = 8;                              // ranks per lane: P <= 16, L >= 2
  unsigned long long w[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int p = ll + k * L;
    w[k] = (act && p < P) ? ld_relaxed_sys_u64(own + p * blk) : ~0ull;
  }
  bool late = false;
  const unsigned long long t0 = xr_clock_ns();
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int p = ll + k * L;
    if (act && p < P) {
      while (w[k] == 0ull) {
        if (xr_clock_ns() - t0 > kXrTimeoutNs) { late = true; break; }
        w[k] = ld_relaxed_sys_u64(own + p * blk);
      }
      st_relaxed_gpu_u64(own + p * blk, 0ull);
    }
  }
  if (late && a.xr_err) atomicOr(a.xr_err, VECINFER_FLAG_P2P_TIMEOUT);
  float lv[kPer], xv[kPer];
  float M = -INFINITY;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int p = ll + k * L;
    const unsigned long long v = ~w[k];
    const bool has = act && p < P && w[k] != 0ull;     // a timed-out rank counts as empty
    xv[k] = has ? __uint_as_float(static_cast<uint32_t>(v)) : 0.f;
    lv[k] = has ? __uint_as_float(static_cast<uint32_t>(v >> 32)) : -INFINITY;
    M = fmaxf(M, lv[k]);
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float o2 = __shfl_xor_sync(0xffffffffu, M, off);
    if (off < L) M = fmaxf(M, o2);
  }
  float ws = 0.f, os = 0.f;
  if (M != -INFINITY) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const float f = lv[k] == -INFINITY ? 0.f : ex2_approx(lv[k] - M);
      ws += f;
      os += f * xv[k];
    }
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float a2 = __shfl_xor_sync(0xffffffffu, ws, off);
    const float b2 = __shfl_xor_sync(0xffffffffu, os, off);
    if (off < L) {
      ws += a2;
      os += b2;
    }
  }
  if (act && ll == 0) {
    const bool emp = !(ws > 0.f);
    const float o_fin = emp ? 0.f : os * __frcp_rn(ws);
    if (a.o_f32) static_cast<float*>(a.o)[slot] = o_fin;
    else static_cast<__nv_bfloat16*>(a.o)[slot] = __float2bfloat16_rn(o_fin);
    if (dim == 0 && a.lse) a.lse[row_lse] = emp ? -INFINITY : (M + __log2f(ws)) * kLn2;
  }
}


// extra tokens' worth of work the split owning the appended row does (its encode), used to
// shorten that split so it does not become the straggler
#ifndef VECINFER_APPEND_TOKEN_COST
#define VECINFER_APPEND_TOKEN_COST 512   // measured: 0 / 160 / 320 / 512 -> 512 best (cfg3, cfg4 fused steps)
#endif
constexpr int64_t kAppendTokenCost = VECINFER_APPEND_TOKEN_COST;

// GQA groups of up to 8 query heads run as hsplit = ceil(G/4) virtual KV heads of <= 4 query
// heads each: virtual head h reads the codes, codebooks and lambda of KV head hc = h / hsplit and
// serves query heads hq0 .. hq0 + gp - 1.  (hsplit = 1: h == hc, hq0 = h * G, gp = G.)
struct HeadMap {
  int hc;    // KV head (codes, codebooks, lambda, k_new/v_new, residual rows)
  int hq0;   // first query head
  int gp;    // query heads in this virtual head (<= 4)
};
__device__ __forceinline__ HeadMap head_map(const AttnArgs& a, int h) {
  HeadMap m;
  if (a.hsplit == 1) {
    m.hc = h; m.hq0 = h * a.G; m.gp = a.G;
  } else {
    m.hc = h >> 1;
    const int half = h & 1;
    m.hq0 = m.hc * a.Gfull + 4 * half;
    m.gp = half ? a.Gfull - 4 : 4;
  }
  return m;
}

// merge of the pieces of a unit split over several CTAs (stream kernel)
constexpr int kMergeNone = 0;   // every unit is processed by one CTA
constexpr int kMergeSpin = 1;   // all CTAs co-resident: publish, then each piece merges a slice
constexpr int kMergeLast = 2;   // persistent grid: the last-arriving piece merges the unit

// floor(x / d) for 0 <= x < 2^53, 1 <= d < 2^31: the double estimate x * (1/d) is within one of the
// quotient (x is exact in double), so one integer fix-up step either way makes it exact
__device__ __forceinline__ int64_t div_fix(int64_t x, int64_t d, double rcp) {
  int64_t q = __double2ll_rz(static_cast<double>(x) * rcp);
  const int64_t r = x - q * d;
  q += (r >= d) ? 1 : 0;
  q -= (r < 0) ? 1 : 0;
  return q;
}

// Token range [r0, r1) of split s within the attended range [beg, e) of a sequence of len tokens.
__device__ __forceinline__ void split_range_len(const AttnArgs& a, int64_t len, int s, int64_t& r0, int64_t& r1,
                                                int64_t* pbeg = nullptr, int64_t* pend = nullptr) {
  if (len > a.n_cap) len = a.n_cap;
  if (len < 0) len = 0;
  int64_t e = a.tok_end < 0 ? len : (a.tok_end < len ? a.tok_end : len);
  int64_t beg = a.tok_begin < e ? a.tok_begin : e;
  if (beg < 0) beg = 0;
  if (pbeg) *pbeg = beg;
  if (pend) *pend = e;
  const int64_t n = e - beg;
  const int64_t extra = a.S > 1 && a.append ? kAppendTokenCost : 0;
  int64_t chunk = (n + extra + a.S - 1) / a.S;
  chunk = (chunk + 31) & ~int64_t(31);
  r0 = beg + s * chunk;
  if (r0 > e) r0 = e;
  r1 = r0 + chunk;
  if (r1 > e) r1 = e;
}
__device__ __forceinline__ void split_range(const AttnArgs& a, int b, int s, int64_t& r0, int64_t& r1,
                                            int64_t* pbeg = nullptr, int64_t* pend = nullptr) {
  split_range_len(a, a.seq_lens[b], s, r0, r1, pbeg, pend);
}

// CTA epilogue shared by all kernels: combine per-warp (m, l, acc) partials held in shared
// memory, then either write the final output (S == 1) or a split partial plus a fused
// last-CTA log-sum-exp merge over the S splits in fixed order s = 0..S-1.
//   wm[NW][4], wl[NW][4] (log2 domain), wacc[NW][4][WROW] (unnormalised, rows WROW floats apart);
//   scratch: >= 4*S + 8 floats of shared memory not aliased with wm/wl/wacc.
// Fixed-order log-sum-exp merge of the S split partials of unit (b, h) into o and lse, in chunks
// of 32 splits: all 2 x 32 loads of a chunk are issued before any use (one memory round trip per
// chunk), then the running-max combine over s = 0..S-1.
template <int NTHREADS, int DH = 128>
__device__ __forceinline__ void merge_splits(const AttnArgs& a, int b, int h) {
  const int64_t unit = static_cast<int64_t>(b) * a.Hkv + h;
  const HeadMap hm = head_map(a, h);
  for (int idx = threadIdx.x; idx < 4 * DH; idx += NTHREADS) {
    const int g = idx / DH, dim = idx % DH;   // partials keep a 128-float row per head
    if (g >= hm.gp) continue;
    const float* pl = a.part_l + unit * a.S * 4 + g;
    const float* po = a.part_o + (unit * a.S * 4 + g) * 128 + dim;
    float m = -INFINITY, wsum = 0.f, osum = 0.f;
    for (int s0 = 0; s0 < a.S; s0 += 32) {
      float lv[32], xv[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const bool ok = s0 + k < a.S;
        lv[k] = ok ? __ldcg(pl + 4 * (s0 + k)) : -INFINITY;
        xv[k] = ok ? __ldcg(po + static_cast<int64_t>(s0 + k) * 512) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 32; ++k)   // consumed: each o element is read by this thread only
        if (s0 + k < a.S) __stcg(const_cast<float*>(po) + static_cast<int64_t>(s0 + k) * 512, 0.f);
      float mc = -INFINITY;
#pragma unroll
      for (int k = 0; k < 32; ++k) mc = fmaxf(mc, lv[k]);
      const float mn = fmaxf(m, mc);
      if (mn == -INFINITY) continue;
      const float sc = m == -INFINITY ? 0.f : ex2_approx(m - mn);
      osum *= sc;
      wsum *= sc;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float f = lv[k] == -INFINITY ? 0.f : ex2_approx(lv[k] - mn);
        wsum += f;
        osum += f * xv[k];
      }
      m = mn;
    }
    const bool empty = !(wsum > 0.f);
    const float ov = empty ? 0.f : osum / wsum;
    const int64_t oi = (static_cast<int64_t>(b) * a.Hq + hm.hq0 + g) * DH + dim;
    if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
    else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
    if (dim == 0 && a.lse) a.lse[static_cast<int64_t>(b) * a.Hq + hm.hq0 + g] = empty ? -INFINITY : (m + __log2f(wsum)) * kLn2;
  }
  // the L partials are read by every dim thread of their head: zero them once all reads are done,
  // so the whole workspace is zero on exit (a later call with another layout may reuse any word)
  __syncthreads();
  for (int i = threadIdx.x; i < a.S * 4; i += NTHREADS)
    if ((i & 3) < hm.gp) __stcg(a.part_l + unit * a.S * 4 + i, 0.f);
}

template <int NTHREADS, int NWARPS, int WROW = 128, int DH = 128, bool PRESCALED = false, bool XR = false>
__device__ __forceinline__ void cta_finish(const AttnArgs& a, int b, int h, int s,
                                           const float* wm, const float* wl, const float* wacc,
                                           float* scratch) {
  // PRESCALED: the warps already rescaled their partials to the CTA-wide running max M of each head
  // (M = max_w wm[w][g]), so the combine is a plain sum over the warps.
  const int tid = threadIdx.x;
  const int64_t unit = static_cast<int64_t>(b) * a.Hkv + h;
  const HeadMap hm = head_map(a, h);
  __shared__ bool s_last;
  // outputs o = g * DH + dim; partials are stored with a 128-float row per head
  for (int idx = tid; idx < 4 * DH; idx += NTHREADS) {
    const int g = idx / DH, dim = idx % DH;
    float M = -INFINITY;
    float osum = 0.f, lsum = 0.f;
    if constexpr (PRESCALED && NWARPS == 16) {
      // head g is warp-uniform (DH is a multiple of 32): lanes l and l + 16 read warp l % 16's
      // (max, l) once, a 16-lane butterfly gives the CTA max and the l sum to every lane
      const int lane = tid & 31;
      M = wm[(lane & 15) * 4 + g];
      lsum = wl[(lane & 15) * 4 + g];
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) {
        M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
      }
#pragma unroll
      for (int w = 0; w < NWARPS; ++w) osum += wacc[(w * 4 + g) * WROW + dim];
    } else if constexpr (PRESCALED) {
#pragma unroll
      for (int w = 0; w < NWARPS; ++w) {
        M = fmaxf(M, wm[w * 4 + g]);
        lsum += wl[w * 4 + g];
        osum += wacc[(w * 4 + g) * WROW + dim];
      }
    } else {
#pragma unroll
      for (int w = 0; w < NWARPS; ++w) M = fmaxf(M, wm[w * 4 + g]);
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < NWARPS; ++w) {
          const float f = ex2_approx(wm[w * 4 + g] - M);
          lsum += f * wl[w * 4 + g];
          osum += f * wacc[(w * 4 + g) * WROW + dim];
        }
      }
    }
    const bool empty = !(lsum > 0.f) || M == -INFINITY;
    const float ov = empty ? 0.f : osum / lsum;
    const float L2 = empty ? -INFINITY : M + __log2f(lsum);
    if (a.S == 1) {
      if (g < hm.gp) {
        const int64_t oi = (static_cast<int64_t>(b) * a.Hq + hm.hq0 + g) * DH + dim;
        if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
        else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
        if (dim == 0 && a.lse) a.lse[static_cast<int64_t>(b) * a.Hq + hm.hq0 + g] = L2 * kLn2;
      }
    } else if (a.merge_spin) {
      // publish (o_s, L_s) as one 64-bit relaxed store of ~(L_s << 32 | o_s) (zero = empty); only
      // for the real heads g < gp, the ones the consumers poll and zero (a padding element left
      // non-zero would be taken as a fresh piece by a later launch reusing the workspace)
      if (g >= hm.gp) continue;
      const int64_t pi = ((unit * a.S + s) * 4 + g) * 128 + dim;
      st_relaxed_gpu_u64(a.part_elem + pi, ~((static_cast<unsigned long long>(__float_as_uint(L2)) << 32) |
                                             __float_as_uint(ov)));
    } else if (g < hm.gp) {   // real heads only: merge_splits consumes (zeroes) exactly these
      const int64_t pi = (unit * a.S + s) * 4 + g;
      a.part_o[pi * 128 + dim] = ov;
      if (dim == 0) a.part_l[pi] = L2;
    }
  }
  if (a.S == 1 || a.merge_kernel) return;
  if (a.merge_spin) {
    // Single-wave grid (all S CTAs of the unit are co-resident), no fence and no atomic: split s
    // merges outputs [s*per, (s+1)*per) of the unit, per = ceil(4*DH/S).  Each output is merged by
    // a group of L lanes (L = the largest power of two <= min(S, 32)); lane l of a group owns
    // splits l, l+L, l+2L, ...  Every lane first issues the loads of all its elements, then polls
    // the ones not yet published (non-zero), consumes them (stores zero back: each element is read
    // exactly once, so the workspace is clean for the next launch) and folds them in split order;
    // the group combines its lanes with a fixed butterfly (deterministic).  One memory round trip
    // once the last split has published; no shared-memory staging, no __syncthreads.
    phase_mark(a.phase, (b * a.Hkv + h) * a.S + s, 8);
    (void)scratch;
    const int S = a.S;
    const int per = (4 * DH + S - 1) / S;
    const int o0 = s * per, nout = max(0, min(4 * DH, o0 + per) - o0);
    const int L = S >= 32 ? 32 : (1 << (31 - __clz(S)));
    const int groups = NTHREADS / L, lg = tid / L, ll = tid % L;
    constexpr int kMaxPer = 4;   // splits per lane: S <= 128 (kMaxSplits)
    // fused cross-rank merge: this launch's slot parity from the own window's epoch counter (read
    // by every CTA before it arrives below; the last arrival advances it)
    uint32_t xr_epoch = 0;
    if constexpr (XR) {
      xr_epoch = ld_acquire_gpu(static_cast<const uint32_t*>(a.xr_win[a.xr_rank])) + 1u;
      if (xr_epoch == 0) xr_epoch = 1u;
    }
    for (int t0 = 0; t0 < nout; t0 += groups) {   // one pass unless S is tiny and DH... (uniform)
      const int t = t0 + lg;
      const int o = o0 + t, g = o / DH, dim = o % DH;
      const bool act = t < nout && g < hm.gp;
      unsigned long long* pp = a.part_elem + (unit * S) * 512 + g * 128 + dim;
      unsigned long long w[kMaxPer];
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k) {
        const int p = ll + k * L;
        w[k] = (act && p < S) ? ld_relaxed_gpu_u64(pp + static_cast<int64_t>(p) * 512) : ~0ull;
      }
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k) {
        const int p = ll + k * L;
        if (act && p < S) {
          while (w[k] == 0ull) {
            if (VECINFER_SPIN_NS > 0) __nanosleep(VECINFER_SPIN_NS);
            w[k] = ld_relaxed_gpu_u64(pp + static_cast<int64_t>(p) * 512);
          }
          st_relaxed_gpu_u64(pp + static_cast<int64_t>(p) * 512, 0ull);
        }
      }
      phase_mark(a.phase, (b * a.Hkv + h) * a.S + s, 10);
      // ~w = (L_s << 32 | o_s); the neutral element ~0 decodes to (o, L) = (0, bits 0) -> mark it
      float lv[kMaxPer], xv[kMaxPer];
      float m = -INFINITY;
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k) {
        const int p = ll + k * L;
        const unsigned long long v = ~w[k];
        const bool has = act && p < S;
        xv[k] = has ? __uint_as_float(static_cast<uint32_t>(v)) : 0.f;
        lv[k] = has ? __uint_as_float(static_cast<uint32_t>(v >> 32)) : -INFINITY;
        m = fmaxf(m, lv[k]);
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {   // butterflies inside the L-lane group (L uniform)
        const float o2 = __shfl_xor_sync(0xffffffffu, m, off);
        if (off < L) m = fmaxf(m, o2);
      }
      float wsum = 0.f, osum = 0.f;
      if (m != -INFINITY) {
#pragma unroll
        for (int k = 0; k < kMaxPer; ++k) {
          const float f = lv[k] == -INFINITY ? 0.f : ex2_approx(lv[k] - m);
          wsum += f;
          osum += f * xv[k];
        }
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float a2 = __shfl_xor_sync(0xffffffffu, wsum, off);
        const float b2 = __shfl_xor_sync(0xffffffffu, osum, off);
        if (off < L) {
          wsum += a2;
          osum += b2;
        }
      }
      if constexpr (XR) {   // the rank partial goes to every rank; o, lse are the final merge
        const int64_t row = static_cast<int64_t>(b) * a.Hq + hm.hq0 + g;
        xr_merge<DH>(a, row, dim, act, ll, L, m, wsum, osum, xr_epoch & 1u, row);
        continue;
      }
      if (act && ll == 0) {
        const bool empty = !(wsum > 0.f);
        const int64_t oi = (static_cast<int64_t>(b) * a.Hq + hm.hq0 + g) * DH + dim;
        const float ov = empty ? 0.f : osum * __frcp_rn(wsum);
        if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
        else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
        if (dim == 0 && a.lse)
          a.lse[static_cast<int64_t>(b) * a.Hq + hm.hq0 + g] = empty ? -INFINITY : (m + __log2f(wsum)) * kLn2;
      }
    }
    if constexpr (XR) {   // arrival; the last CTA of the launch records the epoch it used
      __syncthreads();
      if (tid == 0) {
        uint32_t* hdr = static_cast<uint32_t*>(a.xr_win[a.xr_rank]);
        if (atom_add_acq_rel_gpu(hdr + 1, 1u) == static_cast<uint32_t>(a.n_items - 1)) {
          st_relaxed_gpu(hdr + 1, 0u);
          st_relaxed_gpu(hdr, xr_epoch);
        }
      }
    }
    phase_mark(a.phase, (b * a.Hkv + h) * a.S + s, 5);
    return;
  }
  phase_mark(a.phase, (b * a.Hkv + h) * a.S + s, 6);
  __syncthreads();
  phase_mark(a.phase, (b * a.Hkv + h) * a.S + s, 7);
  // low 32-bit half of the unit's 64-bit barrier word (reset to zero by the merging CTA)
  if (tid == 0) s_last = (atom_add_acq_rel_gpu(&a.counter[2 * unit], 1u) == static_cast<uint32_t>(a.S - 1));
  __syncthreads();
  phase_mark(a.phase, (b * a.Hkv + h) * a.S + s, 5);
  if (!s_last) return;
  merge_splits<NTHREADS, DH>(a, b, h);
  if (tid == 0) a.counter[2 * unit] = 0u;  // ready for the next launch
}

// q~ rows in shared memory: sub-vector m of a head at float offset 4m + 8(m/8), heads kQRow = 164
// floats apart.  The MMA kernels' B-fragment loads (lanes (r, j) read head r/2, sub-vectors 8j+t)
// then hit 8 distinct 16-byte bank groups instead of one (a 16-way conflict with dense rows).
constexpr int kQRow = 164;
__device__ __forceinline__ int qoff(int m) { return 4 * m + 8 * (m >> 3); }

// Query transform of Eq. 7 for the G query heads of KV head h, one warp per head:
// sq[g][:] = ((q_g * lambda) H_pm) * qscale  (fp32 FWHT: 2 register + 5 shuffle stages).
// Heads g >= G are zero (padding of the 4-wide GQA group).
// padded: write in the qoff() layout (MMA kernels), else dense (LUT kernel).
__device__ __forceinline__ void query_transform_warp(const AttnArgs& a, int b, int h, int g, float* sq_g,
                                                     bool padded = false) {
  const int lane = threadIdx.x & 31;
  float x[4] = {0.f, 0.f, 0.f, 0.f};
  const HeadMap hm = head_map(a, h);
  if (g < hm.gp) {
    const uint16_t* qp = a.q + b * a.q_sb + (hm.hq0 + g) * a.q_sh + 4 * lane;
    const uint2 w = *reinterpret_cast<const uint2*>(qp);
    const float4 l = *reinterpret_cast<const float4*>(a.lambda + hm.hc * 128 + 4 * lane);
    x[0] = __uint_as_float(w.x << 16) * l.x;
    x[1] = __uint_as_float(w.x & 0xFFFF0000u) * l.y;
    x[2] = __uint_as_float(w.y << 16) * l.z;
    x[3] = __uint_as_float(w.y & 0xFFFF0000u) * l.w;
  }
  float s0 = x[0] + x[1], s1 = x[0] - x[1], s2 = x[2] + x[3], s3 = x[2] - x[3];
  x[0] = s0 + s2; x[2] = s0 - s2; x[1] = s1 + s3; x[3] = s1 - s3;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float o = __shfl_xor_sync(0xffffffffu, x[i], m);
      x[i] = upper ? (o - x[i]) : (x[i] + o);
    }
  }
  *reinterpret_cast<float4*>(sq_g + (padded ? qoff(lane) : 4 * lane)) =
      make_float4(x[0] * a.qscale, x[1] * a.qscale, x[2] * a.qscale, x[3] * a.qscale);
}

cudaError_t launch_attn_mma(const AttnArgs& a, int kbits, int vbits, cudaStream_t st);
bool attn_mma_supports(int kfmt, int vfmt, int dh);   // a split kernel exists for the format pair
cudaError_t launch_attn_stream(const AttnArgs& a, int kbits, int vbits, cudaStream_t st);
int attn_mma_max_active_clusters(int cluster_size);  // 0 if not schedulable
void launch_attn_lut(const AttnArgs& a, int kbits, int vbits, cudaStream_t st);

}  // namespace vecinfer
