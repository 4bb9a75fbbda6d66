// N3+N4+N5: split-KV fused VQ decode attention, DEQUANT_MMA algorithm (default on sm_100a).
//
// Implements Eq. 10 with Algorithm 1's online softmax:
//   s = q~ VQ^-1(K~_q)^T / sqrt(D),  o = softmax(s) VQ^-1(V_q),  L = logsumexp(s).
// CTA = (split, KV head, batch); each of its 16 warps streams 32-token tiles of packed codes
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
// Shared-memory codebook rows are 256 B: [C_k copies 0..15 | C_v copies 0..15] for centroid c,
// in a 64 KiB-aligned region, so a gather address is ONE byte-permute: PRMT places code byte k
// of a code word into address bits 8..15 next to the per-lane base (bits 0..7, 16..31).
// Epilogue: every warp rescales its partial to the CTA-wide running max (f = 2^(m_warp - M)) and
// the CTA sums the 16 warp partials into the split's (o_s, L_s).  Single-wave grids merge the S
// splits with the fence-free publish/consume protocol (attn_common.cuh cta_finish: each split
// merges a 1/S slice of the outputs, one L-lane group per output, fixed butterfly order =>
// deterministic); multi-wave grids merge in the last-arriving CTA; S <= 16 clusters can merge over
// DSMEM.  See DESIGN.md "N4".
#include "attn_tiles.cuh"
#include "tc.cuh"

#ifndef VECINFER_TC_EXP
#define VECINFER_TC_EXP 0   // != 0 only in timing-experiment builds (results not valid)
#endif
// Code tiles staged by the TMA engine (cp.async.bulk into per-warp shared stages, mbarrier
// completion) instead of LDG into registers: VECINFER_CODE_TMA = stages per warp (0 = LDG path).
// b2d4 / D = 128 / contiguous caches, mma.sync score path.
#ifndef VECINFER_CODE_TMA
#define VECINFER_CODE_TMA 0
#endif

namespace vecinfer {
namespace {

// misc region (below the table): q~ [4][kQRow] f32, warp partials, staged split partials
constexpr int kMiscQ = 0;
constexpr int kMiscNew = 2688;                       // 128 B: codes of the appended token (K at +0, V at +64)
constexpr int kMiscW = 2816;                         // wm[16][4], wl[16][4], wacc[16][4][kWRow]
constexpr int kWRow = 132;   // warp-partial row stride: the 16-byte stores of a warp spread over all banks
constexpr int kMiscWEnd = kMiscW + (kNW * 8 + kNW * 4 * kWRow) * 4;   // 37120
// tcgen05 score path (TC): B operand = q~ hi/lo [16 rows x 128] fp16 in the K-major no-swizzle
// canonical layout (element (n, k) at ((k/8)*2 + n/8)*128 + (n%8)*16 + (k%8)*2; rows 8..15 zero),
// then the TMEM base address and one mbarrier per 4-warp group
constexpr int kMiscTCB = 37888;
constexpr int kMiscTCM = kMiscTCB + 4096;            // [0]: TMEM base, [8 + 8g]: mbarrier of group g
constexpr int kMiscBytes = kMiscTCM + 64;            // 42048
static_assert(kMiscWEnd <= kMiscTCB, "misc layout");
static_assert(4 * kQRow * 4 <= kMiscNew, "q~ rows");
// TMEM columns: group g (warps 4g..4g+3, one per 32-lane quarter) stages its 128-token K^ tile in
// columns [64g, 64g + 64) (128 fp16 dims per lane = token) and gets its scores in [256 + 16g, +16)
constexpr uint32_t kTmemCols = 512;
constexpr int kClusterMax = 16;                      // DSMEM merge buffer: [16][4][128] + m, l
constexpr int kCbufBytes = kClusterMax * 4 * 130 * 4;
constexpr int kTmaSt = VECINFER_CODE_TMA;
constexpr int kTmaStage = 2048;                      // one 32-token tile: K rows (1 KiB) | V rows (1 KiB)
constexpr int kSmemBytes = 65536 + kTab + kCbufBytes + 1024;  // pad + table + cluster buffer + slack
// b2d4 with TMA-staged code tiles: the per-warp stages take the cluster buffer's place (the planner
// never clusters it then)
constexpr bool tma_fmt(int kf, int vf) { return kTmaSt > 0 && kf == 8 && vf == 8; }
constexpr int kSmemBytesTma = 65536 + kTab + kNW * kTmaSt * kTmaStage + 1024;
static_assert(kSmemBytesTma <= 232448 - 1024, "TMA stages exceed 227 KiB");
// 16-bit K and V: no shared table -> only misc + cluster buffer, leaving the L1 to the global
// codebook gathers
constexpr int kSmemBytesNoTab = kMiscBytes + 1024 + kCbufBytes + 1024;
constexpr int kSepTab = 65536;   // one separate (NEXT-2) table per stream that needs it
// shared-memory layout of a format pair: misc at 0; the classic [K | V] 256-row table (4/8-bit
// d = 4, d8b8, d2b8) at the next 64 KiB boundary; separate d8b12 / d4b10 tables (K, then V) after
// it (or after misc when there is no classic table); the cluster-merge buffer last
constexpr bool classic_tab(int f) { return f == 4 || f == 8 || f == kFmtD8B8 || f == kFmtD2B8; }
constexpr bool sep_tab(int f) { return f == kFmtD8B12 || f == kFmtD4B10; }
constexpr int smem_layout_bytes(int kf, int vf) {
  const int nsep = (sep_tab(kf) ? 1 : 0) + (sep_tab(vf) ? 1 : 0);
  if (tma_fmt(kf, vf)) return kSmemBytesTma > kSmemBytes ? kSmemBytesTma : kSmemBytes;
  if (classic_tab(kf) || classic_tab(vf)) return kSmemBytes + nsep * kSepTab;
  if (nsep) return ((kMiscBytes + 1023) & ~1023) + nsep * kSepTab + kCbufBytes + 1024;
  // no shared table (16-bit K and V: the books are gathered through L1/L2): no cluster buffer either
  // (the planner never clusters these), so the smallest carveout leaves the L1 the most capacity
  return kMiscBytes + 1024;
}
static_assert(smem_layout_bytes(kFmtD8B12, kFmtD8B8) <= 232448, "largest layout exceeds 227 KiB");


// K code row of one token for the tcgen05 score path (lane = token): 32 sub-vector codes
template <int KB> struct KRowT { uint4 w[Fmt<KB>::kRow / 16]; };
// shared address of the centroid of sub-vector m of a K row (code byte / nibble -> address bits 8..)
template <int KB, int M>
__device__ __forceinline__ uint32_t krow_addr(const KRowT<KB>& kr, uint32_t base) {
  if constexpr (KB == 8) {
    const uint4& q = kr.w[M / 16];
    constexpr int wi = (M / 4) % 4;
    const uint32_t w = wi == 0 ? q.x : wi == 1 ? q.y : wi == 2 ? q.z : q.w;
    return prmt(w, base, 0x7604u | ((M & 3) << 4));
  } else {
    const uint4& q = kr.w[0];
    constexpr int wi = M / 8;
    const uint32_t w = wi == 0 ? q.x : wi == 1 ? q.y : wi == 2 ? q.z : q.w;
    return Fmt<4>::nib8<M % 8>(w) | base;
  }
}

// XR: the fused cross-rank merge variant (vecinfer_attn_decode_xr; single-wave spin merge only)
// PG: paged code caches (a separate instantiation, so the contiguous kernels carry no translation
// code: the small cfg2 launch is sensitive to any change of its code)
template <int KB, int VB, int DH, bool TC, bool XR = false, bool PG = false>
__global__ void __launch_bounds__(kThreads, 1) attn_mma_kernel(const AttnArgs a) {
  // DH = head dim (128, or 64: NEXT-4).  KS score k-steps (4 sub-vectors each) per 16 tokens,
  // VS V sub-vectors per lane r (2 P.V m-tiles each), NL lanes holding a q~ row.
  // TC: the score contraction runs on tcgen05 (K^ tile in TMEM, q~ in shared memory, fp32 scores
  // in TMEM) instead of mma.sync; contiguous caches, D = 128, 4/8-bit K codebooks only.
  static_assert(!TC || ((KB == 4 || KB == 8) && DH == 128), "TC path: d = 4 K codebooks in the shared table, D = 128");
  using FK = FmtD<KB, DH>;
  using FV = FmtD<VB, DH>;
  constexpr int KR = FK::kRow, VR = FV::kRow;
  constexpr int KS = DH / 16, VS = DH / 32, NL = DH / 4;
  constexpr bool kCanAppend = KB <= 8 && VB <= 8;   // d = 4, 4/8-bit codebooks (D = 128 or 64)
  // fused append of the NEXT-2 formats whose books live in shared memory (d8b8, d2b8, d4b10,
  // d8b12): a 16-warp centroid scan in the owner split (the 1 MiB d8b16 books are not resident:
  // vecinfer_decode_step appends them with the separate filter encode)
  constexpr auto gen_ok = [](int f) { return f == kFmtD8B8 || f == kFmtD2B8 || f == kFmtD4B10 || f == kFmtD8B12; };
  constexpr bool kGenAppend = gen_ok(KB) && gen_ok(VB) && DH == 128;
  constexpr bool kTma = tma_fmt(KB, VB) && DH == 128 && !TC;   // contiguous caches only (runtime)
  // 65 536-entry d = 4 books (gathered through L1/L2): a warp's tile takes ~20 us, so the next
  // tile's code loads go out after the current tile instead of before it -- their HBM latency hides
  // behind the other warps' gathers, and the two tiles' codes are never live together (b4d4 stack
  // 128 -> 56 B, cfg5 b4d4 137.4 -> 127.2 us; d8b16 measured 1.4 % slower this way: kept early)
  constexpr bool kLateNext = (KB == 16 || VB == 16) && DH == 128 && !TC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, j = lane & 3;
  if (a.cluster) cluster_arrive_relaxed();   // paired with cluster_wait() before the DSMEM pushes

  // shared layout: misc at the bottom, the codebook table at the next 64 KiB boundary
  const uint32_t raw_s = smem_u32(smem_raw);
  constexpr bool kClassic = classic_tab(KB) || classic_tab(VB);
  constexpr bool kSepK = Fmt<KB>::kSep, kSepV = Fmt<VB>::kSep;
  uint32_t tab_off;
  if constexpr (!kClassic) {
    tab_off = (kMiscBytes + 1023) & ~1023;   // no classic table: separate tables / cluster buffer start here
  } else {
    tab_off = ((raw_s + 65535u) & ~65535u) - raw_s;
    if (tab_off < static_cast<uint32_t>(kMiscBytes)) tab_off += 65536u;
  }
  unsigned char* tab = smem_raw + tab_off;
  float* sq = reinterpret_cast<float*>(smem_raw + kMiscQ);
  const uint32_t tab_s = raw_s + tab_off;
  constexpr uint32_t kSepOff = kClassic ? kTab : 0;               // relative to tab
  constexpr uint32_t kSepVOff = kSepOff + (kSepK ? kSepTab : 0);
  constexpr uint32_t kCbufOff = kSepVOff + (kSepV ? kSepTab : 0);

  // Work items = (split s, KV head h, batch b), s fastest.  Grids of up to one wave map one item
  // to each CTA; larger problems run persistent CTAs (one per SM) over items, so the per-CTA
  // prologue/epilogue and the wave ramp are paid once per item instead of once per wave.
  const int nblk = gridDim.x * gridDim.y * gridDim.z;
  // tcgen05 state: TMEM columns (allocated once per CTA), one mbarrier per 4-warp group whose phase
  // advances once per issued score MMA batch, the q~ B tile (rows 8..15 stay zero)
  unsigned char* tcb = smem_raw + kMiscTCB;
  uint32_t* tc_misc = reinterpret_cast<uint32_t*>(smem_raw + kMiscTCM);
  uint32_t tc_phase = 0;
  if constexpr (TC) {
    if (warp == 0) tc::alloc(smem_u32(tc_misc), kTmemCols);
    if (tid < 4) tc::mbar_init(smem_u32(tc_misc + 2 + 2 * tid), 1);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (tid < 128) *reinterpret_cast<uint4*>(tcb + ((tid >> 3) * 2 + 1) * 128 + (tid & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
  }
  // TMA-staged code tiles: warp w owns kTmaSt stages of kTmaStage bytes above the table and one
  // mbarrier per stage (misc TCB region, unused without TC); n_iss / n_con count the warp's issued /
  // consumed tiles across work items (stage = n % kTmaSt, phase parity = (n / kTmaSt) & 1)
  const uint32_t tma_stg = tab_s + kTab + static_cast<uint32_t>(warp * kTmaSt * kTmaStage);
  const uint32_t tma_bar = raw_s + kMiscTCB + static_cast<uint32_t>(warp * kTmaSt * 8);
  uint32_t n_iss = 0, n_con = 0;
  if constexpr (kTma) {
    if (lane < kTmaSt) tc::mbar_init(tma_bar + 8 * lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  bool first = true;
  for (int item = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); item < a.n_items; item += nblk) {
  const int s = item % a.S, h = (item / a.S) % a.Hkv, b = item / (a.S * a.Hkv);
  const int cta_id = item;
  phase_mark(a.phase, cta_id, 0);
  if (!first) __syncthreads();   // previous item is done with the table and the misc region

  // static weights first (codebooks): with programmatic dependent launch this overlaps the
  // tail of the previous kernel on the stream; everything dynamic is read after the wait
  const HeadMap hm = head_map(a, h);   // virtual head h -> KV head hm.hc, query heads hm.hq0 ..
  const int hc = hm.hc;
  const uint16_t* cbk = a.ck + hc * a.ck_hs;
  const uint16_t* cbv = a.cv + hc * a.cv_hs;
  const uint4 tabv = table_load<KB, VB>(cbk, cbv, tid);   // stored while seq_lens is in flight
  float4 lam4 = make_float4(0.f, 0.f, 0.f, 0.f);   // warps 0..3: lambda of head h (static)
  if (warp < 4) lam4 = *reinterpret_cast<const float4*>(a.lambda + hc * DH + 4 * (lane & (NL - 1)));
  // early (VECINFER_ATTN_FLAG_EARLY_CACHE): seq_lens, write_pos and the cached codes were not
  // written by the kernel just before on the stream, so the split range and the first tile's code
  // loads go out before the grid-dependency wait too (under programmatic dependent launch they
  // overlap the previous kernel's tail); only q, k_new / v_new and the residual window wait
  const bool wait_late = first && a.early;
  if (first && !a.early) griddep_wait();
  phase_mark(a.phase, cta_id, 9);
  first = false;
  // q of the warp's query head goes out right after the wait, next to the seq_lens read below
  uint2 qw = make_uint2(0u, 0u);
  auto load_q = [&]() {
    if (warp < hm.gp)
      qw = *reinterpret_cast<const uint2*>(a.q + b * a.q_sb + (hm.hq0 + warp) * a.q_sh + 4 * (lane & (NL - 1)));
  };
  if (!wait_late) load_q();

  // seq_lens goes out next; the codebook table (its loads were issued before the wait) is stored
  // while it is in flight, then the split range and the first tile's loads follow
  const int64_t len_b = a.seq_lens[b];
  table_store<KB, VB>(tab, tabv, tid);
  sep_fill<KB>(tab + kSepOff, cbk, tid, kThreads);     // NEXT-2 d8b12 / d4b10 books (no-ops otherwise)
  sep_fill<VB>(tab + kSepVOff, cbv, tid, kThreads);
  int64_t r0, r1, beg, e;
  split_range_len(a, len_b, s, r0, r1, &beg, &e);
  const int ntok = static_cast<int>(r1 - r0);
  const int ntile = (ntok + 31) >> 5;
  const int64_t unit = static_cast<int64_t>(b) * a.Hc + hc;   // cache unit of the codes
  // fused decode append: the split holding row p = write_pos[b] (else split 0) encodes the new token
  bool owner = false;
  int patch_tile = -1, patch_row = 0;
  int64_t p_row = 0;
  if ((kCanAppend || kGenAppend) && a.append) {
    p_row = a.write_pos[b];
    const bool in_range = p_row >= beg && p_row < e;
    owner = in_range ? (p_row >= r0 && p_row < r1) : (s == 0);
    if (owner && in_range) {
      patch_tile = static_cast<int>((p_row - r0) >> 5);
      patch_row = static_cast<int>((p_row - r0) & 31);
    }
  }
  // lane-resolved code pointers of this warp's first tile.  Paged caches: tiles are 32-aligned
  // (tok_begin % 32 == 0, chunks of 32) so a tile never crosses a page; the page of the tile after
  // next is read one tile ahead so its latency hides behind the current tile.
  constexpr bool paged = PG;
  const uint8_t* kcb = a.kcodes + static_cast<int64_t>(r) * KR + FK::kOffK * j;
  const uint8_t* vcb = a.vcodes + static_cast<int64_t>(2 * j) * VR + FV::kOffV * r;
  const int64_t pmask = (int64_t(1) << a.page_shift) - 1;
  auto page_of = [&](int64_t tok) -> int { return a.bt[b * a.bt_stride + (tok >> a.page_shift)]; };
  auto row_in = [&](int pg, int64_t tok) -> int64_t {   // cache row of token tok given its page
    return paged ? ((static_cast<int64_t>(pg) * a.Hc + hc) << a.page_shift) + (tok & pmask) : unit * a.n_cap + tok;
  };
  int pg_ahead = 0;
  const uint8_t* kp;
  const uint8_t* vp;
  {
    const int64_t tok = r0 + 32 * warp;
    const int64_t rw = row_in(paged && warp < ntile ? page_of(tok) : 0, tok);
    kp = kcb + rw * KR;
    vp = vcb + rw * VR;
    if (paged && warp + kNW < ntile) pg_ahead = page_of(tok + 32 * kNW);
  }
  constexpr int kStepK = 32 * kNW * KR, kStepV = 32 * kNW * VR;  // bytes between a warp's tiles

  // first tile's loads go out before the query transform so HBM latency overlaps it
  TileCodes<KB, VB> nxt;
  // TC path (contiguous): K rows by token (lane = row of the warp's tile), V codes as in TileCodes
  const int64_t row0 = unit * a.n_cap + r0;   // cache row of the split's first token
  const uint8_t* const kq = a.kcodes + (row0 + lane) * KR;   // this lane's row of the split's first tile
  const uint8_t* const vq = vcb + row0 * VR;
  auto load_krow = [&](KRowT<KB>& kr, int it) {
    const int rem = ntok - 32 * it;
    const uint8_t* p = kq + static_cast<int64_t>(it) * (32 * KR);
#pragma unroll
    for (int i = 0; i < KR / 16; ++i) kr.w[i] = lane < rem ? ldg_nc_u128(p + 16 * i) : make_uint4(0u, 0u, 0u, 0u);
  };
  auto load_vtile = [&](TileCodes<KB, VB>& tcv, int it) {   // the V half of a TileCodes
    const int rem = ntok - 32 * it;
    const uint8_t* p = vq + static_cast<int64_t>(it) * (32 * VR);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t0 = 16 * q + 2 * j;
      tcv.v[q][0] = (rem >= 32 || t0 < rem) ? FV::ldv(p + (16 * q) * VR) : VCode<VB>{};
      tcv.v[q][1] = (rem >= 32 || t0 + 1 < rem) ? FV::ldv(p + (16 * q + 1) * VR) : VCode<VB>{};
      tcv.v[q][2] = (rem >= 32 || t0 + 8 < rem) ? FV::ldv(p + (16 * q + 8) * VR) : VCode<VB>{};
      tcv.v[q][3] = (rem >= 32 || t0 + 9 < rem) ? FV::ldv(p + (16 * q + 9) * VR) : VCode<VB>{};
    }
  };
  // TMA: lane 0 issues the bulk copies of tile `it` (K rows, then V rows; a ragged tile copies its
  // valid rows only -- the rest of the stage is stale and masked at the shared loads)
  auto tma_issue = [&](int it) {
    const uint32_t st = n_iss % kTmaSt;
    ++n_iss;
    if (lane == 0) {
      const int rows = ntok - 32 * it < 32 ? ntok - 32 * it : 32;
      const uint32_t bar = tma_bar + 8 * st, dst = tma_stg + st * kTmaStage;
      const int64_t row = row0 + 32 * static_cast<int64_t>(it);
      mbar_expect_tx(bar, static_cast<uint32_t>(rows * (KR + VR)));
      bulk_g2s(dst, a.kcodes + row * KR, static_cast<uint32_t>(rows * KR), bar);
      bulk_g2s(dst + kTmaStage / 2, a.vcodes + row * VR, static_cast<uint32_t>(rows * VR), bar);
    }
  };
  const bool tma_on = kTma && !paged;
  KRowT<KB> kfirst0, kfirst1;
  if constexpr (kTma) {
    if (tma_on) {
#pragma unroll
      for (int k = 0; k < kTmaSt; ++k)
        if (warp + kNW * k < ntile) tma_issue(warp + kNW * k);
    }
  }
  if constexpr (TC) {
    if (warp < ntile) { load_krow(kfirst0, warp); load_vtile(nxt, warp); }
    if (warp + kNW < ntile) load_krow(kfirst1, warp + kNW);
  } else if (warp < ntile && !tma_on) {
    const int rem = ntok - 32 * warp;
    if (rem >= 32) load_tile_full<KB, VB, DH>(nxt, kp, vp);
    else load_tile_tail<KB, VB, DH>(nxt, kp, vp, rem, r, j);
  }
  if (wait_late) {
    griddep_wait();
    load_q();
  }
  phase_mark(a.phase, cta_id, 13);   // first tile issued (after seq_lens)
  unsigned char* newcodes = smem_raw + kMiscNew;   // [0,64): K code row, [64,128): V code row
  if (kCanAppend && owner) {
    // Eq. 9: encode the new token (S then H on the key, VQ on both), 8 warps per stream, each
    // scanning 1/8 of the centroids (bf16 codebook -> fp32, pinned distance, lowest index on ties)
    const bool isv = warp >= 8;
    const int w8 = warp & 7;
    const int P = (isv ? (1 << (VB <= 8 ? VB : 8)) : (1 << (KB <= 8 ? KB : 8))) / 8;   // centroids per warp
    float4* stage = reinterpret_cast<float4*>(smem_raw + kMiscW);
    float* sbest = reinterpret_cast<float*>(smem_raw + kMiscW + 8192);
    uint32_t* sidx = reinterpret_cast<uint32_t*>(smem_raw + kMiscW + 10240);
    const uint16_t* cb = isv ? cbv : cbk;
    if (lane < P) stage[warp * 32 + lane] = bf16x4_to_float4(*reinterpret_cast<const uint2*>(cb + 4 * (P * w8 + lane)));
    float x[4];
    const int le = lane & (NL - 1);   // D = 64: the upper half-warp duplicates the lower one
    if (!isv) {
      const bool bad = key_transform_lane(a.knew + b * a.kn_sb + hc * a.kn_sh + 4 * le,
                                          a.inv_lambda + hc * DH + 4 * le, a.inv_sqrt_d, lane, x, NL);
      if (bad && warp == 0 && lane == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_RANGE);
    } else {
      const float4 v = bf16x4_to_float4(*reinterpret_cast<const uint2*>(a.vnew + b * a.vn_sb + hc * a.vn_sh + 4 * le));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    }
    __syncwarp();
    float best = __int_as_float(0x7f800000);
    uint32_t bi = 0;
#pragma unroll 8
    for (int i = 0; i < P; ++i) {
      const float4 c = stage[warp * 32 + i];
      const float dd = pinned_dist4(x[0], x[1], x[2], x[3], c.x, c.y, c.z, c.w);
      if (dd < best) { best = dd; bi = P * w8 + i; }
    }
    sbest[warp * 32 + lane] = best;
    sidx[warp * 32 + lane] = bi;
  }
  if constexpr (kGenAppend) if (owner) {
    // Eq. 9 for the d8b8 / d2b8 / d4b10 formats: warp 0 writes the pinned key transform, warp 8 the
    // raw value to shared memory; then the 8 warps of a stream scan its sub-vectors against every
    // centroid with the pinned distance (fp32 RN, no FMA, left to right over the d dims: reading
    // R9), the minima reduce as (dist_bits << 32 | j) -- lowest index on ties -- and the codes are
    // packed into the row's little-endian bit string (R11)
    float* xs = reinterpret_cast<float*>(smem_raw + kMiscW);                              // [2][128]
    unsigned long long* gbest = reinterpret_cast<unsigned long long*>(smem_raw + kMiscW + 1024);   // [2][64]
    if (warp == 0) {
      float x[4];
      const bool bad = key_transform_lane(a.knew + b * a.kn_sb + hc * a.kn_sh + 4 * lane,
                                          a.inv_lambda + hc * 128 + 4 * lane, a.inv_sqrt_d, lane, x);
      if (bad && lane == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_RANGE);
      *reinterpret_cast<float4*>(xs + 4 * lane) = make_float4(x[0], x[1], x[2], x[3]);
    } else if (warp == 8) {
      *reinterpret_cast<float4*>(xs + 128 + 4 * lane) =
          bf16x4_to_float4(*reinterpret_cast<const uint2*>(a.vnew + b * a.vn_sb + hc * a.vn_sh + 4 * lane));
    }
    __syncthreads();
    const int which = warp >> 3, t = tid & 255;
    const int sub = which ? fmt_sub(VB) : fmt_sub(KB), bits = which ? fmt_bits(VB) : fmt_bits(KB);
    const int M = 128 / sub;
    // centroids come from the stream's shared table (filled above, exact fp16 copies of the bf16
    // book): d4b10 = separate table (64-B rows of 8 replicas), d8b8 / d2b8 = the stream's half of
    // the classic 256-B rows (8 x 16 B / 32 x 4 B replicas).  Warp w (of the stream's 8) scans
    // sub-vectors m = w, w + 8, ... (M / 8 of them) against entries jj = lane, lane + 32, ...: each
    // centroid load serves all of the warp's sub-vectors, the running minima stay in registers
    // (independent chains), and one cross-lane reduction per sub-vector ends the scan.  Replica
    // choice: the 32 lanes' loads of one step hit distinct banks.
    auto scan = [&](auto FF, uint32_t base, int st) {
      constexpr int F = decltype(FF)::value;
      constexpr int kSub = fmt_sub(F), kEnt = 1 << fmt_bits(F), kMW = 128 / kSub / 8;
      const int w8 = warp & 7;
      const float* xw = xs + 128 * st;
      float xm[kMW][kSub];
#pragma unroll
      for (int mi = 0; mi < kMW; ++mi)
#pragma unroll
        for (int u = 0; u < kSub; ++u) xm[mi][u] = xw[(w8 + 8 * mi) * kSub + u];
      unsigned long long key[kMW];
#pragma unroll
      for (int mi = 0; mi < kMW; ++mi) key[mi] = ~0ull;
#pragma unroll 4
      for (int jj = lane; jj < kEnt; jj += 32) {
        float c[kSub];
        if constexpr (F == kFmtD4B10) {
          const uint2 w = lds_u64(base + jj * 64 + ((lane >> 1) & 7) * 8);
          const float2 c01 = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
          const float2 c23 = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
          c[0] = c01.x; c[1] = c01.y; c[2] = c23.x; c[3] = c23.y;
        } else if constexpr (F == kFmtD8B8 || F == kFmtD8B12) {
          // d8b8: 8 replicas in the stream's 128-byte half-row; d8b12: unreplicated 16-byte rows
          // (32 consecutive rows per step: conflict-free)
          const uint4 w = F == kFmtD8B8 ? lds_u128(base + jj * 256 + (lane & 7) * 16) : lds_u128(base + jj * 16);
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 cc = __half22float2(*reinterpret_cast<const __half2*>(&ww[u]));
            c[2 * u] = cc.x; c[2 * u + 1] = cc.y;
          }
        } else {   // d2b8
          const uint32_t w = lds_u32(base + jj * 256 + lane * 4);
          const float2 cc = __half22float2(*reinterpret_cast<const __half2*>(&w));
          c[0] = cc.x; c[1] = cc.y;
        }
#pragma unroll
        for (int mi = 0; mi < kMW; ++mi) {
          float ee = __fsub_rn(xm[mi][0], c[0]);
          float dsum = __fmul_rn(ee, ee);
#pragma unroll
          for (int u = 1; u < kSub; ++u) {
            ee = __fsub_rn(xm[mi][u], c[u]);
            dsum = __fadd_rn(dsum, __fmul_rn(ee, ee));
          }
          const unsigned long long k2 = (static_cast<unsigned long long>(__float_as_uint(dsum)) << 32) | static_cast<uint32_t>(jj);
          key[mi] = k2 < key[mi] ? k2 : key[mi];
        }
      }
#pragma unroll
      for (int mi = 0; mi < kMW; ++mi) {
#pragma unroll
        for (int off = 16; off; off >>= 1) {
          const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, key[mi], off);
          key[mi] = o2 < key[mi] ? o2 : key[mi];
        }
        if (lane == 0) gbest[64 * st + w8 + 8 * mi] = key[mi];
      }
    };
    // (a mixed pair's lighter stream finishing early does not matter: the scan is issue-bound, so
    // the heavier stream's warps get the freed issue slots -- handing them part of its entry range
    // was measured neutral)
    if (which == 0) scan(std::integral_constant<int, KB>{}, Fmt<KB>::kSep ? tab_s + kSepOff : tab_s, 0);
    else scan(std::integral_constant<int, VB>{}, Fmt<VB>::kSep ? tab_s + kSepVOff : tab_s + 128, 1);
    __syncthreads();
    // pack: byte i of the row = bits [8i, 8i + 8) of the bit string (b >= 8: <= 2 codes per byte)
    const int rb = M * bits / 8;
    int pgw = 0;
    const bool pok = p_row >= 0 && p_row < a.n_cap && (!paged || ((pgw = page_of(p_row)) >= 0 && pgw < a.n_pages));
    uint8_t* dst = pok ? (which ? a.vcodes_w + row_in(pgw, p_row) * VR : a.kcodes_w + row_in(pgw, p_row) * KR) : nullptr;
    for (int i = t; i < rb; i += 256) {
      const int p = 8 * i, c0 = p / bits, off = p - c0 * bits;
      uint32_t w = static_cast<uint32_t>(gbest[64 * which + c0] & 0xFFFFFFFFull);
      if (c0 + 1 < M) w |= static_cast<uint32_t>(gbest[64 * which + c0 + 1] & 0xFFFFFFFFull) << bits;
      const uint8_t byte = static_cast<uint8_t>(w >> off);
      newcodes[64 * which + i] = byte;
      if (dst) dst[i] = byte;
    }
    if (!pok && t == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_WRITE_POS);
  }
  // residual window rows handled by this warp: t = s + S * (warp + kNW * k), first one preloaded
  // here so its latency hides behind the prologue; the appended row (decode step into the
  // window) is taken from k_new / v_new by its owner warp, which also writes it to the window
  const int rlen = a.res ? min(a.res_lens[b], static_cast<int32_t>(a.r_cap)) : 0;
  const int t_res0 = s + a.S * warp;
  const int64_t res_off = a.res ? b * a.res_sb + hc * a.res_sh : 0;
  // rows of DH bf16: lane l < NL holds key elements 4l..4l+3, thread (r, j) the DH/8 value
  // elements (DH/8) r .. of its accumulator slots (two uint4 at D = 128, one at D = 64)
  uint2 rk = make_uint2(0u, 0u);
  uint4 rv0 = make_uint4(0u, 0u, 0u, 0u), rv1 = rv0;
  auto res_row = [&](int t) {
    const bool is_new = a.res_append && t == rlen - 1;
    const uint16_t* krow = is_new ? a.knew + b * a.kn_sb + hc * a.kn_sh : a.kres + res_off + static_cast<int64_t>(t) * DH;
    const uint16_t* vrow = is_new ? a.vnew + b * a.vn_sb + hc * a.vn_sh : a.vres + res_off + static_cast<int64_t>(t) * DH;
    rk = lane < NL ? *reinterpret_cast<const uint2*>(krow + 4 * lane) : make_uint2(0u, 0u);
    rv0 = *reinterpret_cast<const uint4*>(vrow + (DH / 8) * r);
    if constexpr (DH == 128) rv1 = *reinterpret_cast<const uint4*>(vrow + 16 * r + 8);
    if (is_new && lane < NL) {   // write the new token's raw rows into the window (this warp is the only writer)
      reinterpret_cast<uint2*>(const_cast<uint16_t*>(a.kres) + res_off + static_cast<int64_t>(t) * DH)[lane] = rk;
      reinterpret_cast<uint2*>(const_cast<uint16_t*>(a.vres) + res_off + static_cast<int64_t>(t) * DH)[lane] =
          *reinterpret_cast<const uint2*>(vrow + 4 * lane);
    }
  };
  if (t_res0 < rlen) res_row(t_res0);
  if (warp < 4) {   // Eq. 7 query transform (heads g >= G are zero padding)
    float* dq = sq + kQRow * warp + qoff(lane);
    if (warp < hm.gp) qtransform_lane(qw, lam4, a.qscale, lane, dq, NL);
    else if (lane < NL) *reinterpret_cast<float4*>(dq) = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (TC) {
      // B operand of the tcgen05 score MMA: row 2g = RN16(q~_g), row 2g+1 = RN16(q~_g - hi), dims in
      // natural order (this lane's sub-vector = K elements 4 lane .. 4 lane + 3)
      const float4 v = *reinterpret_cast<const float4*>(dq);
      const float in[4] = {v.x, v.y, v.z, v.w};
      float hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        hi[i] = __half2float(__float2half_rn(in[i]));
        lo[i] = in[i] - hi[i];
      }
      unsigned char* cm = tcb + (lane >> 1) * 2 * 128 + (lane & 1) * 8;
      *reinterpret_cast<uint2*>(cm + (2 * warp) * 16) = make_uint2(pack_half2(hi[0], hi[1]), pack_half2(hi[2], hi[3]));
      *reinterpret_cast<uint2*>(cm + (2 * warp + 1) * 16) = make_uint2(pack_half2(lo[0], lo[1]), pack_half2(lo[2], lo[3]));
      tc::fence_proxy_async_smem();   // generic-proxy stores -> the tensor core reads them
    }
  }
  phase_mark(a.phase, cta_id, 14);   // thread 0: table stored, q~ written (warp 0)
  if constexpr (TC) tc::fence_before();
  __syncthreads();
  if constexpr (TC) tc::fence_after();
  if (kCanAppend && owner) {
    if (warp == 0 || warp == 8) {
      const float* sbest = reinterpret_cast<const float*>(smem_raw + kMiscW + 8192);
      const uint32_t* sidx = reinterpret_cast<const uint32_t*>(smem_raw + kMiscW + 10240);
      float bb = sbest[warp * 32 + lane];
      uint32_t ii = sidx[warp * 32 + lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) {
        const float c = sbest[(warp + w) * 32 + lane];
        if (c < bb) { bb = c; ii = sidx[(warp + w) * 32 + lane]; }
      }
      if (warp == 0) put_code<(KB <= 8 ? KB : 8)>(newcodes, lane, ii, NL);
      else put_code<(VB <= 8 ? VB : 8)>(newcodes + 64, lane, ii, NL);
      int pgw = 0;
      const bool pok = p_row >= 0 && p_row < a.n_cap && (!paged || ((pgw = page_of(p_row)) >= 0 && pgw < a.n_pages));
      if (pok) {
        const int64_t rw = row_in(pgw, p_row);
        if (warp == 0) put_code<(KB <= 8 ? KB : 8)>(a.kcodes_w + rw * KR, lane, ii, NL);
        else put_code<(VB <= 8 ? VB : 8)>(a.vcodes_w + rw * VR, lane, ii, NL);
      } else if (lane == 0 && a.err) {
        atomicOr(a.err, VECINFER_FLAG_WRITE_POS);
      }
    }
    __syncthreads();
  }
  phase_mark(a.phase, cta_id, 1);

  // B fragments of the score MMA: column n = lane/4 <-> (head n/2, part n%2); rows k
  // <-> sub-vector 8j+t, components {0,1} (b0) and {2,3} (b1)
  uint32_t bq0[TC ? 1 : KS], bq1[TC ? 1 : KS];
  if constexpr (!TC) {
    const int gq = r >> 1, part = r & 1;
#pragma unroll
    for (int t = 0; t < KS; ++t) {
      const float4 v = *reinterpret_cast<const float4*>(sq + kQRow * gq + qoff(KS * j + t));
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

  const uint32_t kbase = (kSepK ? tab_s + kSepOff : tab_s) + table_lane_off<KB>(lane);
  const uint32_t vbase = (kSepV ? tab_s + kSepVOff : tab_s + 128) + table_lane_off<VB>(lane);

  float acc[2 * VS][4];
#pragma unroll
  for (int t = 0; t < 2 * VS; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;

  // ---- residual window (NEXT-1): raw bf16 rows scored with the raw q (q k^T = q~ k~^T, Eq. 7),
  // folded into this warp's online-softmax state before the code tiles; the P.V goes into the hi
  // slots of the MMA accumulator layout (thread (r, j) owns head j, dims 16r + 2t + {0, 1})
  if (t_res0 < rlen) {
    float qr[4][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float4 v = (g < hm.gp && lane < NL) ? bf16x4_to_float4(*reinterpret_cast<const uint2*>(
                                                      a.q + b * a.q_sb + (hm.hq0 + g) * a.q_sh + 4 * lane))
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
      qr[g][0] = v.x * a.qscale_raw; qr[g][1] = v.y * a.qscale_raw;
      qr[g][2] = v.z * a.qscale_raw; qr[g][3] = v.w * a.qscale_raw;
    }
    for (int t = t_res0; t < rlen; t += a.S * kNW) {
      if (t != t_res0) res_row(t);   // rows beyond the first (long windows, few splits)
      const float4 kv = bf16x4_to_float4(rk);
      float sg[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float v = qr[g][0] * kv.x + qr[g][1] * kv.y + qr[g][2] * kv.z + qr[g][3] * kv.w;
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        sg[g] = v;
      }
      const float sj = j == 0 ? sg[0] : j == 1 ? sg[1] : j == 2 ? sg[2] : sg[3];
      if (sj > m_run + kTau) {   // per-lane: all 8 lanes of head j agree
        const float alpha = ex2_approx(m_run - sj);
#pragma unroll
        for (int tt = 0; tt < 2 * VS; ++tt) {
          acc[tt][0] *= alpha; acc[tt][1] *= alpha; acc[tt][2] *= alpha; acc[tt][3] *= alpha;
        }
        l_run *= alpha;
        m_run = sj;
      }
      const float p = ex2_approx(sj - m_run);
      if (r == 0) l_run += p;                         // once per head (lanes r = 0 of each j)
      const uint32_t vw[8] = {rv0.x, rv0.y, rv0.z, rv0.w, rv1.x, rv1.y, rv1.z, rv1.w};
#pragma unroll
      for (int tt = 0; tt < 2 * VS; ++tt) {
        acc[tt][0] += p * __uint_as_float(vw[tt] << 16);             // dim (DH/8) r + 2tt
        acc[tt][2] += p * __uint_as_float(vw[tt] & 0xFFFF0000u);     // dim (DH/8) r + 2tt + 1
      }
    }
  }

  // mask of a ragged tile, online softmax (Alg. 1 l.12-13, 18) and P.V (l.16) of one 32-token tile
  // given its scores sc[q][0/1] (tokens 16q + r / 16q + r + 8, head j; mma accumulator layout)
  auto softmax_pv = [&](float (&sc)[2][2], const TileCodes<KB, VB>& cur, int rem_cur) {
    if (rem_cur < 32) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (16 * q + r >= rem_cur) sc[q][0] = -INFINITY;
        if (16 * q + r + 8 >= rem_cur) sc[q][1] = -INFINITY;
      }
    }

    // ---- online softmax (Alg. 1 l.12-13, 18), lazy rescale.  Common path: every lane checks its
    // own 4 scores against m_run + tau (p <= 2^tau) -- no cross-lane traffic; only when some lane
    // exceeds it are the per-head tile maxima reduced and the accumulators rescaled.
    float mx = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
    if (__any_sync(0xffffffffu, mx > m_run + kTau)) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const bool need = mx > m_run + kTau;           // uniform across the 8 lanes of head j
      const float m_new = need ? mx : m_run;
      const float alpha = need ? ex2_approx(m_run - m_new) : 1.f;  // 0 when m_run was -inf
#pragma unroll
      for (int t = 0; t < 2 * VS; ++t) {
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
      // hi/lo fp16 split: hi = RN16(p), lo = RN16(p - hi)
      const __half2 hh = __floats2half2_rn(p0, p1);
      const float2 hf = __half22float2(hh);
      const __half2 ll = __floats2half2_rn(p0 - hf.x, p1 - hf.y);
      const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hh);
      const uint32_t lb = *reinterpret_cast<const uint32_t*>(&ll);
      const uint32_t bp0 = movmatrix_trans(prmt(hb, lb, 0x5410));  // (hi, lo) of token r
      const uint32_t bp1 = movmatrix_trans(prmt(hb, lb, 0x7632));  // (hi, lo) of token r + 8

      // ---- P.V (Alg. 1 l.16): m-tile t <-> sub-vector VS*r + t/2, components 2(t%2) + {0,1}
      auto pv = [&](auto U, const uint2& g0, const uint2& g1, const uint2& g2, const uint2& g3) {
        constexpr int u = decltype(U)::value;
        mma_16816(acc[2 * u], prmt(g0.x, g1.x, 0x5410), prmt(g0.x, g1.x, 0x7632), prmt(g2.x, g3.x, 0x5410),
                  prmt(g2.x, g3.x, 0x7632), bp0, bp1);
        mma_16816(acc[2 * u + 1], prmt(g0.y, g1.y, 0x5410), prmt(g0.y, g1.y, 0x7632), prmt(g2.y, g3.y, 0x5410),
                  prmt(g2.y, g3.y, 0x7632), bp0, bp1);
      };
      if constexpr (Fmt<VB>::kWide) {   // d8b8: code i of the V chunk = virtual sub-vectors 2i, 2i+1
        static_for<0, VS / 2>([&](auto I) {
          constexpr int i = decltype(I)::value;
          const uint4 w0 = lds_u128(Fmt<VB>::template vaddr<i>(cur.v[q][0], vbase));
          const uint4 w1 = lds_u128(Fmt<VB>::template vaddr<i>(cur.v[q][1], vbase));
          const uint4 w2 = lds_u128(Fmt<VB>::template vaddr<i>(cur.v[q][2], vbase));
          const uint4 w3 = lds_u128(Fmt<VB>::template vaddr<i>(cur.v[q][3], vbase));
          pv(std::integral_constant<int, 2 * i>{}, make_uint2(w0.x, w0.y), make_uint2(w1.x, w1.y), make_uint2(w2.x, w2.y),
             make_uint2(w3.x, w3.y));
          pv(std::integral_constant<int, 2 * i + 1>{}, make_uint2(w0.z, w0.w), make_uint2(w1.z, w1.w), make_uint2(w2.z, w2.w), make_uint2(w3.z, w3.w));
        });
      } else {
        static_for<0, VS>([&](auto U) {
          constexpr int u = decltype(U)::value;
          pv(U, gather_v<VB, u>(cur.v[q][0], vbase, cbv), gather_v<VB, u>(cur.v[q][1], vbase, cbv),
             gather_v<VB, u>(cur.v[q][2], vbase, cbv), gather_v<VB, u>(cur.v[q][3], vbase, cbv));
        });
      }
    }
  };

  if constexpr (!TC) {
    for (int it = warp; it < ntile; it += kNW) {
      TileCodes<KB, VB> cur;
      if constexpr (!kTma) {
        cur = nxt;
      } else if (tma_on) {   // wait for the stage, read the tile's fragments, refill the stage
        const uint32_t st = n_con % kTmaSt, par = (n_con / kTmaSt) & 1u;
        ++n_con;
        tc::mbar_wait(tma_bar + 8 * st, par);
        const int rem = ntok - 32 * it;
        const uint32_t kb = tma_stg + st * kTmaStage + r * KR + FK::kOffK * j;
        const uint32_t vb = tma_stg + st * kTmaStage + kTmaStage / 2 + 2 * j * VR + FV::kOffV * r;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const bool full = rem >= 32;
          cur.k[q][0] = (full || 16 * q + r < rem) ? lds_u64(kb + (16 * q) * KR) : Fmt<KB>::zk();
          cur.k[q][1] = (full || 16 * q + r + 8 < rem) ? lds_u64(kb + (16 * q + 8) * KR) : Fmt<KB>::zk();
          const int t0 = 16 * q + 2 * j;
          cur.v[q][0] = (full || t0 < rem) ? lds_u32(vb + (16 * q) * VR) : VCode<VB>{};
          cur.v[q][1] = (full || t0 + 1 < rem) ? lds_u32(vb + (16 * q + 1) * VR) : VCode<VB>{};
          cur.v[q][2] = (full || t0 + 8 < rem) ? lds_u32(vb + (16 * q + 8) * VR) : VCode<VB>{};
          cur.v[q][3] = (full || t0 + 9 < rem) ? lds_u32(vb + (16 * q + 9) * VR) : VCode<VB>{};
        }
        __syncwarp();   // every lane has read the stage before the async proxy overwrites it
        if (it + kNW * kTmaSt < ntile) {
          if (lane == 0) tc::fence_proxy_async_smem();
          tma_issue(it + kNW * kTmaSt);
        }
      } else {
        cur = nxt;
      }
      if constexpr (kCanAppend || kGenAppend) {
      if (it == patch_tile) {   // the appended row: codes just encoded, not the stale load
        const KCode<KB> nk = new_kchunk<KB, DH>(newcodes, j);
        const VCode<VB> nv = new_vchunk<VB, DH>(newcodes + 64, r);
        const int qp = patch_row >> 4, rr = patch_row & 15;
  #pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q != qp) continue;
          if (r == rr) cur.k[q][0] = nk;
          if (r + 8 == rr) cur.k[q][1] = nk;
          if (2 * j == rr) cur.v[q][0] = nv;
          if (2 * j + 1 == rr) cur.v[q][1] = nv;
          if (2 * j + 8 == rr) cur.v[q][2] = nv;
          if (2 * j + 9 == rr) cur.v[q][3] = nv;
        }
      }
      }
      const int rem_cur = ntok - 32 * it;
      auto issue_next = [&]() {
      if (!tma_on && it + kNW < ntile) {
        if constexpr (paged) {   // row (pg * Hc + hc) * page_size + tok % page_size: 32 x 32 -> 64-bit multiply-adds
          const int tok = static_cast<int>(r0) + 32 * (it + kNW);
          const uint32_t prow = static_cast<uint32_t>(pg_ahead) * static_cast<uint32_t>(a.Hc) + static_cast<uint32_t>(hc);
          const uint32_t tin = static_cast<uint32_t>(tok) & ((1u << a.page_shift) - 1u);
          kp = kcb + static_cast<uint64_t>(prow) * (static_cast<uint32_t>(KR) << a.page_shift) + tin * KR;
          vp = vcb + static_cast<uint64_t>(prow) * (static_cast<uint32_t>(VR) << a.page_shift) + tin * VR;
          if (it + 2 * kNW < ntile) pg_ahead = __ldg(a.bt + b * a.bt_stride + ((tok + 32 * kNW) >> a.page_shift));
        } else {
          kp += kStepK;
          vp += kStepV;
        }
        const int rem = rem_cur - 32 * kNW;
        if (rem >= 32) load_tile_full<KB, VB, DH>(nxt, kp, vp);
        else load_tile_tail<KB, VB, DH>(nxt, kp, vp, rem, r, j);
      }
      };
      if constexpr (!kLateNext) issue_next();
  
      // ---- scores (log2 units) for tile tokens 16q + {r, r+8}, head j; two independent MMA
      // accumulator chains per sub-tile (k-steps 0-3 and 4-7) halve the dependent HMMA latency
      float sc[2][2];
  #pragma unroll
      for (int q = 0; q < 2; ++q) {
        float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (Fmt<KB>::kWide) {   // d8b8: one 16-byte gather = virtual sub-vectors 2i, 2i+1
          static_for<0, KS / 2>([&](auto I) {
            constexpr int i = decltype(I)::value, t = 2 * i;
            const uint4 wa = lds_u128(Fmt<KB>::template kaddr<i>(cur.k[q][0], kbase));
            const uint4 wb = lds_u128(Fmt<KB>::template kaddr<i>(cur.k[q][1], kbase));
            if (t < KS / 2) {
              mma_16816(d0, wa.x, wb.x, wa.y, wb.y, bq0[t], bq1[t]);
              mma_16816(d0, wa.z, wb.z, wa.w, wb.w, bq0[t + 1], bq1[t + 1]);
            } else {
              mma_16816(d1, wa.x, wb.x, wa.y, wb.y, bq0[t], bq1[t]);
              mma_16816(d1, wa.z, wb.z, wa.w, wb.w, bq0[t + 1], bq1[t + 1]);
            }
          });
        } else {
          static_for<0, KS>([&](auto T) {
            constexpr int t = decltype(T)::value;
            const uint2 ea = gather_k<KB, t>(cur.k[q][0], kbase, cbk);
            const uint2 eb = gather_k<KB, t>(cur.k[q][1], kbase, cbk);
            if (t < KS / 2) mma_16816(d0, ea.x, eb.x, ea.y, eb.y, bq0[t], bq1[t]);
            else mma_16816(d1, ea.x, eb.x, ea.y, eb.y, bq0[t], bq1[t]);
          });
        }
        sc[q][0] = (d0[0] + d1[0]) + (d0[1] + d1[1]);
        sc[q][1] = (d0[2] + d1[2]) + (d0[3] + d1[3]);
      }
      softmax_pv(sc, cur, rem_cur);
      if constexpr (kLateNext) issue_next();
    }
  }
  if constexpr (TC) {
    // tcgen05 score path.  Group g = warps 4g..4g+3 (TMEM lane quarters 0..3) processes 128-token
    // chunks; warp 4g+k owns tile it = 4g + k + 16n of iteration n (the same tiles as the mma.sync
    // path).  Per tile: every lane gathers the 32 centroids of ITS token (row = lane) into TMEM
    // columns [64g, 64g + 64) (tcgen05.st, no LSU traffic), the group meets at a named barrier and
    // one thread issues 8 MMAs (M = 128 tokens, N = 16 = 4 heads x {hi, lo} + 8 zero rows, K = 16
    // dims each) committed to the group's mbarrier; the scores come back with tcgen05.ld.16x256b in
    // the mma.sync accumulator layout, so the softmax and the P.V are the same code as above.
    // Software pipeline: MMA(n + 1) is issued before the softmax / P.V of tile n (one A buffer:
    // tile n + 1 is staged only after MMA(n) completed; one D buffer: read before the barrier).
    // warp-uniform by construction (shuffle from lane 0): lets the compiler keep the TMEM addresses
    // and the barrier ids in uniform registers
    const int wu = __shfl_sync(0xffffffffu, warp, 0);
    const int grp = wu >> 2, quarter = wu & 3;
    const int n_g = ntile > 4 * grp ? (ntile - 4 * grp + kNW - 1) / kNW : 0;
    const uint32_t tmem = tc_misc[0];
    const uint32_t lane_sh = static_cast<uint32_t>(32 * quarter) << 16;
    const uint32_t t_a = tmem + 64 * grp, t_d = tmem + 256 + 16 * grp;
    const uint32_t mbar = smem_u32(tc_misc + 2 + 2 * grp);
    const uint32_t b_s = smem_u32(tcb);
    constexpr uint32_t kIdesc = tc::idesc_f16_f32<128, 16>();
    auto issue_scores = [&](const KRowT<KB>& kr, int it) {
      if (it < ntile) {
        KRowT<KB> k = kr;
        if constexpr (kCanAppend) {
          if (it == patch_tile && lane == patch_row) {   // the appended row: codes just encoded
#pragma unroll
            for (int i = 0; i < KR / 16; ++i) k.w[i] = *reinterpret_cast<const uint4*>(newcodes + 16 * i);
          }
        }
        // 4 chunks of 8 sub-vectors (16 TMEM columns); the gathers of chunk c + 1 are in flight
        // while chunk c is stored
        auto gather = [&](auto C, uint32_t (&v)[16]) {
          constexpr int c = decltype(C)::value;
          static_for<0, 8>([&](auto MM) {
            constexpr int mm = decltype(MM)::value;
            const uint2 e = lds_u64(krow_addr<KB, 8 * c + mm>(k, kbase));
            v[2 * mm] = e.x;
            v[2 * mm + 1] = e.y;
          });
        };
        uint32_t va[16], vb[16];
#if VECINFER_TC_EXP == 2   // timing experiment: gathers kept, no TMEM stores
        uint32_t x = 0;
        gather(std::integral_constant<int, 0>{}, va); gather(std::integral_constant<int, 1>{}, vb);
        for (int i = 0; i < 16; ++i) x ^= va[i] ^ vb[i];
        gather(std::integral_constant<int, 2>{}, va); gather(std::integral_constant<int, 3>{}, vb);
        for (int i = 0; i < 16; ++i) x ^= va[i] ^ vb[i];
        if (x == 0x12345678u) tc::st_32x32b_x16(t_a + lane_sh, va);
#else
        gather(std::integral_constant<int, 0>{}, va);
        gather(std::integral_constant<int, 1>{}, vb);
        tc::st_32x32b_x16(t_a + lane_sh, va);
        gather(std::integral_constant<int, 2>{}, va);
        tc::st_32x32b_x16(t_a + lane_sh + 16, vb);
        gather(std::integral_constant<int, 3>{}, vb);
        tc::st_32x32b_x16(t_a + lane_sh + 32, va);
        tc::st_32x32b_x16(t_a + lane_sh + 48, vb);
#endif
#if VECINFER_TC_EXP != 1   // (1: timing experiment without the store wait)
        tc::wait_st();
#endif
      }
      tc::fence_before();
      // the group's quarter-0 warp waits for the other three and issues; they only arrive (their
      // next TMEM write follows the wait for this MMA, so the barrier phases cannot overlap)
      if (quarter == 0) {
#if VECINFER_TC_EXP != 3   // (3: timing experiment without the group barrier)
        tc::bar_sync(1 + grp, 128);
#endif
        tc::fence_after();
        if (lane == 0) {
#pragma unroll
          for (int s8 = 0; s8 < (VECINFER_TC_EXP == 4 ? 0 : 8); ++s8)   // (4: timing experiment, no MMA)
            tc::mma_f16_ts(t_d, t_a + 8 * s8, tc::smem_desc_kmajor(b_s + 512 * s8, 256, 128), kIdesc, s8 > 0 ? 1u : 0u);
          tc::commit(mbar);
        }
      } else {
#if VECINFER_TC_EXP != 3
        tc::bar_arrive(1 + grp, 128);
#endif
      }
    };
    KRowT<KB> kn1 = kfirst1;   // K row of the warp's next tile
    TileCodes<KB, VB> cur = nxt;   // V codes of the current tile
    if (n_g > 0) issue_scores(kfirst0, warp);
    for (int n = 0; n < n_g; ++n) {
      const int it = warp + kNW * n;
      const int rem_cur = ntok - 32 * it;
      KRowT<KB> kn2;
      if (it + 2 * kNW < ntile) load_krow(kn2, it + 2 * kNW);   // K row of tile n + 2 (MMA(n + 2))
      tc::mbar_wait(mbar, tc_phase & 1u);
      ++tc_phase;
      tc::fence_after();
      float sc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
      if (it < ntile && VECINFER_TC_EXP != 5) {   // (5: timing experiment, no TMEM load)
        float d0[4], d1[4];
        tc::ld_16x256b(t_d + lane_sh, d0);                // tokens r, r + 8 (cols 2j, 2j+1 = head j hi, lo)
        tc::ld_16x256b(t_d + lane_sh + (16u << 16), d1);  // tokens 16 + r, 16 + r + 8
        tc::wait_ld();
        sc[0][0] = d0[0] + d0[1];
        sc[0][1] = d0[2] + d0[3];
        sc[1][0] = d1[0] + d1[1];
        sc[1][1] = d1[2] + d1[3];
      }
      if (n + 1 < n_g) issue_scores(kn1, it + kNW);
      if (it + kNW < ntile) load_vtile(nxt, it + kNW);   // V codes of tile n + 1
      if (it < ntile) {
        if constexpr (kCanAppend) {
          if (it == patch_tile) {   // the appended row's V codes
            const VCode<VB> nv = new_vchunk<VB, DH>(newcodes + 64, r);
            const int qp = patch_row >> 4, rr = patch_row & 15;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              if (q != qp) continue;
              if (2 * j == rr) cur.v[q][0] = nv;
              if (2 * j + 1 == rr) cur.v[q][1] = nv;
              if (2 * j + 8 == rr) cur.v[q][2] = nv;
              if (2 * j + 9 == rr) cur.v[q][3] = nv;
            }
          }
        }
        softmax_pv(sc, cur, rem_cur);
      }
      kn1 = kn2;
      cur = nxt;
    }
  }
  // ---- warp partials -> shared memory, rescaled to the CTA-wide running max of each head: every
  // warp posts m_run, reads the 16 maxima back and stores f*acc, f*l with f = 2^(m_run - M), so the
  // combine (cta_finish<PRESCALED>, or the cluster path with f = 1) is a max over wm plus a plain
  // sum over the warps
  phase_mark(a.phase, cta_id, 2);
  griddep_launch_dependents();   // the next kernel may start its (static) prologue
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 4);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 8);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
  float* wm = reinterpret_cast<float*>(smem_raw + kMiscW);
  float* wl = wm + kNW * 4;
  float* wacc = wl + kNW * 4;
  if (r == 0) wm[warp * 4 + j] = m_run;
  __syncthreads();
  // CTA max of head j: lanes (r, j) read warps r and r + 8, then a max over the 8 lanes of head j
  float Mh = fmaxf(wm[r * 4 + j], wm[(r + 8) * 4 + j]);
  Mh = fmaxf(Mh, __shfl_xor_sync(0xffffffffu, Mh, 4));
  Mh = fmaxf(Mh, __shfl_xor_sync(0xffffffffu, Mh, 8));
  Mh = fmaxf(Mh, __shfl_xor_sync(0xffffffffu, Mh, 16));
  const float fsc = m_run == -INFINITY ? 0.f : ex2_approx(m_run - Mh);
  if (r == 0) wl[warp * 4 + j] = l_run * fsc;   // (wm keeps the per-warp maxima: no write-after-read race)
  // thread (r, j): head j, dims (DH/8)r .. (DH/8)r + DH/8 - 1; MMA slots [t][0] + [t][1] hold dim
  // (DH/8)r + 2t, [t][2] + [t][3] dim (DH/8)r + 2t + 1 (hi + lo parts)
  float* dst = wacc + (warp * 4 + j) * kWRow + (DH / 8) * r;
#pragma unroll
  for (int k = 0; k < VS; ++k)
    *reinterpret_cast<float4*>(dst + 4 * k) =
        make_float4((acc[2 * k][0] + acc[2 * k][1]) * fsc, (acc[2 * k][2] + acc[2 * k][3]) * fsc,
                    (acc[2 * k + 1][0] + acc[2 * k + 1][1]) * fsc, (acc[2 * k + 1][2] + acc[2 * k + 1][3]) * fsc);
  __syncthreads();
  phase_mark(a.phase, cta_id, 3);
  if (!a.cluster) {
    cta_finish<kThreads, kNW, kWRow, DH, true, XR>(a, b, h, s, wm, wl, wacc, reinterpret_cast<float*>(tab));
    phase_mark(a.phase, cta_id, 4);
    continue;
  }
  // ---- cluster path: the S splits of (b, h) are one cluster; each CTA combines its warps and
  // pushes (M, l, acc[4][128]) into the leader's buffer over DSMEM; one cluster barrier; the
  // leader merges the S partials in rank order (deterministic) and writes o and the LSE.
  {
    const int g = tid >> 7, dim = tid & 127;     // 512 threads <-> 4 heads x 128 dims
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kNW; ++w) M = fmaxf(M, wm[w * 4 + g]);
    float osum = 0.f, lsum = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kNW; ++w) {
        const float f = 1.f;   // partials are pre-scaled to the CTA max M
        lsum += f * wl[w * 4 + g];
        osum += f * wacc[(w * 4 + g) * kWRow + dim];
      }
    }
    cluster_wait();   // every CTA of the cluster has started: DSMEM of the leader is valid
    const uint32_t rank = cluster_ctarank();
    float* cbuf = reinterpret_cast<float*>(tab + kCbufOff);   // [16][4][128] acc, [16][4] M, l
    float* cM = cbuf + kClusterMax * 4 * 128;
    float* cL = cM + kClusterMax * 4;
    const uint32_t cb_s = smem_u32(cbuf);
    st_cluster_f32(mapa_shared(cb_s + 4u * ((rank * 4 + g) * 128 + dim), 0), osum);
    if (dim == 0) {
      st_cluster_f32(mapa_shared(smem_u32(cM + rank * 4 + g), 0), M);
      st_cluster_f32(mapa_shared(smem_u32(cL + rank * 4 + g), 0), lsum);
    }
    cluster_sync_all();
    phase_mark(a.phase, cta_id, 5);
    if (rank == 0 && g < hm.gp) {
      float Mx = -INFINITY;
      for (int q = 0; q < a.S; ++q) Mx = fmaxf(Mx, cM[q * 4 + g]);
      float os = 0.f, ls = 0.f;
      if (Mx != -INFINITY) {
        for (int q = 0; q < a.S; ++q) {
          const float f = ex2_approx(cM[q * 4 + g] - Mx);
          ls += f * cL[q * 4 + g];
          os += f * cbuf[(q * 4 + g) * 128 + dim];
        }
      }
      const bool empty = !(ls > 0.f);
      const int64_t oi = (static_cast<int64_t>(b) * a.Hq + hm.hq0 + g) * 128 + dim;
      const float ov = empty ? 0.f : os / ls;
      if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
      else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
      if (dim == 0 && a.lse) a.lse[static_cast<int64_t>(b) * a.Hq + hm.hq0 + g] = empty ? -INFINITY : (Mx + __log2f(ls)) * kLn2;
    }
  }
  phase_mark(a.phase, cta_id, 4);
  }  // item loop
  if constexpr (TC) {   // every issued MMA was waited for; all TMEM reads are done after this barrier
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::dealloc(tc_misc[0], kTmemCols);
  }
}

}  // namespace

using AttnKernel = void (*)(const AttnArgs);

static int smem_for(int kf, int vf) { return smem_layout_bytes(kf, vf); }

// the NEXT-2 (K, V) format pairs with a kernel: each format with itself and the paper's mixed
// configurations K-d4b10 / V-d8b12 (2-bit) and K-d8b12 / V-d8b8 (1.25-bit), Table 3 / P:993-999
#define VECINFER_NEXT2_PAIRS(X)                                                   \
  X(kFmtD8B8, kFmtD8B8) X(kFmtD8B12, kFmtD8B12) X(kFmtD4B10, kFmtD4B10)           \
  X(kFmtD2B8, kFmtD2B8) X(kFmtD4B10, kFmtD8B12) X(kFmtD8B12, kFmtD8B8) X(kFmtD8B16, kFmtD8B16)

// tcgen05 score path (VECINFER_ATTN_DEQUANT_TC; the host validated the formats: d = 4 shared-table K
// codebooks, D = 128, contiguous caches)
static AttnKernel kernel_tc(int kf, int vf) {
  static const AttnKernel table[2][3] = {
      {attn_mma_kernel<4, 4, 128, true>, attn_mma_kernel<4, 8, 128, true>, attn_mma_kernel<4, 16, 128, true>},
      {attn_mma_kernel<8, 4, 128, true>, attn_mma_kernel<8, 8, 128, true>, attn_mma_kernel<8, 16, 128, true>}};
  return table[kf == 8 ? 1 : 0][vf == 4 ? 0 : vf == 8 ? 1 : 2];
}

template <bool PG>
static AttnKernel kernel_for_t(int kf, int vf, int dh) {
#define VECINFER_PAIR(K, V) \
  if (kf == K && vf == V) return dh == 128 ? attn_mma_kernel<K, V, 128, false, false, PG> : nullptr;
  VECINFER_NEXT2_PAIRS(VECINFER_PAIR)
#undef VECINFER_PAIR
  const int ki = kf == 4 ? 0 : kf == 8 ? 1 : kf == 16 ? 2 : -1, vi = vf == 4 ? 0 : vf == 8 ? 1 : vf == 16 ? 2 : -1;
  if (ki < 0 || vi < 0) return nullptr;
  static const AttnKernel table[2][3][3] = {
      {{attn_mma_kernel<4, 4, 128, false, false, PG>, attn_mma_kernel<4, 8, 128, false, false, PG>,
        attn_mma_kernel<4, 16, 128, false, false, PG>},
       {attn_mma_kernel<8, 4, 128, false, false, PG>, attn_mma_kernel<8, 8, 128, false, false, PG>,
        attn_mma_kernel<8, 16, 128, false, false, PG>},
       {attn_mma_kernel<16, 4, 128, false, false, PG>, attn_mma_kernel<16, 8, 128, false, false, PG>,
        attn_mma_kernel<16, 16, 128, false, false, PG>}},
      {{attn_mma_kernel<4, 4, 64, false, false, PG>, attn_mma_kernel<4, 8, 64, false, false, PG>,
        attn_mma_kernel<4, 16, 64, false, false, PG>},
       {attn_mma_kernel<8, 4, 64, false, false, PG>, attn_mma_kernel<8, 8, 64, false, false, PG>,
        attn_mma_kernel<8, 16, 64, false, false, PG>},
       {attn_mma_kernel<16, 4, 64, false, false, PG>, attn_mma_kernel<16, 8, 64, false, false, PG>,
        attn_mma_kernel<16, 16, 64, false, false, PG>}}};
  return table[dh == 64 ? 1 : 0][ki][vi];
}
static AttnKernel kernel_for(int kf, int vf, int dh = 128, bool pg = false) {
  return pg ? kernel_for_t<true>(kf, vf, dh) : kernel_for_t<false>(kf, vf, dh);
}

// fused cross-rank merge variants: d = 4 K / V books, D = 128
static AttnKernel kernel_xr(int kf, int vf) {
  const int ki = kf == 4 ? 0 : kf == 8 ? 1 : kf == 16 ? 2 : -1, vi = vf == 4 ? 0 : vf == 8 ? 1 : vf == 16 ? 2 : -1;
  if (ki < 0 || vi < 0) return nullptr;
  static const AttnKernel table[3][3] = {
      {attn_mma_kernel<4, 4, 128, false, true>, attn_mma_kernel<4, 8, 128, false, true>,
       attn_mma_kernel<4, 16, 128, false, true>},
      {attn_mma_kernel<8, 4, 128, false, true>, attn_mma_kernel<8, 8, 128, false, true>,
       attn_mma_kernel<8, 16, 128, false, true>},
      {attn_mma_kernel<16, 4, 128, false, true>, attn_mma_kernel<16, 8, 128, false, true>,
       attn_mma_kernel<16, 16, 128, false, true>}};
  return table[ki][vi];
}

static void set_attr(AttnKernel k, int smem) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // carveout = the smallest that fits: the rest of the 256 KiB stays L1 (16-bit books live there)
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxL1);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

static void set_attrs_once() {
  static bool done = false;  // benign race: idempotent attributes
  if (!done) {
    for (int dh : {128, 64})
      for (int kb : {4, 8, 16})
        for (int vb : {4, 8, 16})
          for (bool pg : {false, true}) set_attr(kernel_for(kb, vb, dh, pg), smem_for(kb, vb));
    for (int kb : {4, 8})
      for (int vb : {4, 8, 16}) set_attr(kernel_tc(kb, vb), smem_for(kb, vb));
    for (int kb : {4, 8, 16})
      for (int vb : {4, 8, 16}) set_attr(kernel_xr(kb, vb), smem_for(kb, vb));
#define VECINFER_PAIR(K, V) set_attr(kernel_for(K, V), smem_for(K, V)); set_attr(kernel_for(K, V, 128, true), smem_for(K, V));
    VECINFER_NEXT2_PAIRS(VECINFER_PAIR)
#undef VECINFER_PAIR
    done = true;
  }
}

bool attn_mma_supports(int kfmt, int vfmt, int dh) { return kernel_for(kfmt, vfmt, dh) != nullptr; }

int attn_mma_max_active_clusters(int cluster_size) {
  static int cache[kClusterMax + 1] = {0};
  if (cluster_size < 1 || cluster_size > kClusterMax) return 0;
  if (cache[cluster_size] == 0) {
    set_attrs_once();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster_size, 64, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kernel_for(8, 8), &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[cluster_size] = n > 0 ? n : -1;
  }
  return cache[cluster_size] > 0 ? cache[cluster_size] : 0;
}

cudaError_t launch_attn_mma(const AttnArgs& a, int kbits, int vbits, cudaStream_t st) {
  // kbits / vbits: format ids (b for d = 4, else 100d + b)
  set_attrs_once();
  cudaLaunchConfig_t cfg = {};
  if (a.cluster) {
    cfg.gridDim = dim3(a.S, a.Hkv, a.B);
  } else {
    const int sms = device_sm_count();
    cfg.gridDim = dim3(a.n_items < sms ? a.n_items : sms, 1, 1);   // persistent beyond one wave
  }
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem_for(kbits, vbits);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (a.cluster) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = a.S;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  const AttnKernel k = a.xr_P > 0 ? kernel_xr(kbits, vbits) : a.tc ? kernel_tc(kbits, vbits) : kernel_for(kbits, vbits, a.D, a.bt != nullptr);
  if (!k) return cudaErrorInvalidDeviceFunction;
  return cudaLaunchKernelEx(&cfg, k, a);
}

}  // namespace vecinfer
