// N3+N4+N5: fused VQ decode attention, DEQUANT_MMA algorithm, stream-partition kernel (batch decode:
// B*H_kv >= #SMs).  The split kernel for fewer units is attn_mma.cu; both share attn_tiles.cuh.
//
// Implements Eq. 10 with Algorithm 1's online softmax:
//   s = q~ VQ^-1(K~_q)^T / sqrt(D),  o = softmax(s) VQ^-1(V_q),  L = logsumexp(s).
//
// Work partition (stream-K over units, "fractional splits").  The U = B*H_kv units (b, h_kv)
// and the V virtual CTAs tile the same line of U*V ticks: unit u owns [u*V, (u+1)*V), CTA c owns
// [c*U, (c+1)*U).  Every CTA therefore gets the same share of the total work whatever U is; a
// unit crossed by CTA boundaries is split into pieces (one per CTA touching it) whose token
// ranges follow the tick boundaries (rounded down to 16 tokens).  V <= #SMs: one CTA per SM, all
// co-resident; explicit num_splits S gives V = U*S (pieces = the classic S splits; V > #SMs runs
// persistent CTAs).  A CTA processes its segments (unit intersections) in rounds of up to two:
// the round's 16-token sub-tiles are spread evenly over the 16 warps in contiguous ranges, one warp
// may straddle the two segments (it flushes its softmax state in between), and each segment has
// its own codebook table (two 64 KiB tables).  Partials of split units are merged in fixed piece
// order by log-sum-exp (spin: every piece merges a slice after all arrived; last: the last piece).
//
// Per warp and 16-token sub-tile (codes stream from HBM straight into registers, one 32-token
// tile of prefetch -- no dequantised cache, no shared-memory staging of codes):
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
// See DESIGN.md "Kernel N4".
#include "attn_tiles.cuh"

namespace vecinfer {
namespace {

// misc region (below the tables, which start at the next 64 KiB boundary of the shared window)
constexpr int kWRow = 132;         // row stride (floats) of the warp partials: conflict-free 16-B stores
constexpr int kSlots = 17;         // warp partial slots: warp w's last piece -> w, the straddler's first -> 16
constexpr int kQSeg = 4 * kQRow;   // q~ rows of a segment (kQRow, qoff: attn_common.cuh)
constexpr int kMiscQ = 0;          // q~ [2 segments][4][kQRow] f32
constexpr int kMiscNew = 5376;     // appended-token codes [2][128 B] (K at +0, V at +64)
constexpr int kMiscWM = 5632;      // wm [17][4] f32 (log2-domain running max per warp piece)
constexpr int kMiscWL = 6144;      // wl [17][4] f32
constexpr int kMiscSeg = 6656;     // SegSh [2], RoundSh
constexpr int kMiscFlag = 6912;    // merge bookkeeping (ints)
constexpr int kMiscStage = 7424;   // append encode: float4 [16 warps][32] centroids, dist [16][32],
                                   // index [16][32]; later combine weights / merge staging
constexpr int kMiscBest = kMiscStage + 8192;
constexpr int kMiscIdx = kMiscBest + 2048;
constexpr int kStageBytes = 12288;
constexpr int kMiscW = kMiscStage + kStageBytes;   // warp partials [17][4][132] f32
constexpr int kMiscBytes = kMiscW + kSlots * 4 * kWRow * 4;   // 54336
constexpr int kSmemBytes = 65536 + 2 * kTab + 1024;  // misc (below 64 KiB) + 2 tables + slack
constexpr int kSmemBytesNoTab = kMiscBytes + 1024;  // 16-bit K and V: codebooks in L1/L2

// one segment = the intersection of a CTA with a unit (computed once per round, shared)
struct SegSh {
  long long t0, t1;    // token rows [t0, t1) of the unit handled by this piece
  long long p_row;     // append row (write_pos[b]) when appending
  long long res_off;   // element offset of the unit's residual rows
  int u, b, h;         // unit, batch, virtual KV head (head_map: GQA groups > 4)
  int hc, hq0, gp;     // KV head of the codes, first query head, query heads (<= 4)
  int cu;              // cache unit b * Hc + hc (code rows)
  int k, P;            // piece index and number of pieces of the unit
  int rlen;            // residual rows of the unit
  int owner;           // this piece encodes the appended token
  int patch;           // ... and the appended row lies in [t0, t1) (read from registers, not HBM)
};
// warp assignment of a round (written by one thread, re-read through volatile loads so that none
// of it stays live in registers across the main loop)
struct RoundSh {
  int nsA, ns;     // sub-tiles of segment A, of the round
  int nwA, b0;     // segment A = warps [0, nwA), segment B = warps [b0, 16)
  int strad;       // the warp in both (-1: none)
  int sameB;       // segment B reuses table A (same codebooks)
  int pad[2];
};
static_assert(sizeof(SegSh) * 2 + sizeof(RoundSh) <= kMiscFlag - kMiscSeg, "SegSh/RoundSh");
static_assert(2 * kQSeg * 4 <= kMiscNew, "q~ rows");

// token offset (within the unit's attended range of n tokens) of local tick tau in [0, V]:
// proportional, rounded down to 16 tokens; X = extra virtual tokens at the end of the range that
// account for the encode of the appended row so its piece is not the straggler
// Xs = virtual tokens at the START of a split unit that stand for the fixed cost of a segment
// (table fill, first-tile latency, combine): a CTA gets one more segment per unit start inside its
// tick range, and these virtual tokens shorten its real share accordingly
__device__ __forceinline__ int64_t piece_tok(int64_t tau, int64_t V, double rcpV, int64_t n, int64_t X,
                                             int64_t Xs = 0) {
  if (tau >= V) return n;
  int64_t t = div_fix(tau * (n + X + Xs), V, rcpV) - Xs;
  t = t < 0 ? 0 : (t & ~int64_t(15));
  return t < n ? t : n;
}

__device__ __forceinline__ void compute_seg(const AttnArgs& a, int vc, int u, SegSh& o) {
  const int64_t U = a.U, V = a.V;
  const int b = div_small(u, a.Hkv), h = u - b * a.Hkv;
  const int64_t uV = static_cast<int64_t>(u) * V;
  const int64_t c1 = div_fix(uV, U, a.rcpU), c2 = div_fix(uV + V - 1, U, a.rcpU);
  const int64_t x0 = static_cast<int64_t>(vc) * U, x1 = x0 + U;
  const int64_t tau0 = (x0 > uV ? x0 : uV) - uV;
  const int64_t tau1 = (x1 < uV + V ? x1 : uV + V) - uV;
  int64_t len = a.seq_lens[b];
  if (len > a.n_cap) len = a.n_cap;
  if (len < 0) len = 0;
  const int64_t e = a.tok_end < 0 ? len : (a.tok_end < len ? a.tok_end : len);
  int64_t beg = a.tok_begin < e ? a.tok_begin : e;
  if (beg < 0) beg = 0;
  const int P = static_cast<int>(c2 - c1 + 1);
  const int64_t X = (a.append && P > 1) ? kAppendTokenCost : 0;
  const int64_t Xs = P > 1 ? a.seg_cost : 0;
  o.t0 = beg + piece_tok(tau0, V, a.rcpV, e - beg, X, Xs);
  o.t1 = beg + piece_tok(tau1, V, a.rcpV, e - beg, X, Xs);
  o.u = u; o.b = b; o.h = h;
  const HeadMap hm = head_map(a, h);
  o.hc = hm.hc; o.hq0 = hm.hq0; o.gp = hm.gp;
  o.cu = b * a.Hc + hm.hc;
  o.k = static_cast<int>(vc - c1);
  o.P = P;
  o.owner = 0; o.patch = 0; o.p_row = -1;
  if (a.append) {
    const int64_t p = a.write_pos[b];
    const bool in = p >= beg && p < e;
    o.p_row = p;
    o.owner = in ? (p >= o.t0 && p < o.t1) : (o.k == 0);
    o.patch = o.owner && in;
  }
  int rl = 0;
  if (a.res) {
    const int64_t x = a.res_lens[b];
    rl = static_cast<int>(x < 0 ? 0 : (x > a.r_cap ? a.r_cap : x));
  }
  o.rlen = rl;
  o.res_off = a.res ? b * a.res_sb + hm.hc * a.res_sh : 0;
}



// warp state -> shared memory: m, l per head (lanes r = 0) and acc as rows [4 heads][kWRow];
// thread (r, j) owns head j, dims 16r..16r+15 (float4 k = dims 16r+4k..16r+4k+3; the MMA slots
// [t][0] + [t][1] hold dim 16r+2t, [t][2] + [t][3] dim 16r+2t+1).  Row stride 132 spreads the
// 16-byte stores of the 32 lanes over all banks (4 wavefronts per store).
template <int DH>
__device__ __forceinline__ void store_state(float* dacc, float* dm, float* dl, int r, int j, float m, float l,
                                            const float (&acc)[DH / 16][4]) {
  if (r == 0) { dm[j] = m; dl[j] = l; }
  float* d = dacc + j * kWRow + (DH / 8) * r;
#pragma unroll
  for (int k = 0; k < DH / 32; ++k)
    *reinterpret_cast<float4*>(d + 4 * k) =
        make_float4(acc[2 * k][0] + acc[2 * k][1], acc[2 * k][2] + acc[2 * k][3],
                    acc[2 * k + 1][0] + acc[2 * k + 1][1], acc[2 * k + 1][2] + acc[2 * k + 1][3]);
}

// Last-arriver merge (persistent grids): the P published pieces (slots slot0 .. slot0+P-1) of output
// element (b, h, g, dim), combined in slot order by log-sum-exp (Alg. 1 l.729-730) and consumed
// (zeroed) for the next launch.  Chunks of 8 loads in flight.
__device__ __noinline__ void merge_consume(const AttnArgs& a, unsigned long long* part, int b, int hq0, int g, int dim,
                                           int64_t slot0, int P, int dh) {
  unsigned long long* pp = part + (slot0 * 4 + g) * 128 + dim;
  float m = -INFINITY, wsum = 0.f, osum = 0.f;
  for (int s0 = 0; s0 < P; s0 += 8) {
    float lv[8], xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      unsigned long long w = 0ull;
      if (s0 + k < P) {
        w = ~ld_relaxed_gpu_u64(pp + static_cast<int64_t>(s0 + k) * 512);
        st_relaxed_gpu_u64(pp + static_cast<int64_t>(s0 + k) * 512, 0ull);
      }
      lv[k] = s0 + k < P ? __uint_as_float(static_cast<uint32_t>(w >> 32)) : -INFINITY;
      xv[k] = __uint_as_float(static_cast<uint32_t>(w));
    }
    float mc = -INFINITY;
#pragma unroll
    for (int k = 0; k < 8; ++k) mc = fmaxf(mc, lv[k]);
    const float mn = fmaxf(m, mc);
    if (mn == -INFINITY) continue;
    const float sc = m == -INFINITY ? 0.f : ex2_approx(m - mn);
    osum *= sc;
    wsum *= sc;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float f = lv[k] == -INFINITY ? 0.f : ex2_approx(lv[k] - mn);
      wsum += f;
      osum += f * xv[k];
    }
    m = mn;
  }
  const bool empty = !(wsum > 0.f);
  const float ov = empty ? 0.f : osum / wsum;
  const int64_t oi = (static_cast<int64_t>(b) * a.Hq + hq0 + g) * dh + dim;
  if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
  else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
  if (dim == 0 && a.lse) a.lse[static_cast<int64_t>(b) * a.Hq + hq0 + g] = empty ? -INFINITY : (m + __log2f(wsum)) * kLn2;
}

// PG: paged code caches (a separate instantiation: the translation must not cost the contiguous path).
// DH: head dim 128, or 64 (NEXT-4; contiguous, no residual window, no fused append: the host routes
// those to the split kernel).  Published partials keep 128-float rows per head either way.
template <int KB, int VB, bool PG, int DH>
__global__ void __launch_bounds__(kThreads, 1) attn_stream_kernel(const __grid_constant__ AttnArgs a) {
  static_assert(DH == 128 || (DH == 64 && !PG), "D = 64: contiguous caches");
  using FK = FmtD<KB, DH>;
  using FV = FmtD<VB, DH>;
  constexpr int KR = FK::kRow, VR = FV::kRow;
  constexpr int KS = DH / 16, VS = DH / 32, NL = DH / 4, NO = 4 * DH;   // k-steps, V m-tile pairs, q lanes, outputs
  constexpr bool kCanAppend = KB <= 8 && VB <= 8 && DH == 128;
  constexpr bool kTable = Fmt<KB>::kSmem || Fmt<VB>::kSmem;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, j = lane & 3;

  // shared layout: misc at the bottom, the two codebook tables at the next 64 KiB boundary (the
  // host checks that the misc region fits below it)
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t tab_off = kTable ? ((raw_s + 65535u) & ~65535u) - raw_s : static_cast<uint32_t>(kMiscBytes);
  unsigned char* tab = smem_raw + tab_off;
  const uint32_t tab_s = raw_s + tab_off;
  float* sq = reinterpret_cast<float*>(smem_raw + kMiscQ);
  unsigned char* newcodes = smem_raw + kMiscNew;
  float* wm = reinterpret_cast<float*>(smem_raw + kMiscWM);
  float* wl = reinterpret_cast<float*>(smem_raw + kMiscWL);
  float* wacc = reinterpret_cast<float*>(smem_raw + kMiscW);
  SegSh* segs = reinterpret_cast<SegSh*>(smem_raw + kMiscSeg);
  volatile RoundSh* rsh = reinterpret_cast<volatile RoundSh*>(smem_raw + kMiscSeg + 2 * sizeof(SegSh));
  // merge bookkeeping: [0..1] last-arriver flag per segment; [2] number of deferred merge records;
  // [4 + 4i ..] record i = {u, k, P}
  int* sflag = reinterpret_cast<int*>(smem_raw + kMiscFlag);
  unsigned long long* part = a.part_elem;
  if (tid == 0) sflag[2] = 0;

  bool first = true;
  for (int vc = blockIdx.x; vc < a.V; vc += gridDim.x) {
    const int64_t x0 = static_cast<int64_t>(vc) * a.U;
    const int u_first = static_cast<int>(div_fix(x0, a.V, a.rcpV));
    const int u_last = static_cast<int>(div_fix(x0 + a.U - 1, a.V, a.rcpV));
    phase_mark(a.phase, vc, 0);
    for (int ua = u_first; ua <= u_last; ua += 2) {
      const int nseg = ua + 1 <= u_last ? 2 : 1;
      if (!first) __syncthreads();   // the previous round is done with the tables and misc

      // ---- static inputs (codebooks, lambda) first: with programmatic dependent launch this
      // overlaps the tail of the previous kernel; everything dynamic is read after the wait
      const int bA = div_small(ua, a.Hkv), hA = ua - bA * a.Hkv;   // virtual heads of the round's units
      const int hB = hA + 1 == a.Hkv ? 0 : hA + 1;
      const HeadMap hmA = head_map(a, hA), hmB = head_map(a, hB);
      const uint16_t* cbkA = a.ck + hmA.hc * a.ck_hs;
      const uint16_t* cbvA = a.cv + hmA.hc * a.cv_hs;
      const uint16_t* cbkB = a.ck + hmB.hc * a.ck_hs;
      const uint16_t* cbvB = a.cv + hmB.hc * a.cv_hs;
      const bool sameB = nseg == 1 || (cbkB == cbkA && cbvB == cbvA);   // B reuses table A
      // warp 0 skips the fill: it goes straight to the (dynamic) segment computation below
      if constexpr (kTable) {
        if (warp > 0) {
          for (int t = tid - 32; t < 512; t += kThreads - 32) {
            fill_tables<KB, VB>(tab, cbkA, cbvA, t);
            if (!sameB) fill_tables<KB, VB>(tab + kTab, cbkB, cbvB, t);
          }
        }
      }
      const int qseg = (warp - 8) >> 2, qg = warp & 3;   // warps 8..11: heads of segment A, 12..15: of B
      const bool qwarp = warp >= 8 && warp < 8 + 4 * nseg;
      float4 lam4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (qwarp) lam4 = *reinterpret_cast<const float4*>(a.lambda + (qseg ? hmB.hc : hmA.hc) * DH + 4 * (lane & (NL - 1)));
      const int q_gp = qseg ? hmB.gp : hmA.gp;
      // VECINFER_ATTN_FLAG_EARLY_CACHE (no residual window): the segments (seq_lens, write_pos) and
      // the first tiles' code loads go out before the grid-dependency wait; q after it
      const bool wait_late = first && a.early && !a.res;
      if (first && !wait_late) griddep_wait();
      first = false;

      // ---- dynamic inputs
      uint2 qw = make_uint2(0u, 0u);
      auto load_q = [&]() {
        if (qwarp && qg < q_gp) {
          const int bq = qseg && hB == 0 ? bA + 1 : bA, hq0 = qseg ? hmB.hq0 : hmA.hq0;
          qw = *reinterpret_cast<const uint2*>(a.q + bq * a.q_sb + (hq0 + qg) * a.q_sh + 4 * (lane & (NL - 1)));
        }
      };
      if (!wait_late) load_q();
      // ---- segments and warp assignment: the round's 16-token sub-tiles (A's, then B's) go to
      // the warps in contiguous balanced ranges [w*ns/16, (w+1)*ns/16); segment A = warps
      // [0, nwA), segment B = warps [b0, 16) (at most one warp in both: it straddles).  Warp 0
      // (15) nominally belongs to an empty A (B).
      if (warp == 0) {
        if (lane < nseg) compute_seg(a, vc, ua + lane, segs[lane]);
        __syncwarp();
        const int nsA = static_cast<int>((segs[0].t1 - segs[0].t0 + 15) >> 4);
        const int nsB = nseg > 1 ? static_cast<int>((segs[1].t1 - segs[1].t0 + 15) >> 4) : 0;
        const int ns = nsA + nsB;
        const unsigned ba = __ballot_sync(0xffffffffu, lane < kNW && (lane == 0 || ((static_cast<int64_t>(lane) * ns) >> 4) < nsA));
        const unsigned bb = __ballot_sync(0xffffffffu, lane < kNW && nseg > 1 &&
                                                           (lane == kNW - 1 || ((static_cast<int64_t>(lane + 1) * ns) >> 4) > nsA));
        if (lane == 0) {
          const int nwA = __popc(ba), b0 = bb ? __ffs(bb) - 1 : kNW - 1;
          rsh->nsA = nsA; rsh->ns = ns; rsh->nwA = nwA; rsh->b0 = b0;
          rsh->strad = (nseg > 1 && nwA - 1 >= b0) ? nwA - 1 : -1;
          rsh->sameB = sameB;
          if (a.merge == kMergeSpin) {   // deferred merges: the split units this CTA has a piece of
            for (int sgi = 0; sgi < nseg; ++sgi) {
              if (segs[sgi].P == 1) continue;
              int* rec = sflag + 4 + 4 * sflag[2];
              rec[0] = segs[sgi].u; rec[1] = segs[sgi].k; rec[2] = segs[sgi].P;
              sflag[2] += 1;
            }
          }
        }
      }
      __syncthreads();
      if (ua == u_first) phase_mark(a.phase, vc, 6);
      const bool inA = warp < rsh->nwA;
      const bool inB = nseg > 1 && warp >= rsh->b0;
      const int np = static_cast<int>(inA) + static_cast<int>(inB);

      // per-piece state (piece 0 set up here so its first loads overlap the prologue)
      int seg = inA ? 0 : 1;
      int64_t tok0 = 0;
      int ntok = 0, ntile = 0, patch_tile = -1, patch_row = 0;
      int t_res = 0, t_step = 1, rlen = 0;
      int64_t res_off = 0;
      const uint8_t* kp = nullptr;
      const uint8_t* vp = nullptr;
      TileCodes<KB, VB> nxt;
      // paged code caches (NEXT-4): pieces start at 16-token multiples (tok_begin % 32 == 0) and
      // pages hold >= 32 tokens, so every 16-token sub-tile lies in one page; each sub-tile is
      // translated through the block table, whose entries are read one tile ahead
      constexpr bool paged = PG;
      int pgn0 = 0, pgn1 = 0;   // pages of the two sub-tiles of the next tile to load
      auto page_of = [&](int bb, int64_t tok) -> int { return a.bt[bb * a.bt_stride + (tok >> a.page_shift)]; };
      // this lane's K / V bytes of row 0 of page 0 of the piece's KV head (set by setup_piece):
      // row (pg, t) of the head = pkb + pg * (Hc * page_size * KR) + (t % page_size) * KR
      const uint8_t* pkb = nullptr;
      const uint8_t* pvb = nullptr;
      // both sub-tiles translated unconditionally (sub-tile 1 of a tile inside one page has p1 = p0):
      // per sub-tile one 32 x 32 -> 64-bit multiply-add for the page plus the in-page row, no branch
      // (tokens, page ids and the bytes between pages of one head fit 32 bits)
      auto load_paged = [&](int tstart, int p0, int p1, int rem) {
        const uint32_t pmask = (1u << a.page_shift) - 1u;
        const uint32_t rows_pg = static_cast<uint32_t>(a.Hc) << a.page_shift;   // rows between page indices
        const uint32_t i0 = static_cast<uint32_t>(tstart) & pmask, i1 = static_cast<uint32_t>(tstart + 16) & pmask;
        const uint8_t* k0 = pkb + static_cast<uint64_t>(static_cast<uint32_t>(p0)) * (rows_pg * KR) + i0 * KR;
        const uint8_t* v0 = pvb + static_cast<uint64_t>(static_cast<uint32_t>(p0)) * (rows_pg * VR) + i0 * VR;
        const uint8_t* k1 = pkb + static_cast<uint64_t>(static_cast<uint32_t>(p1)) * (rows_pg * KR) + i1 * KR;
        const uint8_t* v1 = pvb + static_cast<uint64_t>(static_cast<uint32_t>(p1)) * (rows_pg * VR) + i1 * VR;
        if (rem >= 32) {   // one (warp-uniform) branch per tile: full tiles load unpredicated
          load_subtile<KB, VB, 0>(nxt, k0, v0, 16, r, j);
          load_subtile<KB, VB, 1>(nxt, k1, v1, 16, r, j);
        } else {
          load_subtile<KB, VB, 0>(nxt, k0, v0, rem, r, j);
          load_subtile<KB, VB, 1>(nxt, k1, v1, rem - 16, r, j);
        }
      };
      // block-table entries of a tile starting at token t (rem = tokens from t): the pages of its two
      // sub-tiles, both read (predicated, no branch).  (Reusing the previous tile's entries and reading
      // the table only at page starts was measured slower: the reads become conditional and chained.)
      const int32_t* btp = nullptr;   // block-table row of the piece's sequence (setup_piece)
      auto tile_pages = [&](int t, int rem, int& p0, int& p1) {
        p0 = rem > 0 ? __ldg(btp + (t >> a.page_shift)) : 0;
        p1 = rem > 16 ? __ldg(btp + ((t + 16) >> a.page_shift)) : p0;
      };
      // sets up piece `seg` of this warp and issues its first tile loads
      auto setup_piece = [&]() {
        const SegSh& sg = segs[seg];
        const int nsA = rsh->nsA, ns = rsh->ns;
        const int lo = static_cast<int>((static_cast<int64_t>(warp) * ns) >> 4);
        const int hi = static_cast<int>((static_cast<int64_t>(warp + 1) * ns) >> 4);
        const int s0 = seg == 0 ? min(lo, nsA) : max(lo, nsA) - nsA;
        const int s1 = seg == 0 ? min(hi, nsA) : max(hi, nsA) - nsA;
        tok0 = sg.t0 + 16 * static_cast<int64_t>(s0);
        const int64_t tend = sg.t0 + 16 * static_cast<int64_t>(s1);
        ntok = static_cast<int>(max(int64_t(0), min(tend, static_cast<int64_t>(sg.t1)) - tok0));
        ntile = (ntok + 31) >> 5;
        const int64_t unit = sg.cu;   // cache unit of the codes
        kp = a.kcodes + (unit * a.n_cap + tok0 + r) * KR + FK::kOffK * j;
        vp = a.vcodes + (unit * a.n_cap + tok0 + 2 * j) * VR + FV::kOffV * r;
        patch_tile = -1;
        if (kCanAppend && sg.patch) {
          const int64_t rel = sg.p_row - tok0;
          if (rel >= 0 && rel < ntok) {
            patch_tile = static_cast<int>(rel >> 5);
            patch_row = static_cast<int>(rel & 31);
          }
        }
        if constexpr (paged) {
          pkb = a.kcodes + ((static_cast<int64_t>(sg.hc) << a.page_shift) + r) * KR + Fmt<KB>::kOffK * j;
          pvb = a.vcodes + ((static_cast<int64_t>(sg.hc) << a.page_shift) + 2 * j) * VR + Fmt<VB>::kOffV * r;
          btp = a.bt + sg.b * a.bt_stride;
          const int t0 = static_cast<int>(tok0);
          int p0, p1;
          tile_pages(t0, ntok, p0, p1);
          if (ntile > 0) load_paged(t0, p0, p1, ntok);
          tile_pages(t0 + 32, ntok - 32, pgn0, pgn1);
        } else if (ntile > 0) {
          load_tile_tail<KB, VB, DH>(nxt, kp, vp, ntok, r, j);   // (predicated: one code path)
        }
        // residual rows of the unit: row t belongs to piece t % P, and within the piece's warps
        // (rank rho of nw) to rows t = k + P * (rho + nw * i)
        rlen = sg.rlen;
        res_off = sg.res_off;
        const int rho = seg == 0 ? warp : warp - rsh->b0;
        const int nw = seg == 0 ? rsh->nwA : kNW - rsh->b0;
        t_res = sg.k + sg.P * rho;
        t_step = sg.P * nw;
      };
      if (np > 0) setup_piece();
      if (wait_late) {
        griddep_wait();
        load_q();
      }
      if (ua == u_first) phase_mark(a.phase, vc, 12);

      // ---- query transform (Eq. 7): sq[seg][g] = ((q_g * lambda) H) * qscale
      if (qwarp) {
        float* dq = sq + kQSeg * qseg + kQRow * qg + qoff(lane);
        if (qg < q_gp) qtransform_lane(qw, lam4, a.qscale, lane, dq, NL);
        else if (lane < NL) *reinterpret_cast<float4*>(dq) = make_float4(0.f, 0.f, 0.f, 0.f);
      }

      if (ua == u_first) phase_mark(a.phase, vc, 11);
      // ---- fused decode append: the owner piece of a unit encodes its new token (Eq. 9: S then H
      // on the key, VQ on both; bf16 codebook -> fp32, pinned distance, lowest index on ties).  The
      // round's owner segments (G = 1 or 2) are encoded in ONE phase: the 16 warps form 2G groups
      // (segment, K or V) of 8 / G warps, each warp scanning n_ent * G / 8 centroids in batches of 32
      // staged by itself, then one barrier and a per-group reduction in warp order.
      if constexpr (kCanAppend) {
        if (a.append) {
          int own0 = -1, own1 = -1;
          for (int sgi = 0; sgi < nseg; ++sgi)
            if (segs[sgi].owner) { if (own0 < 0) own0 = sgi; else own1 = sgi; }
          const int G = own0 < 0 ? 0 : (own1 < 0 ? 1 : 2);
          if (G > 0) {
            const int wps = 8 / G;                      // warps per (segment, stream)
            const int grp = warp / wps, wi = warp - grp * wps;
            const int sgi = (grp >> 1) ? own1 : own0;
            const bool isv = grp & 1;
            const SegSh& sg = segs[sgi];
            const int bb = sg.b, hh = sg.hc;
            const int n_ent = isv ? (1 << VB) : (1 << KB);
            const int P = n_ent / wps;                  // centroids of this warp
            float4* stage = reinterpret_cast<float4*>(smem_raw + kMiscStage);
            float* sbest = reinterpret_cast<float*>(smem_raw + kMiscBest);
            uint32_t* sidx = reinterpret_cast<uint32_t*>(smem_raw + kMiscIdx);
            const uint16_t* cb = isv ? (sgi ? cbvB : cbvA) : (sgi ? cbkB : cbkA);
            // the first batch's centroids go out before the key transform (its loads + shuffles hide
            // the L2 round trip).  Batches of 32 centroids are staged as 16 pairs in the
            // pinned_dist4_x2 layout (two centroids per paired FADD2 / FMUL2, per-element RN)
            // (P <= 64: at most two batches, both loaded here)
            uint2 cwa[2], cwb[2];
#pragma unroll
            for (int bt = 0; bt < 2; ++bt) {
              const int nbb = P - 32 * bt < 32 ? P - 32 * bt : 32;
              cwa[bt] = cwb[bt] = make_uint2(0u, 0u);
              if (lane < nbb / 2) {
                cwa[bt] = *reinterpret_cast<const uint2*>(cb + 4 * (P * wi + 32 * bt + 2 * lane));
                cwb[bt] = *reinterpret_cast<const uint2*>(cb + 4 * (P * wi + 32 * bt + 2 * lane + 1));
              }
            }
            float x[4];
            if (!isv) {
              const bool bad = key_transform_lane(a.knew + bb * a.kn_sb + hh * a.kn_sh + 4 * lane,
                                                  a.inv_lambda + hh * 128 + 4 * lane, a.inv_sqrt_d, lane, x);
              if (bad && wi == 0 && lane == 0 && a.err) atomicOr(a.err, VECINFER_FLAG_RANGE);
            } else {
              const float4 v = bf16x4_to_float4(*reinterpret_cast<const uint2*>(a.vnew + bb * a.vn_sb + hh * a.vn_sh + 4 * lane));
              x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
            }
            if (ua == u_first) phase_mark(a.phase, vc, 13);   // (thread 0: its K transform done)
            float best = __int_as_float(0x7f800000);
            uint32_t bi = 0;
            uint4* sp = reinterpret_cast<uint4*>(stage) + warp * 32;   // 16 pairs x 32 B
#pragma unroll
            for (int bt = 0; bt < 2; ++bt) {             // batches of 32 centroids staged by this warp
              const int c0 = 32 * bt;
              if (c0 >= P) break;
              const int nb = P - c0 < 32 ? P - c0 : 32;  // (even: books of 16 / 256 entries)
              const int j0 = P * wi + c0;
              if (lane < nb / 2) {   // the pair layout of stage_centroid_pair
                const uint2 ca = cwa[bt], cbb = cwb[bt];
                sp[2 * lane] = make_uint4(ca.x << 16, cbb.x << 16, ca.x & 0xFFFF0000u, cbb.x & 0xFFFF0000u);
                sp[2 * lane + 1] = make_uint4(ca.y << 16, cbb.y << 16, ca.y & 0xFFFF0000u, cbb.y & 0xFFFF0000u);
              }
              __syncwarp();
#pragma unroll 4
              for (int pi = 0; pi < nb / 2; ++pi) {
                const float2 d = pinned_dist4_x2(x[0], x[1], x[2], x[3], sp[2 * pi], sp[2 * pi + 1]);
                if (d.x < best) { best = d.x; bi = j0 + 2 * pi; }       // lower index first: ties keep it
                if (d.y < best) { best = d.y; bi = j0 + 2 * pi + 1; }
              }
              __syncwarp();   // the batch is read before the next one overwrites it
            }
            sbest[warp * 32 + lane] = best;
            sidx[warp * 32 + lane] = bi;
            if (ua == u_first) phase_mark(a.phase, vc, 14);   // (thread 0: its scan done)
            __syncthreads();
            if (ua == u_first) phase_mark(a.phase, vc, 10);   // (every warp's scan done)
            if (wi == 0) {   // reduce the group's warps in warp (= centroid index) order
              float bbst = sbest[warp * 32 + lane];
              uint32_t ii = sidx[warp * 32 + lane];
              for (int w = 1; w < wps; ++w) {
                const float c = sbest[(warp + w) * 32 + lane];
                if (c < bbst) { bbst = c; ii = sidx[(warp + w) * 32 + lane]; }
              }
              unsigned char* nc = newcodes + 128 * sgi;
              if (!isv) put_code<KB>(nc, lane, ii);
              else put_code<VB>(nc + 64, lane, ii);
              const int64_t p = sg.p_row;
              int pgw = 0;
              if (p >= 0 && p < a.n_cap && (!paged || ((pgw = page_of(sg.b, p)) >= 0 && pgw < a.n_pages))) {
                const int64_t row = paged ? ((static_cast<int64_t>(pgw) * a.Hc + sg.hc) << a.page_shift) +
                                                (p & ((int64_t(1) << a.page_shift) - 1))
                                          : static_cast<int64_t>(sg.cu) * a.n_cap + p;
                if (!isv) put_code<KB>(a.kcodes_w + row * KR, lane, ii);
                else put_code<VB>(a.vcodes_w + row * VR, lane, ii);
              } else if (lane == 0 && a.err) {
                atomicOr(a.err, VECINFER_FLAG_WRITE_POS);
              }
            }
          }
        }
      }
      __syncthreads();
      if (ua == u_first) phase_mark(a.phase, vc, 1);

      // ---- main loop over this warp's pieces (<= 2)
      float acc[2 * VS][4];
      float m_run = -INFINITY, l_run = 0.f;
#pragma unroll 1
      for (int wp = 0; wp < np; ++wp) {
        if (wp > 0) {   // the straddling warp: flush piece A's state, start piece B
          l_run += __shfl_xor_sync(0xffffffffu, l_run, 4);
          l_run += __shfl_xor_sync(0xffffffffu, l_run, 8);
          l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
          store_state<DH>(wacc + (kSlots - 1) * 4 * kWRow, wm + (kSlots - 1) * 4, wl + (kSlots - 1) * 4, r, j, m_run, l_run, acc);
          seg = 1;
          setup_piece();
        }
        m_run = -INFINITY;
        l_run = 0.f;
#pragma unroll
        for (int t = 0; t < 2 * VS; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
        const uint16_t* cbk = seg ? cbkB : cbkA;
        const uint16_t* cbv = seg ? cbvB : cbvA;
        const uint32_t kbase = tab_s + ((seg && !rsh->sameB) ? kTab : 0) + (lane & 15) * 8;
        const uint32_t vbase = kbase + 128;

        // B fragments of the score MMA: column n = lane/4 <-> (head n/2, part n%2); rows k
        // <-> sub-vector 8j+t, components {0,1} (b0) and {2,3} (b1)
        uint32_t bq0[KS], bq1[KS];
        {
          const int gq = r >> 1, part = r & 1;
          const float* sqs = sq + kQSeg * seg + kQRow * gq;
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const float4 v = *reinterpret_cast<const float4*>(sqs + qoff(KS * j + t));
            const float in[4] = {v.x, v.y, v.z, v.w};
            float o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const __half hh = __float2half_rn(in[i]);
              o[i] = part == 0 ? __half2float(hh) : (in[i] - __half2float(hh));
            }
            bq0[t] = pack_half2(o[0], o[1]);
            bq1[t] = pack_half2(o[2], o[3]);
          }
        }

        // ---- residual window (NEXT-1): raw bf16 rows scored with the raw q (q k^T = q~ k~^T,
        // Eq. 7), folded into this warp's online-softmax state before the code tiles; the P.V
        // goes into the hi slots of the MMA accumulator layout (thread (r, j) owns head j, dims
        // 16r + 2t + {0, 1})
        if constexpr (DH == 128) if (t_res < rlen) {
          const SegSh& sgr = segs[seg];
          const int bb = sgr.b, hh = sgr.hc;
          float qr[4][4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 v = g < sgr.gp ? bf16x4_to_float4(*reinterpret_cast<const uint2*>(
                                              a.q + bb * a.q_sb + (sgr.hq0 + g) * a.q_sh + 4 * lane))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            qr[g][0] = v.x * a.qscale_raw; qr[g][1] = v.y * a.qscale_raw;
            qr[g][2] = v.z * a.qscale_raw; qr[g][3] = v.w * a.qscale_raw;
          }
          for (int t = t_res; t < rlen; t += t_step) {
            // the appended row (decode step into the window) comes from k_new / v_new; this warp
            // is its only reader and also writes it into the window
            const bool is_new = a.res_append && t == rlen - 1;
            const uint16_t* krow = is_new ? a.knew + bb * a.kn_sb + hh * a.kn_sh : a.kres + res_off + t * 128;
            const uint16_t* vsrc = is_new ? a.vnew + bb * a.vn_sb + hh * a.vn_sh : a.vres + res_off + t * 128;
            const uint2 rk = *reinterpret_cast<const uint2*>(krow + 4 * lane);
            const uint4 rv0 = *reinterpret_cast<const uint4*>(vsrc + 16 * r);
            const uint4 rv1 = *reinterpret_cast<const uint4*>(vsrc + 16 * r + 8);
            if (is_new) {
              reinterpret_cast<uint2*>(const_cast<uint16_t*>(a.kres) + res_off + t * 128)[lane] = rk;
              reinterpret_cast<uint2*>(const_cast<uint16_t*>(a.vres) + res_off + t * 128)[lane] =
                  *reinterpret_cast<const uint2*>(vsrc + 4 * lane);
            }
            const float4 kv = bf16x4_to_float4(rk);
            float sgv[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float v = qr[g][0] * kv.x + qr[g][1] * kv.y + qr[g][2] * kv.z + qr[g][3] * kv.w;
#pragma unroll
              for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
              sgv[g] = v;
            }
            const float sj = j == 0 ? sgv[0] : j == 1 ? sgv[1] : j == 2 ? sgv[2] : sgv[3];
            if (sj > m_run + kTau) {   // per-lane: all 8 lanes of head j agree
              const float alpha = ex2_approx(m_run - sj);
#pragma unroll
              for (int tt = 0; tt < 8; ++tt) {
                acc[tt][0] *= alpha; acc[tt][1] *= alpha; acc[tt][2] *= alpha; acc[tt][3] *= alpha;
              }
              l_run *= alpha;
              m_run = sj;
            }
            const float p = ex2_approx(sj - m_run);
            if (r == 0) l_run += p;                         // once per head (lanes r = 0 of each j)
            const uint32_t vw[8] = {rv0.x, rv0.y, rv0.z, rv0.w, rv1.x, rv1.y, rv1.z, rv1.w};
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
              acc[tt][0] += p * __uint_as_float(vw[tt] << 16);             // dim 16r + 2tt
              acc[tt][2] += p * __uint_as_float(vw[tt] & 0xFFFF0000u);     // dim 16r + 2tt + 1
            }
          }
        }

        for (int it = 0; it < ntile; ++it) {
          TileCodes<KB, VB> cur = nxt;
#ifndef EXP_NOPATCH
          if constexpr (kCanAppend) {
#else
          if constexpr (false) {
#endif
            if (it == patch_tile) {   // the appended row: codes just encoded, not the stale load
              const unsigned char* nc = newcodes + 128 * seg;
              KCode<KB> nk;
              VCode<VB> nv;
              if constexpr (KB == 8) nk = *reinterpret_cast<const uint2*>(nc + 8 * j);
              else nk = *reinterpret_cast<const uint32_t*>(nc + Fmt<KB>::kOffK * j);
              if constexpr (VB == 8) nv = *reinterpret_cast<const uint32_t*>(nc + 64 + 4 * r);
              else nv = *reinterpret_cast<const uint16_t*>(nc + 64 + Fmt<VB>::kOffV * r);
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
          if (it + 1 < ntile) {
            const int rem = rem_cur - 32;
            if constexpr (paged) {
              const int tn = static_cast<int>(tok0) + 32 * (it + 1);
              load_paged(tn, pgn0, pgn1, rem);
              tile_pages(tn + 32, rem - 32, pgn0, pgn1);
            } else {
              kp += 32 * KR;
              vp += 32 * VR;
              if (rem >= 32) load_tile_full<KB, VB, DH>(nxt, kp, vp);
              else load_tile_tail<KB, VB, DH>(nxt, kp, vp, rem, r, j);
            }
          }
          };
          // 65 536-entry books: the next tile's codes are loaded after this tile (as in the split
          // kernel: tiles are long, the HBM latency hides behind the other warps' gathers, and the
          // two tiles' codes are never live together)
          constexpr bool kLateNext = (KB == 16 || VB == 16) && DH == 128;
          if constexpr (!kLateNext) issue_next();
          // tile body, specialised on whether sub-tile 1 holds tokens (a trailing half tile skips it);
          // the common full-tile instance is straight-line code the scheduler can interleave
          auto tile_body = [&](auto TWO) {
            constexpr bool kTwo = decltype(TWO)::value;
            // ---- scores (log2 units) for tile tokens 16q + {r, r+8}, head j; two independent MMA
            // accumulator chains per sub-tile (k-steps 0-3 and 4-7) halve the dependent HMMA latency
            float sc[2][2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              if constexpr (!kTwo) {
                if (q == 1) {
                  sc[1][0] = sc[1][1] = -INFINITY;
                  break;
                }
              }
              float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
              static_for<0, KS>([&](auto T) {
                constexpr int t = decltype(T)::value;
                const uint2 ea = gather_k<KB, t>(cur.k[q][0], kbase, cbk);
                const uint2 eb = gather_k<KB, t>(cur.k[q][1], kbase, cbk);
                if (t < KS / 2) mma_16816(d0, ea.x, eb.x, ea.y, eb.y, bq0[t], bq1[t]);
                else mma_16816(d1, ea.x, eb.x, ea.y, eb.y, bq0[t], bq1[t]);
              });
              sc[q][0] = (d0[0] + d1[0]) + (d0[1] + d1[1]);
              sc[q][1] = (d0[2] + d1[2]) + (d0[3] + d1[3]);
            }
            if (rem_cur < 32) {
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                if (16 * q + r >= rem_cur) sc[q][0] = -INFINITY;
                if (16 * q + r + 8 >= rem_cur) sc[q][1] = -INFINITY;
              }
            }

            // ---- online softmax (Alg. 1 l.12-13, 18), lazy rescale.  Common path: every lane checks
            // its own 4 scores against m_run + tau (p <= 2^tau) -- no cross-lane traffic; only when
            // some lane exceeds it are the per-head tile maxima reduced and the accumulators rescaled.
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
              if constexpr (!kTwo) {
                if (q == 1) break;
              }
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

              // ---- P.V (Alg. 1 l.16): m-tile t <-> sub-vector 4r + t/2, components 2(t%2) + {0,1}
              static_for<0, VS>([&](auto Uc) {
                constexpr int u = decltype(Uc)::value;
                const uint2 g0 = gather_v<VB, u>(cur.v[q][0], vbase, cbv);
                const uint2 g1 = gather_v<VB, u>(cur.v[q][1], vbase, cbv);
                const uint2 g2 = gather_v<VB, u>(cur.v[q][2], vbase, cbv);
                const uint2 g3 = gather_v<VB, u>(cur.v[q][3], vbase, cbv);
                mma_16816(acc[2 * u], prmt(g0.x, g1.x, 0x5410), prmt(g0.x, g1.x, 0x7632), prmt(g2.x, g3.x, 0x5410),
                          prmt(g2.x, g3.x, 0x7632), bp0, bp1);
                mma_16816(acc[2 * u + 1], prmt(g0.y, g1.y, 0x5410), prmt(g0.y, g1.y, 0x7632), prmt(g2.y, g3.y, 0x5410),
                          prmt(g2.y, g3.y, 0x7632), bp0, bp1);
              });
            }
          };
#ifdef EXP_ONEBODY
          tile_body(std::true_type{});
#else
          if (rem_cur > 16) tile_body(std::true_type{});
          else tile_body(std::false_type{});
#endif
          if constexpr (kLateNext) issue_next();
        }
      }

      // ---- this warp's last piece -> its partial slot (misc region, no barrier needed)
      l_run += __shfl_xor_sync(0xffffffffu, l_run, 4);
      l_run += __shfl_xor_sync(0xffffffffu, l_run, 8);
      l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
      if (np > 0) store_state<DH>(wacc + warp * 4 * kWRow, wm + warp * 4, wl + warp * 4, r, j, m_run, l_run, acc);
      const bool last_round = ua + 2 > u_last && vc + static_cast<int>(gridDim.x) >= a.V;
      if (ua + 2 > u_last) phase_mark(a.phase, vc, 2);
      if (last_round) griddep_launch_dependents();   // the next kernel may start its static prologue
      __syncthreads();
      if (ua + 2 > u_last) phase_mark(a.phase, vc, 7);

      // ---- combine the warp pieces of each segment (thread = (segment, head, dim)): M = max_w m_w,
      // f_w = 2^(m_w - M), o = sum_w f_w acc_w / sum_w f_w l_w over the segment's warps (segment A =
      // warps [0, nwA) with the straddler's A piece in slot 16, segment B = warps [b0, 16)).  Whole
      // units write o and L; pieces of split units publish (o_s, L_s) per element as one 64-bit
      // relaxed store of ~(L_s << 32 | o_s) to slot c + u (zero = empty: see the merge).
      const int nwA = rsh->nwA, b0 = rsh->b0, strad = rsh->strad;
      // per (slot, head) weights f = 2^(m_slot - M_seg) and per (segment, head) maxima, computed once
      // by 76 threads into the (idle) staging region, so the per-output combine below is a plain
      // weighted sum: no exponentials, no max scans
      float* sfw = reinterpret_cast<float*>(smem_raw + kMiscStage);   // [kSlots][4]
      float* sMx = sfw + kSlots * 4;                                   // [2][4]
      if (tid < kSlots * 4 + 8) {
        const bool wslot = tid < kSlots * 4;
        const int sl = wslot ? tid >> 2 : -1, g = tid & 3;
        int sgi;
        if (!wslot) sgi = (tid - kSlots * 4) >> 2;
        else if (sl == kSlots - 1) sgi = strad >= 0 ? 0 : -1;
        else if (sl == strad) sgi = 1;
        else if (sl < nwA) sgi = 0;
        else sgi = (nseg > 1 && sl >= b0) ? 1 : -1;
        float M = -INFINITY, f = 0.f;
        if (sgi >= 0 && sgi < nseg) {
          const int w_lo = sgi == 0 ? 0 : b0, w_hi = sgi == 0 ? nwA : kNW;
          const int xs = sgi == 0 ? strad : -1;   // the straddler's A piece lives in slot 16
          for (int w = w_lo; w < w_hi; ++w) M = fmaxf(M, wm[(w == xs ? kSlots - 1 : w) * 4 + g]);
          if (wslot) {
            const float mv = wm[sl * 4 + g];
            f = (M == -INFINITY || mv == -INFINITY) ? 0.f : ex2_approx(mv - M);   // empty piece: 0
          }
        }
        if (wslot) sfw[tid] = f;
        else sMx[tid - kSlots * 4] = M;
      }
      __syncthreads();
#pragma unroll 1
      for (int idx = tid; idx < nseg * NO; idx += kThreads) {
        const int sgi = idx / NO, g = (idx / DH) & 3, dim = idx % DH;
        const int w_lo = sgi == 0 ? 0 : b0, w_hi = sgi == 0 ? nwA : kNW;
        const int xs = sgi == 0 ? strad : -1;   // the straddler's A piece lives in slot 16
        const float M = sMx[sgi * 4 + g];
        float ov = 0.f, lsum = 0.f;
        if (M != -INFINITY) {
#pragma unroll 4
          for (int w = w_lo; w < w_hi; ++w) {
            const int sl = w == xs ? kSlots - 1 : w;
            const float f = sfw[sl * 4 + g];
            lsum += f * wl[sl * 4 + g];
            ov += f * wacc[(sl * 4 + g) * kWRow + dim];
          }
        }
        const bool empty = !(lsum > 0.f);
        ov = empty ? 0.f : ov * __frcp_rn(lsum);
        const float L2 = empty ? -INFINITY : M + __log2f(lsum);
        const SegSh& sg = segs[sgi];
        if (sg.P == 1) {
          if (g < sg.gp) {
            const int64_t oi = (static_cast<int64_t>(sg.b) * a.Hq + sg.hq0 + g) * DH + dim;
            if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
            else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
            if (dim == 0 && a.lse) a.lse[static_cast<int64_t>(sg.b) * a.Hq + sg.hq0 + g] = L2 * kLn2;
          }
        } else if (g < sg.gp) {
          // only the real heads are published: the consumers poll (and zero) g < gp only, so a
          // padding slot written here would stay non-zero in the workspace for a later launch
          const int64_t pi = ((static_cast<int64_t>(vc) + sg.u) * 4 + g) * 128 + dim;
          st_relaxed_gpu_u64(part + pi, ~((static_cast<unsigned long long>(__float_as_uint(L2)) << 32) |
                                          __float_as_uint(ov)));
        }
      }
      if (ua + 2 > u_last) phase_mark(a.phase, vc, 9);

      // ---- persistent grid (V > #SMs): the last-arriving piece of a split unit merges it
      if (a.merge == kMergeLast) {
        __syncthreads();   // this CTA's partial stores happen-before thread 0's release below
        if (tid < nseg) {
          const SegSh& sg = segs[tid];
          int lastp = 0;
          if (sg.P > 1) {
            unsigned long long* bar = reinterpret_cast<unsigned long long*>(a.counter) + sg.u;
            const unsigned long long old = atom_add_acq_rel_gpu_u64(bar, 1ull);
            lastp = (old & 0xFFFFFFFFull) == static_cast<unsigned long long>(sg.P - 1);
            if (lastp) red_add_release_gpu_u64(bar, 0ull - static_cast<unsigned long long>(sg.P));   // back to zero
          }
          sflag[tid] = lastp;
        }
        __syncthreads();
#pragma unroll 1
        for (int sgi = 0; sgi < nseg; ++sgi) {
          if (!sflag[sgi]) continue;
          const SegSh& sg = segs[sgi];
          const int64_t c1 = div_fix(static_cast<int64_t>(sg.u) * a.V, a.U, a.rcpU);
          const int g = tid / DH, dim = tid % DH;
          if (tid < NO && g < sg.gp) merge_consume(a, part, sg.b, sg.hq0, g, dim, c1 + sg.u, sg.P, DH);
        }
      }
      if (ua + 2 > u_last) phase_mark(a.phase, vc, 3);
    }
  }

  // ---- deferred merges (all CTAs co-resident): piece k of a split unit with P pieces merges
  // outputs [k*per, (k+1)*per), per = ceil(512/P), of the unit.  One thread per (output, piece)
  // element polls it until published (non-zero), consumes it (stores zero back: every element is
  // read exactly once, so the workspace is clean for the next launch), and stages it in shared
  // memory; then one thread per output combines its P pieces in order (Alg. 1 l.729-730).
  if (a.merge == kMergeSpin) {
    __syncthreads();
    const int nrec = sflag[2];
    if (nrec > 0) {
      float2* stage = reinterpret_cast<float2*>(smem_raw + kMiscStage);
      int E[2] = {0, 0}, nout[2] = {0, 0}, per[2] = {0, 0};
      for (int i = 0; i < nrec; ++i) {
        const int* rec = sflag + 4 + 4 * i;
        per[i] = (NO + rec[2] - 1) / rec[2];
        nout[i] = max(0, min(NO, (rec[1] + 1) * per[i]) - rec[1] * per[i]);
        E[i] = nout[i] * rec[2];
      }
#pragma unroll 1
      for (int e = tid; e < E[0] + E[1]; e += kThreads) {
        const int i = e < E[0] ? 0 : 1, ee = e - (i ? E[0] : 0);
        const int* rec = sflag + 4 + 4 * i;
        const int u = rec[0], k = rec[1], P = rec[2];
        const int oo = ee / P, p = ee - oo * P;
        const int o = k * per[i] + oo;   // g * DH + dim
        float2 v = make_float2(0.f, -INFINITY);
        const int bu = div_small(u, a.Hkv);
        if (o / DH < head_map(a, u - bu * a.Hkv).gp) {
          const int64_t c1 = div_fix(static_cast<int64_t>(u) * a.V, a.U, a.rcpU);
          unsigned long long* pp = part + (c1 + u + p) * 512 + (o / DH) * 128 + o % DH;
          unsigned long long w;
          while ((w = ld_relaxed_gpu_u64(pp)) == 0ull) if (VECINFER_SPIN_NS > 0) __nanosleep(VECINFER_SPIN_NS);
          st_relaxed_gpu_u64(pp, 0ull);
          w = ~w;
          v = make_float2(__uint_as_float(static_cast<uint32_t>(w)), __uint_as_float(static_cast<uint32_t>(w >> 32)));
        }
        stage[e] = v;
      }
      __syncthreads();
      phase_mark(a.phase, blockIdx.x, 5);
#pragma unroll 1
      for (int t = tid; t < nout[0] + nout[1]; t += kThreads) {
        const int i = t < nout[0] ? 0 : 1, tt = t - (i ? nout[0] : 0);
        const int* rec = sflag + 4 + 4 * i;
        const int u = rec[0], k = rec[1], P = rec[2];
        const int o = k * per[i] + tt, g = o / DH, dim = o % DH;
        const int b = div_small(u, a.Hkv);
        const HeadMap hmu = head_map(a, u - b * a.Hkv);
        if (g >= hmu.gp) continue;
        const float2* sv = stage + (i ? E[0] : 0) + tt * P;
        float M = -INFINITY;
        for (int p = 0; p < P; ++p) M = fmaxf(M, sv[p].y);
        float wsum = 0.f, osum = 0.f;
        if (M != -INFINITY) {
          for (int p = 0; p < P; ++p) {
            const float f = sv[p].y == -INFINITY ? 0.f : ex2_approx(sv[p].y - M);
            wsum += f;
            osum += f * sv[p].x;
          }
        }
        const bool empty = !(wsum > 0.f);
        const int64_t oi = (static_cast<int64_t>(b) * a.Hq + hmu.hq0 + g) * DH + dim;
        const float ov = empty ? 0.f : osum * __frcp_rn(wsum);
        if (a.o_f32) static_cast<float*>(a.o)[oi] = ov;
        else static_cast<__nv_bfloat16*>(a.o)[oi] = __float2bfloat16_rn(ov);
        if (dim == 0 && a.lse) a.lse[static_cast<int64_t>(b) * a.Hq + hmu.hq0 + g] = empty ? -INFINITY : (M + __log2f(wsum)) * kLn2;
      }
    }
  }
  phase_mark(a.phase, blockIdx.x, 4);

}

}  // namespace

using AttnKernel = void (*)(const AttnArgs);

static int smem_for(int kb, int vb) { return (kb > 8 && vb > 8) ? kSmemBytesNoTab : kSmemBytes; }

static AttnKernel kernel_for(int kb, int vb, bool paged = false, int dh = 128) {
  const int ki = kb == 4 ? 0 : kb == 8 ? 1 : 2, vi = vb == 4 ? 0 : vb == 8 ? 1 : 2;
  static const AttnKernel table[3][3][3] = {
      {{attn_stream_kernel<4, 4, false, 128>, attn_stream_kernel<4, 8, false, 128>, attn_stream_kernel<4, 16, false, 128>},
       {attn_stream_kernel<8, 4, false, 128>, attn_stream_kernel<8, 8, false, 128>, attn_stream_kernel<8, 16, false, 128>},
       {attn_stream_kernel<16, 4, false, 128>, attn_stream_kernel<16, 8, false, 128>, attn_stream_kernel<16, 16, false, 128>}},
      {{attn_stream_kernel<4, 4, true, 128>, attn_stream_kernel<4, 8, true, 128>, attn_stream_kernel<4, 16, true, 128>},
       {attn_stream_kernel<8, 4, true, 128>, attn_stream_kernel<8, 8, true, 128>, attn_stream_kernel<8, 16, true, 128>},
       {attn_stream_kernel<16, 4, true, 128>, attn_stream_kernel<16, 8, true, 128>, attn_stream_kernel<16, 16, true, 128>}},
      {{attn_stream_kernel<4, 4, false, 64>, attn_stream_kernel<4, 8, false, 64>, attn_stream_kernel<4, 16, false, 64>},
       {attn_stream_kernel<8, 4, false, 64>, attn_stream_kernel<8, 8, false, 64>, attn_stream_kernel<8, 16, false, 64>},
       {attn_stream_kernel<16, 4, false, 64>, attn_stream_kernel<16, 8, false, 64>, attn_stream_kernel<16, 16, false, 64>}}};
  return table[dh == 64 ? 2 : paged ? 1 : 0][ki][vi];
}

static void set_attrs_once() {
  static bool done = false;  // benign race: idempotent attributes
  if (!done) {
    for (int var : {0, 1, 2})
      for (int kb : {4, 8, 16})
        for (int vb : {4, 8, 16})
          cudaFuncSetAttribute(kernel_for(kb, vb, var == 1, var == 2 ? 64 : 128),
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem_for(kb, vb));
    done = true;
  }
}

cudaError_t launch_attn_stream(const AttnArgs& a, int kbits, int vbits, cudaStream_t st) {
  set_attrs_once();
  // the misc region must fit below the first 64 KiB boundary of the shared window (the dynamic
  // allocation starts after the per-block reserved shared memory)
  static int reserved = -1;
  if (reserved < 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) v = 1024;
    reserved = v;
  }
  if (reserved + kMiscBytes > 65536) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg = {};
  const int sms = device_sm_count();
  cfg.gridDim = dim3(a.V < sms ? a.V : sms, 1, 1);   // persistent beyond one CTA per SM
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem_for(kbits, vbits);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel_for(kbits, vbits, a.bt != nullptr, a.D), a);
}

}  // namespace vecinfer
