// Host side of vecinfer_attn_decode: validation, split heuristic, workspace layout, dispatch.
#include <stdlib.h>

#include "attn_common.cuh"


using namespace vecinfer;

namespace vecinfer {
// Separate split-merge kernel (PDL): launched right behind the attention kernel, it waits for the
// attention grid to complete (griddepcontrol.wait gives completion + visibility of the partials,
// so the attention CTAs need no fence/atomic), then merges the S partials of one (b, h_kv) unit.
__global__ void __launch_bounds__(512) split_merge_kernel(const AttnArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  merge_splits<512>(a, blockIdx.x % a.B, blockIdx.x / a.B);
}
}  // namespace vecinfer

namespace {

// VECINFER_MERGE=kernel selects the separate merge kernel, =fused the last-CTA merge (default)
int merge_mode_from_env() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("VECINFER_MERGE");
    mode = (e && e[0] == 'k') ? 1 : 0;
  }
  return mode;
}

constexpr int kMaxSplits = 128;
constexpr int64_t kMinTokensPerSplit = 256;   // measured: N = 1024 runs S = 4 (5.4 us) instead of S = 2 (6.1 us)

bool vq_d4(const vecinfer_vq_t& c) {
  return (c.head_dim == 128 || c.head_dim == 64) && c.sub_dim == 4 &&
         (c.code_bits == 4 || c.code_bits == 8 || c.code_bits == 16);
}
// the paper's other configurations (NEXT-2): D = 128, d8b8, d8b12, d4b10, d2b8
bool vq_next2(const vecinfer_vq_t& c) {
  return c.head_dim == 128 && ((c.sub_dim == 8 && (c.code_bits == 8 || c.code_bits == 12 || c.code_bits == 16)) ||
                               (c.sub_dim == 4 && c.code_bits == 10) || (c.sub_dim == 2 && c.code_bits == 8));
}
bool vq_ok(const vecinfer_vq_t& c) { return vq_d4(c) || vq_next2(c); }
// kernel format id: b for the d = 4 byte-aligned formats, else 100 d + b (attn_tiles.cuh)
int fmt_id(const vecinfer_vq_t& c) { return vq_d4(c) ? c.code_bits : 100 * c.sub_dim + c.code_bits; }

struct WsLayout {
  size_t part_o, part_l, counter, elem, total;
};

// counters: one 64-bit word per unit; split partials (split/LUT kernels): U*S x (L [4], o [4][128])
// fp32; stream elements (stream kernel, auto mode only): (U + #SMs) x [4][128] 64-bit words.  The
// layout depends on the call's (B, H_kv, S), so one workspace reused by calls of different shapes
// sees every word in several roles: every kernel therefore leaves EVERY word it wrote at zero on
// exit (counters return to zero, published elements and fp32 partials are zeroed by their
// consumer), and zero is the "empty" value of every region.
WsLayout ws_layout(int32_t B, int32_t H_kv, int32_t S, bool stream_region) {
  WsLayout w;
  const size_t units = static_cast<size_t>(B) * H_kv;
  w.counter = 0;
  w.part_l = ((units * sizeof(unsigned long long)) + 255) & ~size_t(255);   // 64-bit counters / barriers
  w.part_o = w.part_l + ((units * S * 4 * sizeof(float) + 255) & ~size_t(255));
  w.elem = w.part_o + ((units * S * 4 * 128 * sizeof(float) + 255) & ~size_t(255));
  // (explicit S with the forced stream algo: U*S pieces)
  const size_t v = static_cast<size_t>(device_sm_count()) > units * S ? device_sm_count() : units * S;
  const size_t slots = stream_region ? units + v : 0;
  w.total = w.elem + slots * 4 * 128 * sizeof(unsigned long long);
  return w;
}

// GQA groups of 5..8 query heads run as two virtual KV heads per KV head (head_map in
// attn_common.cuh); every plan below is made over the virtual heads.
static int hsplit_of(int32_t H_q, int32_t H_kv) {
  return (H_kv > 0 && H_q % H_kv == 0 && H_q / H_kv > 4) ? 2 : 1;
}

// Stream kernel (attn_stream.cu) for batch decode: B*H_kv >= #SMs units over V = #SMs CTAs (a
// unit crossing a CTA boundary is split in two and merged).  VECINFER_STREAM=0 disables it,
// =1 forces it for any auto-split call (experiments).
// stream partition: virtual tokens charged for each split-unit start (a CTA's extra segment costs
// its table fill, first-tile latency and combine; measured at cfg3: CTAs with 5 segments ran their
// rounds 6 us longer than those with 4).  Sweep 0 / 512 / 1024 / 2048 / 3072 over five batch shapes
// (profiles/r02/exp_stream_seg_cost.txt): 1024 is best overall (cfg3 105.8 -> 103.9 us).
// VECINFER_SEG_COST overrides (experiments).
static int seg_cost_tokens() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VECINFER_SEG_COST");
    v = e ? atoi(e) : 1024;
    if (v < 0) v = 0;
  }
  return v;
}

static int stream_mode_from_env() {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("VECINFER_STREAM");
    mode = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  return mode;
}
}  // namespace

// the algo argument without / with the VECINFER_ATTN_FLAG_EARLY_CACHE launch-ordering bit
static vecinfer_attn_algo_t algo_base(vecinfer_attn_algo_t a) {
  return static_cast<vecinfer_attn_algo_t>(static_cast<uint32_t>(a) & ~static_cast<uint32_t>(VECINFER_ATTN_FLAG_EARLY_CACHE));
}
static bool algo_early(vecinfer_attn_algo_t a) {
  return (static_cast<uint32_t>(a) & static_cast<uint32_t>(VECINFER_ATTN_FLAG_EARLY_CACHE)) != 0;
}

namespace vecinfer {
int encode_launch_count(int64_t nbt, int H, const vecinfer_vq_t& k, const vecinfer_vq_t& v);   // encode.cu
}

struct SplitPlan;
static SplitPlan plan_splits(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits);

// Stream partition (attn_stream.cu) or split kernel (attn_mma.cu)?  With B*H_kv >= #SMs the split
// kernel's whole-unit waves leave SMs idle, so the stream partition runs.  With fewer units the
// split plan may still leave SMs idle (units * S CTAs rounded to waves) while the stream partition
// gives every SM the same token count but pays more per CTA (segment setup, one more piece merge):
// a cost model in tokens of one CTA picks the cheaper (steady state ~2.98 ns per token and CTA on
// B200; fixed costs ~6.5 us split with merge, ~4 us single split, ~10 us stream -- fitted to the
// B = 2..16 x N = 8k..128k timings in DESIGN.md).
static bool use_stream(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits, bool lut,
                       bool forced = false);

// Split plan: one CTA per SM (kernel N4: 16 warps, all 64K registers), so the grid B*H_kv*S
// is sized in waves of SMs.  Cost model in "tokens of one CTA" (calibrated from the phase
// timeline on B200, scripts/phase_attn.py): prologue ~370, DSMEM cluster merge ~250, global
// fence/atomic/last-CTA merge ~1200, single split ~125.  Cluster path: the S <= 16 splits of a
// (b, h_kv) form one thread-block cluster (limited by cudaOccupancyMaxActiveClusters).
struct SplitPlan {
  int S;
  int cluster;
};

static SplitPlan plan_splits(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits) {
  const int64_t units = static_cast<int64_t>(B) * H_kv;
  const int sms = device_sm_count();
  if (num_splits > 0) {
    const int S = num_splits > kMaxSplits ? kMaxSplits : num_splits;
    const bool cl = S > 1 && S <= 16 && attn_mma_max_active_clusters(S) > 0;
    return {S, cl ? 1 : 0};
  }
  int64_t smax = (n_tokens_max + kMinTokensPerSplit - 1) / kMinTokensPerSplit;
  if (smax < 1) smax = 1;
  if (smax > kMaxSplits) smax = kMaxSplits;
  SplitPlan best{1, 0};
  double best_cost = 1e300;
  for (int s = 1; s <= smax; ++s) {
    const double per = static_cast<double>((n_tokens_max + s - 1) / s) + 370.0;
    // global-merge (or single-split) path
    const int64_t waves = (units * s + sms - 1) / sms;
    const double cg = static_cast<double>(waves) * (per + (s == 1 ? 125.0 : 1200.0));
    if (cg < best_cost - 1e-9) { best_cost = cg; best = {s, 0}; }
    if (s >= 2 && s <= 16) {
      const int mac = attn_mma_max_active_clusters(s);
      if (mac > 0) {
        const int64_t wc = (units + mac - 1) / mac;
        const double cc = static_cast<double>(wc) * (per + 250.0);
        if (cc < best_cost - 1e-9) { best_cost = cc; best = {s, 1}; }
      }
    }
  }
  return best;
}

static bool use_stream(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits, bool lut, bool forced) {
  if (forced) return true;
  if (lut || num_splits > 0) return false;
  const int m = stream_mode_from_env();
  if (m >= 0) return m == 1;
  const int64_t U = static_cast<int64_t>(B) * H_kv;
  const int sms = device_sm_count();
  if (U >= sms) return true;
  if (n_tokens_max <= 0) return false;
  const SplitPlan p = plan_splits(B, H_kv, n_tokens_max, 0);
  int64_t waves;
  if (p.cluster) {
    const int mac = attn_mma_max_active_clusters(p.S);
    waves = (U + (mac > 0 ? mac : 1) - 1) / (mac > 0 ? mac : 1);
  } else {
    waves = (U * p.S + sms - 1) / sms;
  }
  const double chunk = static_cast<double>((n_tokens_max + p.S - 1) / p.S);
  const double t_split = static_cast<double>(waves) * (chunk + (p.S > 1 ? 2200.0 : 1350.0));
  const double t_stream = static_cast<double>(U) * static_cast<double>(n_tokens_max) / sms + 3350.0;
  return t_stream < t_split;
}

// diagnostics: max co-resident clusters of the attention kernel for a cluster size (0 = none)
extern "C" int32_t vecinfer_debug_attn_max_clusters(int32_t cluster_size) {
  return attn_mma_max_active_clusters(cluster_size);
}

extern "C" int32_t vecinfer_attn_num_splits(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits) {
  if (B <= 0 || H_kv <= 0) return 1;
  if (use_stream(B, H_kv, n_tokens_max, num_splits, false)) {
    const int64_t U = static_cast<int64_t>(B) * H_kv, V = device_sm_count();
    return static_cast<int32_t>((V + U - 1) / U);   // pieces per unit (upper bound)
  }
  return plan_splits(B, H_kv, n_tokens_max, num_splits).S;
}

extern "C" int32_t vecinfer_attn_num_ctas(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits) {
  if (B <= 0 || H_kv <= 0) return 0;
  if (use_stream(B, H_kv, n_tokens_max, num_splits, false)) return device_sm_count();
  return B * H_kv * plan_splits(B, H_kv, n_tokens_max, num_splits).S;
}

extern "C" size_t vecinfer_attn_workspace_bytes(int32_t B, int32_t H_q, int32_t H_kv, int32_t D, int64_t n_tokens_max,
                                                int32_t num_splits) {
  (void)H_q; (void)D;
  if (B <= 0 || H_kv <= 0) return 0;
  const int32_t Hv = H_kv * hsplit_of(H_q, H_kv);
  const int32_t S = plan_splits(B, Hv, n_tokens_max, num_splits).S;
  return ws_layout(B, Hv, S, true).total;
}

struct AppendArgs {
  const void* k_new;
  const void* v_new;
  int64_t kn_sb, kn_sh, vn_sb, vn_sh;
  const float* inv_lambda;
  const int32_t* write_pos;
  uint32_t* err;
};

static vecinfer_status_t attn_impl(const void* q_bf16, int32_t B, int32_t H_q, int32_t H_kv,
                                   int64_t q_stride_b, int64_t q_stride_h, const float* lambda,
                                   const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride,
                                   int64_t cv_head_stride, vecinfer_vq_t kcfg, vecinfer_vq_t vcfg,
                                   const uint8_t* k_codes, const uint8_t* v_codes, int64_t n_cap,
                                   const int32_t* seq_lens, int64_t tok_begin, int64_t tok_end,
                                   float softmax_scale, int32_t num_splits, vecinfer_attn_algo_t algo,
                                   void* o, vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                   size_t workspace_bytes, vecinfer_stream_t stream, const AppendArgs* app,
                                   const vecinfer_residual_t* res, bool res_append,
                                   const vecinfer_paged_t* pg = nullptr, const vecinfer_xrank_t* xr = nullptr) {
  const bool early = algo_early(algo);
  algo = algo_base(algo);
  if (!q_bf16 || !lambda || !ck_bf16 || !cv_bf16 || !k_codes || !v_codes || !seq_lens || !o)
    return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: NULL pointer");
  if (o_dtype != VECINFER_BF16 && o_dtype != VECINFER_F32) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: bad o_dtype");
  if (algo != VECINFER_ATTN_AUTO && algo != VECINFER_ATTN_DEQUANT_MMA && algo != VECINFER_ATTN_LUT &&
      algo != VECINFER_ATTN_DEQUANT_MMA_STREAM && algo != VECINFER_ATTN_DEQUANT_TC)
    return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: bad algo");
  const bool tc = algo == VECINFER_ATTN_DEQUANT_TC;
  if (tc && (pg || kcfg.head_dim != 128 || vcfg.head_dim != 128 || kcfg.sub_dim != 4 || vcfg.sub_dim != 4 ||
             (kcfg.code_bits != 4 && kcfg.code_bits != 8) || (vcfg.code_bits != 4 && vcfg.code_bits != 8 && vcfg.code_bits != 16)))
    return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: DEQUANT_TC needs a contiguous cache, D = 128, d = 4 and K codes "
                "of 4 or 8 bits");
  if (B <= 0 || H_q <= 0 || H_kv <= 0 || n_cap <= 0) return fail(VECINFER_ERR_SHAPE, "attn_decode: non-positive size");
  if (H_q % H_kv != 0) return fail(VECINFER_ERR_SHAPE, "attn_decode: H_q %% H_kv != 0");
  const int Gfull = H_q / H_kv;
  if (Gfull > 8) return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: GQA group %d > 8", Gfull);
  if (Gfull > 4 && algo == VECINFER_ATTN_LUT)
    return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: the LUT variant supports GQA groups <= 4");
  const int hsplit = hsplit_of(H_q, H_kv);
  const int G = hsplit == 1 ? Gfull : 4;   // query heads per virtual head (the last may hold fewer)
  const int32_t H_kv_real = H_kv;
  H_kv *= hsplit;                          // from here on: virtual KV heads
  if (!vq_ok(kcfg) || !vq_ok(vcfg))
    return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: supported configs are D in {64, 128} with d=4, code_bits in "
                "{4,8,16}, and D = 128 d8b8 / d8b12 / d4b10 / d2b8");
  const bool next2 = vq_next2(kcfg) || vq_next2(vcfg);
  const int kf = fmt_id(kcfg), vf = fmt_id(vcfg);
  if (next2 && (!attn_mma_supports(kf, vf, kcfg.head_dim) || algo == VECINFER_ATTN_LUT ||
                algo == VECINFER_ATTN_DEQUANT_MMA_STREAM))
    return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: d8b8 / d8b12 / d4b10 / d2b8 run the split DEQUANT_MMA kernel for "
                "the pairs (f, f), (d4b10, d8b12), (d8b12, d8b8)");
  if (kcfg.head_dim != vcfg.head_dim) return fail(VECINFER_ERR_SHAPE, "attn_decode: K and V head_dim differ");
  const int D = kcfg.head_dim;
  if (D == 64 && (algo == VECINFER_ATTN_LUT ||
                  (algo == VECINFER_ATTN_DEQUANT_MMA_STREAM && (res || app || pg))))
    return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: head_dim 64 runs the stream kernel only without a residual "
                "window, fused append or paging");
  if (algo == VECINFER_ATTN_LUT && (kcfg.code_bits != 8 || vcfg.code_bits != 8))
    return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: the LUT variant is implemented for b2d4 only");
  if (tok_begin < 0 || (tok_end >= 0 && tok_end < tok_begin))
    return fail(VECINFER_ERR_SHAPE, "attn_decode: bad token range [%lld, %lld)", (long long)tok_begin, (long long)tok_end);
  if (!(softmax_scale > 0.f) || !isfinite(softmax_scale)) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: softmax_scale must be finite > 0");
  if (num_splits < 0) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: num_splits < 0");
  if (q_stride_h % 4 || q_stride_b % 4 || q_stride_h < 0 || q_stride_b < 0 || !aligned(q_bf16, 8))
    return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: q must be 8-byte aligned with strides multiple of 4");
  if (!aligned(lambda, 16) || !aligned(ck_bf16, 8) || !aligned(cv_bf16, 8) || !aligned(k_codes, 16) ||
      !aligned(v_codes, 16) || ck_head_stride % 4 || cv_head_stride % 4 || ck_head_stride < 0 || cv_head_stride < 0)
    return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: misaligned lambda/codebooks/codes");
  const int64_t range = tok_end >= 0 ? (tok_end - tok_begin < n_cap ? tok_end - tok_begin : n_cap) : n_cap;
  const bool lut = algo == VECINFER_ATTN_LUT;
  if (pg) {   // paged code cache: split or stream kernel, 32-aligned token ranges
    const vecinfer_status_t v = check_paged(pg, n_cap, "attn_decode_paged");
    if (v != VECINFER_OK) return v;
    if (lut) return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode_paged: paged caches run the DEQUANT_MMA kernels only");
    if (tok_begin % 32 != 0) return fail(VECINFER_ERR_SHAPE, "attn_decode_paged: tok_begin must be a multiple of 32");
  }
  const int64_t n_sms = device_sm_count();
  if (xr) {   // fused cross-rank merge: the single-wave spin merge of the split kernel
    if (xr->world < 1 || xr->world > 16 || xr->rank < 0 || xr->rank >= xr->world)
      return fail(VECINFER_ERR_SHAPE, "attn_decode_xr: rank %d / world %d outside [0, world), world in 1..16",
                  xr->rank, xr->world);
    if (!xr->windows) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode_xr: NULL windows");
    if (xr->rows_max < static_cast<int64_t>(B) * H_q)
      return fail(VECINFER_ERR_SHAPE, "attn_decode_xr: windows sized for %lld rows < B*H_q", (long long)xr->rows_max);
    if (pg || lut || tc || next2 || D != 128 || algo == VECINFER_ATTN_DEQUANT_MMA_STREAM ||
        static_cast<int64_t>(B) * H_kv * 2 > n_sms)
      return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode_xr: needs the single-wave split kernel (contiguous cache, "
                  "D = 128 with d = 4 books, B*H_kv*2 <= %lld SMs, DEQUANT_MMA / AUTO); use attn_decode + "
                  "merge_lse_p2p", (long long)n_sms);
  }
  // stream partition: D = 128, or D = 64 without a residual window, fused append or paging (those
  // run the split kernel's persistent grid)
  const bool use_sk = !xr && !tc && !next2 && (D == 128 || (!res && !app && !pg)) && use_stream(B, H_kv, range, num_splits, lut, algo == VECINFER_ATTN_DEQUANT_MMA_STREAM);
  SplitPlan plan = use_sk ? SplitPlan{1, 0} : plan_splits(B, H_kv, range, num_splits);
  if (xr) {   // 2 <= S <= #SMs / (B*H_kv), no cluster: every CTA co-resident for the spin merge
    const int64_t smax = n_sms / (static_cast<int64_t>(B) * H_kv);
    if (plan.S < 2) plan.S = 2;
    if (plan.S > smax) plan.S = static_cast<int>(smax);
    plan.cluster = 0;
  }
  if (D == 64) plan.cluster = 0;   // the DSMEM cluster merge is written for 128-dim rows
  // formats without any shared table (b4d4 d = 4 and d8b16 books through L1/L2) get the smallest
  // shared allocation -- no cluster buffer, so never the DSMEM cluster merge
  if ((kf == 16 || kf == 816) && (vf == 16 || vf == 816)) plan.cluster = 0;
#ifndef VECINFER_CODE_TMA
#define VECINFER_CODE_TMA 0
#endif
  if (VECINFER_CODE_TMA > 0 && kf == 8 && vf == 8) plan.cluster = 0;   // TMA stages replace the cluster buffer
  const int32_t S = plan.S;
  // (the offsets follow the planner's S, as vecinfer_attn_workspace_bytes sized it; the xr path's
  // S <= max(2, that S) fits the element region, which holds max(#SMs, units * S) + units rows)
  const WsLayout wl = ws_layout(B, H_kv, plan_splits(B, H_kv, range, num_splits).S, true);
  const int64_t U = static_cast<int64_t>(B) * H_kv;
  const int64_t sms = device_sm_count();
  const int64_t V = use_sk ? (num_splits > 0 ? U * (num_splits > kMaxSplits ? kMaxSplits : num_splits) : sms) : U * S;
  if (use_sk && U * V >= (int64_t(1) << 42))
    return fail(VECINFER_ERR_SHAPE, "attn_decode: B*H_kv*num_splits too large for the stream partition");
  const bool stream_split = use_sk && (V > U || U % V != 0);
  if (((S > 1 && !plan.cluster) || stream_split) && (!workspace || workspace_bytes < wl.total || !aligned(workspace, 256)))
    return fail(VECINFER_ERR_WORKSPACE, "attn_decode: workspace needs %zu bytes (256-B aligned)", wl.total);
  if (B > 65535 || H_kv > 65535) return fail(VECINFER_ERR_SHAPE, "attn_decode: grid too large");
  if (res) {
    if (algo == VECINFER_ATTN_LUT) return fail(VECINFER_ERR_UNSUPPORTED, "attn_decode: residual window needs the MMA kernel");
    if (!res->k || !res->v || !res->lens) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: residual NULL pointer");
    if (res->r_cap <= 0) return fail(VECINFER_ERR_SHAPE, "attn_decode: residual r_cap <= 0");
    if (!aligned(res->k, 16) || !aligned(res->v, 16) || res->stride_b % 8 || res->stride_h % 8 || res->stride_b < 0 ||
        res->stride_h < 0)
      return fail(VECINFER_ERR_INVALID_ARG, "attn_decode: residual rows must be 16-byte aligned (strides multiple of 8)");
  }

  AttnArgs a;
  a.q = static_cast<const uint16_t*>(q_bf16);
  a.q_sb = q_stride_b; a.q_sh = q_stride_h;
  a.B = B; a.Hq = H_q; a.Hkv = H_kv; a.G = G;
  a.Hc = H_kv_real; a.hsplit = hsplit; a.Gfull = Gfull;
  a.lambda = lambda;
  a.ck = static_cast<const uint16_t*>(ck_bf16);
  a.cv = static_cast<const uint16_t*>(cv_bf16);
  a.ck_hs = ck_head_stride; a.cv_hs = cv_head_stride;
  a.kcodes = k_codes; a.vcodes = v_codes; a.n_cap = n_cap;
  a.bt = pg ? pg->block_table : nullptr;
  a.bt_stride = pg ? pg->bt_stride : 0;
  a.page_shift = pg ? __builtin_ctz(static_cast<unsigned>(pg->page_size)) : 0;
  a.n_pages = pg ? pg->n_pages : 0;
  a.seq_lens = seq_lens; a.tok_begin = tok_begin; a.tok_end = tok_end;
  a.D = D;
  a.qscale = static_cast<float>((1.0 / sqrt(static_cast<double>(D))) * static_cast<double>(softmax_scale) *
                                1.4426950408889634);
  a.S = S;
  a.n_items = B * H_kv * S;
  a.U = static_cast<int>(U);
  a.seg_cost = seg_cost_tokens();
  a.V = static_cast<int>(V);
  a.rcpU = 1.0 / static_cast<double>(U);
  a.rcpV = 1.0 / static_cast<double>(V);
  a.merge = !stream_split ? kMergeNone : (V <= sms ? kMergeSpin : kMergeLast);
  a.cluster = plan.cluster;
  a.tc = tc ? 1 : 0;
  a.merge_kernel = (!xr && S > 1 && !plan.cluster && algo != VECINFER_ATTN_LUT && D == 128) ? merge_mode_from_env() : 0;
  // every CTA co-resident (one CTA per SM, grid <= SMs): spin-barrier + sliced merge
  a.merge_spin = (S > 1 && !plan.cluster && !a.merge_kernel && algo != VECINFER_ATTN_LUT &&
                  static_cast<int64_t>(B) * H_kv * S <= n_sms && (xr || !getenv("VECINFER_NO_SPIN"))) ? 1 : 0;
  a.early = early ? 1 : 0;
  a.xr_P = xr ? xr->world : 0;
  a.xr_rank = xr ? xr->rank : 0;
  a.xr_win = xr ? xr->windows : nullptr;
  a.xr_rows = xr ? xr->rows_max : 0;
  a.xr_err = xr ? xr->err_flags : nullptr;
  a.o = o; a.o_f32 = (o_dtype == VECINFER_F32); a.lse = lse;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  a.counter = S > 1 ? reinterpret_cast<uint32_t*>(ws + wl.counter) : nullptr;
  a.part_l = S > 1 ? reinterpret_cast<float*>(ws + wl.part_l) : nullptr;
  a.part_o = S > 1 ? reinterpret_cast<float*>(ws + wl.part_o) : nullptr;
  a.part_elem = (stream_split || a.merge_spin) ? reinterpret_cast<unsigned long long*>(ws + wl.elem) : nullptr;
  if (stream_split) a.counter = reinterpret_cast<uint32_t*>(ws + wl.counter);
  a.phase = phase_buffer();
  a.append = app != nullptr && !res_append;   // encode into the codes (not a residual append)
  a.knew = app ? static_cast<const uint16_t*>(app->k_new) : nullptr;
  a.vnew = app ? static_cast<const uint16_t*>(app->v_new) : nullptr;
  a.kn_sb = app ? app->kn_sb : 0; a.kn_sh = app ? app->kn_sh : 0;
  a.vn_sb = app ? app->vn_sb : 0; a.vn_sh = app ? app->vn_sh : 0;
  a.inv_lambda = app ? app->inv_lambda : nullptr;
  a.write_pos = app ? app->write_pos : nullptr;
  a.err = app ? app->err : nullptr;
  a.kcodes_w = const_cast<uint8_t*>(k_codes);
  a.vcodes_w = const_cast<uint8_t*>(v_codes);
  a.inv_sqrt_d = static_cast<float>(1.0 / sqrt(static_cast<double>(D)));
  a.res = res != nullptr;
  a.kres = res ? static_cast<const uint16_t*>(res->k) : nullptr;
  a.vres = res ? static_cast<const uint16_t*>(res->v) : nullptr;
  a.res_sb = res ? res->stride_b : 0;
  a.res_sh = res ? res->stride_h : 0;
  a.r_cap = res ? res->r_cap : 0;
  a.res_lens = res ? res->lens : nullptr;
  a.res_append = res_append ? 1 : 0;
  a.qscale_raw = static_cast<float>(static_cast<double>(softmax_scale) * 1.4426950408889634);
  cudaStream_t st = as_stream(stream);
  if (lut) {
    launch_attn_lut(a, kcfg.code_bits, vcfg.code_bits, st);
    return check_launch("attn_decode (lut)");
  }
  const cudaError_t e = use_sk ? launch_attn_stream(a, kcfg.code_bits, vcfg.code_bits, st)
                               : launch_attn_mma(a, kf, vf, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(VECINFER_ERR_CUDA, "attn_decode: launch failed: %s", cudaGetErrorString(e));
  }
  if (a.merge_kernel) {
    const cudaError_t e2 = launch_pdl(split_merge_kernel, dim3(static_cast<unsigned>(B) * H_kv), dim3(512), 0, st, a);
    if (e2 != cudaSuccess) {
      cudaGetLastError();
      return fail(VECINFER_ERR_CUDA, "attn_decode: merge launch failed: %s", cudaGetErrorString(e2));
    }
  }
  return check_launch("attn_decode");
}

extern "C" vecinfer_status_t vecinfer_attn_decode(const void* q_bf16, int32_t B, int32_t H_q, int32_t H_kv,
                                                  int64_t q_stride_b, int64_t q_stride_h, const float* lambda,
                                                  const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride,
                                                  int64_t cv_head_stride, vecinfer_vq_t kcfg, vecinfer_vq_t vcfg,
                                                  const uint8_t* k_codes, const uint8_t* v_codes, int64_t n_cap,
                                                  const int32_t* seq_lens, int64_t tok_begin, int64_t tok_end,
                                                  float softmax_scale, int32_t num_splits, vecinfer_attn_algo_t algo,
                                                  void* o, vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                                  size_t workspace_bytes, vecinfer_stream_t stream,
                                                  const vecinfer_residual_t* residual) {
  return attn_impl(q_bf16, B, H_q, H_kv, q_stride_b, q_stride_h, lambda, ck_bf16, cv_bf16, ck_head_stride,
                   cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, seq_lens, tok_begin, tok_end, softmax_scale,
                   num_splits, algo, o, o_dtype, lse, workspace, workspace_bytes, stream, nullptr, residual, false);
}

extern "C" vecinfer_status_t vecinfer_attn_decode_paged(const void* q_bf16, int32_t B, int32_t H_q, int32_t H_kv,
                                                  int64_t q_stride_b, int64_t q_stride_h, const float* lambda,
                                                  const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride,
                                                  int64_t cv_head_stride, vecinfer_vq_t kcfg, vecinfer_vq_t vcfg,
                                                  const uint8_t* k_codes, const uint8_t* v_codes, int64_t n_cap,
                                                  const int32_t* seq_lens, int64_t tok_begin, int64_t tok_end,
                                                  float softmax_scale, int32_t num_splits, vecinfer_attn_algo_t algo,
                                                  void* o, vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                                  size_t workspace_bytes, vecinfer_stream_t stream,
                                                  const vecinfer_residual_t* residual, const vecinfer_paged_t* paged) {
  if (!paged) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode_paged: NULL paged descriptor");
  return attn_impl(q_bf16, B, H_q, H_kv, q_stride_b, q_stride_h, lambda, ck_bf16, cv_bf16, ck_head_stride,
                   cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, seq_lens, tok_begin, tok_end, softmax_scale,
                   num_splits, algo, o, o_dtype, lse, workspace, workspace_bytes, stream, nullptr, residual, false, paged);
}

// Whether vecinfer_decode_step runs the append-encode inside the attention launch.  Split kernel:
// only single-wave grids (the owner CTA's encode then hides behind the other CTAs' longer splits;
// with several waves every wave would carry it, and one separate append launch is cheaper).
// Stream kernel: always when every CTA is resident (the partition budgets the encode).  Never for
// 16-bit codebooks or the LUT variant.
static bool decode_fuses(int32_t B, int32_t H_kv, int64_t n_cap, vecinfer_vq_t kcfg, vecinfer_vq_t vcfg,
                         int32_t num_splits, vecinfer_attn_algo_t algo, bool paged = false) {
  if (algo == VECINFER_ATTN_LUT || B <= 0 || H_kv <= 0) return false;
  // NEXT-2 formats: the split kernel fuses the append for the books in its shared tables (d8b8,
  // d2b8, d4b10, d8b12 -- VECINFER_NO_FUSE_D8B12 keeps d8b12 on the separate launches, experiments);
  // d8b16 keeps the separate encode launch
  auto small_next2 = [](const vecinfer_vq_t& c) {
    return vq_next2(c) && ((c.sub_dim == 8 && c.code_bits == 8) || (c.sub_dim == 4 && c.code_bits == 10) ||
                           (c.sub_dim == 2 && c.code_bits == 8) ||
                           (c.sub_dim == 8 && c.code_bits == 12 && !getenv("VECINFER_NO_FUSE_D8B12")));
  };
  const bool n2 = vq_next2(kcfg) || vq_next2(vcfg);
  if (n2 && !(small_next2(kcfg) && small_next2(vcfg))) return false;
  if (!n2 && (kcfg.code_bits > 8 || vcfg.code_bits > 8)) return false;
  if (kcfg.head_dim != 128 && kcfg.head_dim != 64) return false;
  const int64_t units = static_cast<int64_t>(B) * H_kv;
  if (algo == VECINFER_ATTN_DEQUANT_MMA_STREAM)   // (D = 64: the stream kernel has no fused append)
    return kcfg.head_dim == 128 && (num_splits == 0 || units * num_splits <= device_sm_count());
  if (!n2 && algo != VECINFER_ATTN_DEQUANT_TC && kcfg.head_dim == 128 && use_stream(B, H_kv, n_cap, num_splits, false)) return true;
  const SplitPlan plan = plan_splits(B, H_kv, n_cap, num_splits);
  const int mac = plan.cluster ? attn_mma_max_active_clusters(plan.S) : 0;
  const int64_t waves = plan.cluster ? (units + (mac > 0 ? mac : 1) - 1) / (mac > 0 ? mac : 1)
                                     : (units * plan.S + device_sm_count() - 1) / device_sm_count();
  return waves <= 1;
}

// which attention kernel a call runs: 0 split (attn_mma.cu), 1 stream (attn_stream.cu), 2 LUT
extern "C" int32_t vecinfer_attn_kernel_kind(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits,
                                             vecinfer_attn_algo_t algo) {
  algo = algo_base(algo);
  if (algo == VECINFER_ATTN_LUT) return 2;
  if (algo == VECINFER_ATTN_DEQUANT_TC) return 0;
  return use_stream(B, H_kv, n_tokens_max, num_splits, false, algo == VECINFER_ATTN_DEQUANT_MMA_STREAM) ? 1 : 0;
}

// kernel launches of one vecinfer_decode_step call (1 = append fused into the attention launch)
extern "C" int32_t vecinfer_decode_step_launches(int32_t B, int32_t H_kv, int64_t n_cap, vecinfer_vq_t kcfg,
                                                 vecinfer_vq_t vcfg, int32_t num_splits, vecinfer_attn_algo_t algo,
                                                 int32_t residual_append) {
  if (residual_append) return 1;
  algo = algo_base(algo);
  if (decode_fuses(B, H_kv, n_cap, kcfg, vcfg, num_splits, algo)) return 1;
  // separate append: 16-bit d = 4 and d8b12 / d8b16 books take a filter + selection launch pair
  // (plus a generic launch for the other stream of a mixed NEXT-2 pair); others one encode launch
  return 1 + encode_launch_count(B, H_kv, kcfg, vcfg);
}

extern "C" size_t vecinfer_decode_step_workspace_bytes(int32_t B, int32_t H_q, int32_t H_kv, int64_t n_cap,
                                                       vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, int32_t num_splits) {
  const size_t a = (vecinfer_attn_workspace_bytes(B, H_q, H_kv, 128, n_cap, num_splits) + 255) & ~size_t(255);
  return a + vecinfer_encode_workspace_bytes(B, 1, H_kv, kcfg, vcfg);
}

static vecinfer_status_t decode_step_impl(const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16,
                                                  int32_t B, int32_t H_q, int32_t H_kv, const int64_t q_strides[2],
                                                  const int64_t k_new_strides[2], const int64_t v_new_strides[2],
                                                  const float* lambda, const float* inv_lambda, const void* ck_bf16,
                                                  const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
                                                  vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                                  uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                                  const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
                                                  vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype,
                                                  float* lse, uint32_t* err_flags, void* workspace,
                                                  size_t workspace_bytes, vecinfer_stream_t stream,
                                                  const vecinfer_residual_t* residual, const vecinfer_paged_t* pg,
                                                  const vecinfer_xrank_t* xr = nullptr) {
  if (!k_new_bf16 || !v_new_bf16 || !inv_lambda || !write_pos || !q_strides || !k_new_strides || !v_new_strides)
    return fail(VECINFER_ERR_INVALID_ARG, "decode_step: NULL pointer");
  for (int i = 0; i < 2; ++i)
    if (k_new_strides[i] % 4 || v_new_strides[i] % 4 || k_new_strides[i] < 0 || v_new_strides[i] < 0)
      return fail(VECINFER_ERR_INVALID_ARG, "decode_step: k_new/v_new strides must be non-negative multiples of 4");
  if (!aligned(k_new_bf16, 8) || !aligned(v_new_bf16, 8) || !aligned(inv_lambda, 16))
    return fail(VECINFER_ERR_INVALID_ARG, "decode_step: misaligned k_new/v_new/inv_lambda");
  const vecinfer_attn_algo_t algo_b = algo_base(algo);   // (the early-cache bit stays on `algo`)
  if (residual && residual->append_new) {   // the new token goes to the residual window (raw copy)
    if (algo_b == VECINFER_ATTN_LUT) return fail(VECINFER_ERR_UNSUPPORTED, "decode_step: residual needs the MMA kernel");
    AppendArgs app{k_new_bf16, v_new_bf16, k_new_strides[0], k_new_strides[1], v_new_strides[0], v_new_strides[1],
                   inv_lambda, write_pos, err_flags};
    return attn_impl(q_bf16, B, H_q, H_kv, q_strides[0], q_strides[1], lambda, ck_bf16, cv_bf16, ck_head_stride,
                     cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, seq_lens, 0, -1, softmax_scale, num_splits,
                     algo, o, o_dtype, lse, workspace, workspace_bytes, stream, &app, residual, true, pg, xr);
  }
  const bool fuse = decode_fuses(B, H_kv * hsplit_of(H_q, H_kv), n_cap, kcfg, vcfg, num_splits, algo_b, pg != nullptr);
  if (!fuse) {   // separate append + attention launches (always for the paper-faithful LUT variant)
    const int64_t ks[3] = {k_new_strides[0], 0, k_new_strides[1]};
    const int64_t vs[3] = {v_new_strides[0], 0, v_new_strides[1]};
    // encode workspace (16-bit codebooks) lives behind the attention workspace
    const size_t aw = (vecinfer_attn_workspace_bytes(B, H_q, H_kv, 128, n_cap, num_splits) + 255) & ~size_t(255);
    const size_t ew = vecinfer_encode_workspace_bytes(B, 1, H_kv, kcfg, vcfg);
    if (ew && (!workspace || workspace_bytes < aw + ew))
      return fail(VECINFER_ERR_WORKSPACE, "decode_step: workspace needs %zu bytes", aw + ew);
    void* ews = ew ? static_cast<void*>(static_cast<unsigned char*>(workspace) + aw) : nullptr;
    vecinfer_status_t st =
        pg ? vecinfer_encode_kv_paged(k_new_bf16, v_new_bf16, B, 1, H_kv, ks, vs, inv_lambda, ck_bf16, cv_bf16,
                                      ck_head_stride, cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, write_pos,
                                      err_flags, ews, ew, stream, pg)
           : vecinfer_encode_kv(k_new_bf16, v_new_bf16, B, 1, H_kv, ks, vs, inv_lambda, ck_bf16, cv_bf16,
                                ck_head_stride, cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, write_pos,
                                err_flags, ews, ew, stream);
    if (st != VECINFER_OK) return st;
    // the encode launch just wrote the cache: the attention must not read it before its wait
    return attn_impl(q_bf16, B, H_q, H_kv, q_strides[0], q_strides[1], lambda, ck_bf16, cv_bf16, ck_head_stride,
                     cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, seq_lens, 0, -1, softmax_scale, num_splits,
                     algo_b, o, o_dtype, lse, workspace, workspace_bytes, stream, nullptr, residual, false, pg, xr);
  }
  AppendArgs app{k_new_bf16, v_new_bf16, k_new_strides[0], k_new_strides[1], v_new_strides[0], v_new_strides[1],
                 inv_lambda, write_pos, err_flags};
  return attn_impl(q_bf16, B, H_q, H_kv, q_strides[0], q_strides[1], lambda, ck_bf16, cv_bf16, ck_head_stride,
                   cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, seq_lens, 0, -1, softmax_scale, num_splits,
                   algo, o, o_dtype, lse, workspace, workspace_bytes, stream, &app, residual, false, pg, xr);
}

extern "C" vecinfer_status_t vecinfer_decode_step(const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16,
                                                  int32_t B, int32_t H_q, int32_t H_kv, const int64_t q_strides[2],
                                                  const int64_t k_new_strides[2], const int64_t v_new_strides[2],
                                                  const float* lambda, const float* inv_lambda, const void* ck_bf16,
                                                  const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
                                                  vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                                  uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                                  const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
                                                  vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype,
                                                  float* lse, uint32_t* err_flags, void* workspace,
                                                  size_t workspace_bytes, vecinfer_stream_t stream,
                                                  const vecinfer_residual_t* residual) {
  return decode_step_impl(q_bf16, k_new_bf16, v_new_bf16, B, H_q, H_kv, q_strides, k_new_strides, v_new_strides,
                          lambda, inv_lambda, ck_bf16, cv_bf16, ck_head_stride, cv_head_stride, kcfg, vcfg, k_codes,
                          v_codes, n_cap, write_pos, seq_lens, softmax_scale, num_splits, algo, o, o_dtype, lse,
                          err_flags, workspace, workspace_bytes, stream, residual, nullptr);
}

extern "C" vecinfer_status_t vecinfer_decode_step_paged(
    const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16, int32_t B, int32_t H_q, int32_t H_kv,
    const int64_t q_strides[2], const int64_t k_new_strides[2], const int64_t v_new_strides[2], const float* lambda,
    const float* inv_lambda, const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
    vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes, uint8_t* v_codes, int64_t n_cap,
    const int32_t* write_pos, const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
    vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype, float* lse, uint32_t* err_flags, void* workspace,
    size_t workspace_bytes, vecinfer_stream_t stream, const vecinfer_residual_t* residual,
    const vecinfer_paged_t* paged) {
  if (!paged) return fail(VECINFER_ERR_INVALID_ARG, "decode_step_paged: NULL paged descriptor");
  return decode_step_impl(q_bf16, k_new_bf16, v_new_bf16, B, H_q, H_kv, q_strides, k_new_strides, v_new_strides,
                          lambda, inv_lambda, ck_bf16, cv_bf16, ck_head_stride, cv_head_stride, kcfg, vcfg, k_codes,
                          v_codes, n_cap, write_pos, seq_lens, softmax_scale, num_splits, algo, o, o_dtype, lse,
                          err_flags, workspace, workspace_bytes, stream, residual, paged);
}

extern "C" size_t vecinfer_xr_window_bytes(int32_t P, int64_t rows, int32_t D) {
  if (P <= 0 || rows <= 0 || D <= 0) return 0;
  return static_cast<size_t>(kXrHeaderWords) * 8 + static_cast<size_t>(2) * P * rows * D * 8;
}

extern "C" vecinfer_status_t vecinfer_attn_decode_xr(const void* q_bf16, int32_t B, int32_t H_q, int32_t H_kv,
                                                     int64_t q_stride_b, int64_t q_stride_h, const float* lambda,
                                                     const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride,
                                                     int64_t cv_head_stride, vecinfer_vq_t kcfg, vecinfer_vq_t vcfg,
                                                     const uint8_t* k_codes, const uint8_t* v_codes, int64_t n_cap,
                                                     const int32_t* seq_lens, int64_t tok_begin, int64_t tok_end,
                                                     float softmax_scale, int32_t num_splits, vecinfer_attn_algo_t algo,
                                                     void* o, vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                                     size_t workspace_bytes, vecinfer_stream_t stream,
                                                     const vecinfer_residual_t* residual, const vecinfer_xrank_t* xr) {
  if (!xr) return fail(VECINFER_ERR_INVALID_ARG, "attn_decode_xr: NULL xr descriptor");
  return attn_impl(q_bf16, B, H_q, H_kv, q_stride_b, q_stride_h, lambda, ck_bf16, cv_bf16, ck_head_stride,
                   cv_head_stride, kcfg, vcfg, k_codes, v_codes, n_cap, seq_lens, tok_begin, tok_end, softmax_scale,
                   num_splits, algo, o, o_dtype, lse, workspace, workspace_bytes, stream, nullptr, residual, false,
                   nullptr, xr);
}

extern "C" vecinfer_status_t vecinfer_decode_step_xr(
    const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16, int32_t B, int32_t H_q, int32_t H_kv,
    const int64_t q_strides[2], const int64_t k_new_strides[2], const int64_t v_new_strides[2], const float* lambda,
    const float* inv_lambda, const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
    vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes, uint8_t* v_codes, int64_t n_cap,
    const int32_t* write_pos, const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
    vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype, float* lse, uint32_t* err_flags, void* workspace,
    size_t workspace_bytes, vecinfer_stream_t stream, const vecinfer_residual_t* residual,
    const vecinfer_xrank_t* xr) {
  if (!xr) return fail(VECINFER_ERR_INVALID_ARG, "decode_step_xr: NULL xr descriptor");
  return decode_step_impl(q_bf16, k_new_bf16, v_new_bf16, B, H_q, H_kv, q_strides, k_new_strides, v_new_strides,
                          lambda, inv_lambda, ck_bf16, cv_bf16, ck_head_stride, cv_head_stride, kcfg, vcfg, k_codes,
                          v_codes, n_cap, write_pos, seq_lens, softmax_scale, num_splits, algo, o, o_dtype, lse,
                          err_flags, workspace, workspace_bytes, stream, residual, nullptr, xr);
}
