"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bars (BASELINE north_star): codes bit-exact; attention outputs within 2e-3 max-abs relative
error per (b, h_q) row on the fp32 output, |dL| <= 2e-3; calibration bit-exact.
Inputs: seeded synthetic (synth/) + frozen oracle-fitted codebooks; nothing the oracle sees comes
from the CUDA path.
"""
import numpy as np
import pytest

import synth
from oracle import ref
from helpers import TOL_L, TOL_O, load_codebooks, row_rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402

DEV = "cuda"
CB = load_codebooks()


def t_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(DEV).to(torch.bfloat16)


def t_f32(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(DEV)


def t_u8(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint8)).to(DEV)


def t_i32(x):
    return torch.tensor(np.asarray(x, dtype=np.int32), device=DEV)


# ------------------------------------------------------------------------ calibrate (Eq. 4)
@pytest.mark.parametrize("n_tok", [1, 7, 4096, 131072])
def test_calibrate_bit_exact(n_tok):
    k = synth.gen_calibration_keys(8, 128, n_samples=1, sample_len=n_tok, seed_base=50)
    if n_tok == 7:
        k[:, 3, 5] = 0.0                                  # zero channel -> eps floor
    lam_ref, inv_ref = ref.calibrate_smooth(k)
    lam, inv = vi.calibrate_smooth(t_bf16(k))
    assert np.array_equal(lam.cpu().numpy().view(np.uint32), lam_ref.view(np.uint32))
    assert np.array_equal(inv.cpu().numpy().view(np.uint32), inv_ref.view(np.uint32))


def test_calibrate_strided_input():
    k = synth.gen_calibration_keys(4, 128, n_samples=1, sample_len=300, seed_base=60)
    big = torch.zeros(300, 6, 136, dtype=torch.bfloat16, device=DEV)
    big[:, 1:5, 4:132] = t_bf16(k)
    view = big[:, 1:5, 4:132]                               # non-16B-aligned strides -> scalar path
    lam, inv = vi.calibrate_smooth(view)
    lam_ref, _ = ref.calibrate_smooth(k)
    assert np.array_equal(lam.cpu().numpy(), lam_ref)


def test_calibrate_frozen_lambda_matches():
    """The frozen lambda (oracle, scripts/fit_codebooks.py) is reproduced bit-exactly on the GPU."""
    kcal = synth.gen_calibration_keys(8, 128)
    lam, inv = vi.calibrate_smooth(t_bf16(kcal))
    assert np.array_equal(lam.cpu().numpy(), CB["lambda"])
    assert np.array_equal(inv.cpu().numpy(), CB["inv_lambda"])


# ----------------------------------------------------------------- encode (Eq. 2, 8, 9)
def _encode_gpu(k, v, inv, ck, cv, n_cap, write_pos, kcfg, vcfg, err=None):
    B, T, H, D = k.shape
    kc = torch.zeros(B, H, n_cap, kcfg.row_bytes, dtype=torch.uint8, device=DEV)
    vc = torch.zeros(B, H, n_cap, vcfg.row_bytes, dtype=torch.uint8, device=DEV)
    vi.encode_kv(t_bf16(k), t_bf16(v), t_f32(inv), t_bf16(ck), t_bf16(cv), kc, vc, t_i32(write_pos), kcfg, vcfg,
                 err_flags=err)
    return kc.cpu().numpy(), vc.cpu().numpy()


def _encode_ref(k, v, inv, ck, cv, n_cap, write_pos, kcfg, vcfg):
    B, T, H, D = k.shape
    kc = np.zeros((B, H, n_cap, kcfg.row_bytes), np.uint8)
    vc = np.zeros((B, H, n_cap, vcfg.row_bytes), np.uint8)
    for h in range(H):
        ckh = ck[h] if ck.ndim == 3 else ck
        cvh = cv[h] if cv.ndim == 3 else cv
        kk, vv = ref.encode_kv(k[:, :, h], v[:, :, h], inv[h], ckh, cvh)
        for b in range(B):
            p = write_pos[b]
            kc[b, h, p:p + T] = ref.pack_codes(kk[b], kcfg.code_bits)
            vc[b, h, p:p + T] = ref.pack_codes(vv[b], vcfg.code_bits)
    return kc, vc


@pytest.mark.parametrize("name,cfg", [("b2d4", vi.B2D4), ("b1d4", vi.B1D4)])
@pytest.mark.parametrize("B,T", [(1, 1), (2, 37), (1, 300), (1, 600)])  # 600 x 8 heads > 4096: bulk kernel
def test_encode_bit_exact(name, cfg, B, T):
    k = synth.gen_keys(T, 8, 128, seed=100 + T, batch=B)
    v = synth.gen_values(T, 8, 128, seed=200 + T, batch=B)
    n_cap = T + 10
    wp = [3 + b for b in range(B)]
    ck, cv = CB[f"ck_{name}"], CB[f"cv_{name}"]
    got = _encode_gpu(k, v, CB["inv_lambda"], ck, cv, n_cap, wp, cfg, cfg)
    want = _encode_ref(k, v, CB["inv_lambda"], ck, cv, n_cap, wp, cfg, cfg)
    assert np.array_equal(got[0], want[0]), "key codes differ"
    assert np.array_equal(got[1], want[1]), "value codes differ"


def test_encode_b4d4_bit_exact_shared_codebook():
    T = 24
    k = synth.gen_keys(T, 2, 128, seed=300)
    v = synth.gen_values(T, 2, 128, seed=301)
    ck, cv = CB["ck_b4d4"], CB["cv_b4d4"]                  # one codebook for all heads (stride 0)
    got = _encode_gpu(k, v, CB["inv_lambda"][:2], ck, cv, T, [0], vi.B4D4, vi.B4D4)
    want = _encode_ref(k, v, CB["inv_lambda"][:2], ck, cv, T, [0], vi.B4D4, vi.B4D4)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_encode_mixed_bits_bit_exact():
    T = 20
    k = synth.gen_keys(T, 2, 128, seed=310)
    v = synth.gen_values(T, 2, 128, seed=311)
    got = _encode_gpu(k, v, CB["inv_lambda"][:2], CB["ck_b2d4"][:2], CB["cv_b1d4"][:2], T, [0], vi.B2D4, vi.B1D4)
    want = _encode_ref(k, v, CB["inv_lambda"][:2], CB["ck_b2d4"][:2], CB["cv_b1d4"][:2], T, [0], vi.B2D4, vi.B1D4)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("n_levels,cfg", [(2, vi.B1D4), (4, vi.B2D4), (16, vi.B4D4)])
def test_encode_product_grid_ties(n_levels, cfg):
    """Closed-form NN with genuine fp32 ties through the untransformed V path: lowest index wins
    (16 / 256 / 65536 entries)."""
    cb = synth.product_grid_codebook(n_levels, 4, step=0.5)
    T = 8 if n_levels == 16 else 64
    pts = synth.dyadic_points(T * 32, 4, n_levels, 0.5, seed=n_levels).reshape(1, T, 1, 128)
    lv = synth.grid_levels(n_levels, 0.5)
    digit = np.argmin(np.abs(pts.reshape(-1, 4)[:, :, None].astype(np.float64) - lv), axis=2)
    want = (digit * (n_levels ** np.arange(4))).sum(1).reshape(T, 32)
    k = np.zeros_like(pts)
    _, vc = _encode_gpu(k, pts, np.ones((1, 128), np.float32), cb, cb, T, [0], cfg, cfg)
    assert np.array_equal(ref.unpack_codes(vc[0, 0], cfg.code_bits), want)


def test_encode_flags_range_and_write_pos():
    k = np.zeros((1, 2, 1, 128), np.float32)
    k[0, 0, 0, 0] = 2.0 ** 40                                 # |k * inv_lambda| >= 2^32
    v = np.zeros_like(k)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    _encode_gpu(k, v, np.ones((1, 128), np.float32), CB["ck_b2d4"][:1], CB["cv_b2d4"][:1], 2, [0], vi.B2D4, vi.B2D4,
                err=err)
    assert int(err.item()) & 1
    err.zero_()
    _encode_gpu(np.zeros_like(k), v, np.ones((1, 128), np.float32), CB["ck_b2d4"][:1], CB["cv_b2d4"][:1], 2, [1],
                vi.B2D4, vi.B2D4, err=err)                    # row 1 + t=1 == n_cap -> flagged
    assert int(err.item()) & 2


# ------------------------------------------------------------------- attention (Eq. 10)
def _attn_case(B, Hkv, G, n_cap, seq_lens, seed, codes_from="random"):
    rng = np.random.default_rng(seed)
    heads = rng.choice(8, size=Hkv, replace=False) if Hkv < 8 else np.arange(8)
    lam = CB["lambda"][heads]
    ck, cv = CB["ck_b2d4"][heads], CB["cv_b2d4"][heads]
    if codes_from == "random":
        kc = synth.gen_codes(n_cap, Hkv, 32, 8, seed=seed, batch=B)
        vc = synth.gen_codes(n_cap, Hkv, 32, 8, seed=seed + 1, batch=B)
    else:   # codes of realistic synthetic keys, encoded by the ORACLE
        k = synth.gen_keys(n_cap, 8, 128, seed=seed, batch=B)[:, :, heads]
        v = synth.gen_values(n_cap, 8, 128, seed=seed + 1, batch=B)[:, :, heads]
        kc = np.zeros((B, Hkv, n_cap, 32), np.int64)
        vc = np.zeros_like(kc)
        for i in range(Hkv):
            kk, vv = ref.encode_kv(k[:, :, i], v[:, :, i], CB["inv_lambda"][heads[i]], ck[i], cv[i])
            kc[:, i], vc[:, i] = kk, vv
    q = synth.gen_queries(B, 8 * G, 8, 128, seed=seed + 2).reshape(B, 8, G, 128)[:, heads].reshape(B, Hkv * G, 128)
    return dict(q=q, lam=lam, ck=ck, cv=cv, kc=kc, vc=vc, seq_lens=np.asarray(seq_lens))


def _run_gpu(c, **kw):
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]),
                          t_u8(c["kc"]), t_u8(c["vc"]), t_i32(c["seq_lens"]), **kw)
    return o.float().cpu().numpy(), L.cpu().numpy()


def _run_ref(c, tok_begin=0, tok_end=None):
    return ref.attention_decode_batch(c["q"], c["lam"], c["ck"], c["cv"], c["kc"], c["vc"], c["seq_lens"],
                                      tok_begin, tok_end)


def _assert_close(o, L, o_ref, L_ref):
    err = row_rel_err(o, o_ref)
    assert err.max() <= TOL_O, f"max row rel err {err.max():.3e}"
    fin = np.isfinite(L_ref)
    assert np.array_equal(np.isfinite(L), fin)
    assert np.all(np.abs(L[fin] - L_ref[fin]) <= TOL_L), f"max |dL| {np.abs(L[fin] - L_ref[fin]).max():.3e}"
    assert np.all(o[~fin] == 0)


@pytest.mark.parametrize("algo", ["mma", "lut"])
def test_attn_cfg1_oracle_encoded(algo):
    """BASELINE configs[0]: 1 batch, 1 KV head (G = 4), seq 1024, b2d4, codes from the oracle encoder."""
    c = _attn_case(1, 1, 4, 1024, [1024], seed=0, codes_from="oracle")
    o, L = _run_gpu(c, algo=algo)
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("algo", ["mma", "lut"])
@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 31, 33, 100, 513, 2047, 4097])
def test_attn_ragged_lengths(algo, n):
    c = _attn_case(2, 2, 4, 4200, [n, max(1, n // 3)], seed=n)
    o, L = _run_gpu(c, algo=algo)
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("splits", [1, 2, 3, 7, 16, 18, 40])  # <= 16: DSMEM cluster merge; else global
def test_attn_fixed_splits_and_determinism(splits):
    c = _attn_case(1, 4, 4, 3000, [2999], seed=splits)
    o1, L1 = _run_gpu(c, num_splits=splits)
    o2, L2 = _run_gpu(c, num_splits=splits)
    assert np.array_equal(o1, o2) and np.array_equal(L1, L2)      # bitwise deterministic
    _assert_close(o1, L1, *_run_ref(c))


@pytest.mark.parametrize("G", [1, 2, 3, 4, 5, 6, 7, 8])   # > 4: two virtual KV heads per KV head
@pytest.mark.parametrize("splits", [0, 3])
def test_attn_gqa_groups(G, splits):
    c = _attn_case(2, 3, G, 700, [700, 450], seed=10 + G)
    o, L = _run_gpu(c, num_splits=splits)
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("G", [5, 8])
def test_decode_step_fused_gqa_over_4(G):
    """Qwen2.5-14B-like group (40 q / 8 kv = 5) and G = 8: both virtual heads of a KV head run the
    owner encode and write identical codes; codes bit-exact, output vs the oracle."""
    lens = [900, 333]
    B = len(lens)
    c = _attn_case(B, 8, G, max(lens) + 2, lens, seed=30 + G)
    kn = synth.gen_keys(1, 8, 128, seed=31, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=32, batch=B)[:, 0]
    wp = [n - 1 for n in lens]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens))
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]], c["vc"][b, h, wp[b]] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), c["kc"].astype(np.uint8))
    assert np.array_equal(vcodes.cpu().numpy(), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


@pytest.mark.parametrize("rng_", [(0, 500), (500, -1), (100, 101), (1000, 3000), (250, 250)])
def test_attn_token_ranges(rng_):
    """Sharding hook: tokens [tok_begin, min(tok_end, seq_len)); empty shard -> o = 0, L = -inf."""
    a, e = rng_
    c = _attn_case(2, 2, 4, 1200, [1200, 700], seed=21)
    o, L = _run_gpu(c, tok_begin=a, tok_end=e)
    _assert_close(o, L, *_run_ref(c, a, None if e < 0 else e))


def test_attn_empty_sequence():
    c = _attn_case(1, 2, 4, 64, [0], seed=22)
    o, L = _run_gpu(c)
    assert np.all(o == 0) and np.all(np.isneginf(L))


def test_attn_bf16_output_is_rounded_fp32():
    c = _attn_case(1, 2, 4, 900, [900], seed=23)
    of, Lf = _run_gpu(c, num_splits=3)
    ob, Lb = _run_gpu(c, num_splits=3, o_dtype=torch.bfloat16)
    assert np.array_equal(synth.round_to_bf16(of.astype(np.float32)), ob.astype(np.float32))
    assert np.array_equal(Lf, Lb)


def test_attn_identity_codebook_equals_full_precision():
    """If every transformed key sub-vector is a centroid, VQ attention = Eq. 1 attention on the
    ORIGINAL keys (Eq. 7 invariance); GPU vs the fp64 full-precision Eq. 1 oracle."""
    c = _attn_case(1, 1, 4, 512, [512], seed=24)
    H = ref.hadamard(128)
    K = ref.vq_decode(c["kc"][0, 0], c["ck"][0]) @ H.T * c["lam"][0][None].astype(np.float64)
    V = ref.vq_decode(c["vc"][0, 0], c["cv"][0])
    o_ref, L_ref = ref.attention_full(c["q"][0], K, V)
    o, L = _run_gpu(c)
    _assert_close(o[0], L[0], o_ref, L_ref)


def test_attn_single_token_and_identical_keys():
    c = _attn_case(1, 1, 4, 40, [1], seed=25)
    o, L = _run_gpu(c)
    assert np.max(row_rel_err(o[0], np.repeat(ref.vq_decode(c["vc"][0, 0, :1], c["cv"][0]), 4, 0))) <= TOL_O
    c["kc"][:] = c["kc"][:, :, :1]                                  # all keys identical
    c["seq_lens"] = np.array([40])
    o, L = _run_gpu(c)
    want = ref.vq_decode(c["vc"][0, 0, :40], c["cv"][0]).mean(0)
    assert np.max(row_rel_err(o[0], np.tile(want, (4, 1)))) <= TOL_O


# ----------------------------------------------------------------------- merge (LSE)
def test_merge_lse_vs_oracle():
    rng = np.random.default_rng(30)
    P, B, Hq = 5, 2, 32
    o = rng.standard_normal((P, B, Hq, 128)).astype(np.float32)
    L = (rng.standard_normal((P, B, Hq)) * 3).astype(np.float32)
    L[2, 0, :4] = -np.inf
    L[:, 1, 5] = -np.inf
    got_o, got_L = vi.merge_lse(t_f32(o), t_f32(L))
    want_o, want_L = ref.merge_lse(o, L)
    _assert_close(got_o.cpu().numpy(), got_L.cpu().numpy(), want_o, want_L)


def test_sharded_attention_plus_merge_equals_unsharded():
    """Single-GPU emulation of the sequence-sharded multi-GPU path: attn_decode on P contiguous
    token shards + merge_lse == oracle over the whole sequence."""
    c = _attn_case(1, 8, 4, 6000, [5990], seed=31)
    parts = [_run_gpu(c, tok_begin=a, tok_end=e) for a, e in ((0, 1500), (1500, 3000), (3000, 4500), (4500, 6000))]
    o_p = np.stack([p[0] for p in parts]).astype(np.float32)
    L_p = np.stack([p[1] for p in parts]).astype(np.float32)
    mo, mL = vi.merge_lse(t_f32(o_p), t_f32(L_p))
    _assert_close(mo.cpu().numpy(), mL.cpu().numpy(), *_run_ref(c))


# ------------------------------------------------------ BASELINE configs at full size
def _sampled_units_check(B, N, n_units, seed, units=None, **kw):
    """Full-size launch (auto splits, as bench.py) checked on sampled (b, h_kv) units, or on the
    explicit list `units` (every unit, deterministically, where the oracle is fast enough)."""
    rng = np.random.default_rng(seed)
    q = synth.gen_queries(B, 32, 8, 128, seed=seed)
    kc = synth.gen_codes_torch((B, 8, N, 32), 8, seed=seed, device=DEV)
    vc = synth.gen_codes_torch((B, 8, N, 32), 8, seed=seed + 1, device=DEV)
    o, L = vi.attn_decode(t_bf16(q), t_f32(CB["lambda"]), t_bf16(CB["ck_b2d4"]), t_bf16(CB["cv_b2d4"]), kc, vc,
                          t_i32([N] * B), **kw)
    o, L = o.cpu().numpy(), L.cpu().numpy()
    if units is None:
        units = [(int(rng.integers(B)), int(rng.integers(8))) for _ in range(n_units)]
    for b, h in units:
        kk = kc[b, h].cpu().numpy().astype(np.int64)   # synthetic inputs (synth/), not CUDA results
        vv = vc[b, h].cpu().numpy().astype(np.int64)
        o_ref, L_ref = ref.attention_vq(q[b, 4 * h:4 * h + 4], CB["lambda"][h], CB["ck_b2d4"][h], CB["cv_b2d4"][h],
                                        kk, vv)
        _assert_close(o[b, 4 * h:4 * h + 4], L[b, 4 * h:4 * h + 4], o_ref, L_ref)


def test_cfg2_full_size_all_units():
    """BASELINE configs[1] at full size (the bench's default launch): all 8 (b, h_kv) units, i.e.
    all 32 query heads, each checked against the oracle."""
    _sampled_units_check(1, 32768, 0, seed=40, units=[(0, h) for h in range(8)])


def test_cfg3_full_size_sampled_units():
    _sampled_units_check(64, 8192, 6, seed=41)


def test_cfg4_full_size_sampled_units():
    _sampled_units_check(1, 196608, 2, seed=42)


@pytest.mark.parametrize("B,N,kind", [(16, 32768, "stream"), (8, 32768, "stream"), (4, 32768, "split"),
                                      (2, 32768, "split")])
def test_mid_batch_auto_plan_sampled_units(B, N, kind):
    """B*H_kv < #SMs: AUTO picks the stream partition when the cost model says the split plan's
    waves waste more SMs (B = 8, 16 at 32k) and the split kernel otherwise; both checked on
    sampled units at the full shape."""
    assert vi.attn_kernel_kind(B, 8, N) == kind
    _sampled_units_check(B, N, 3, seed=43 + B)


# ------------------------------------------------- fused decode step (append + attention)
@pytest.mark.parametrize("splits", [0, 1, 3, 8, 18])
@pytest.mark.parametrize("lens", [[2048], [1500, 37], [33, 1]])
def test_decode_step_fused_equals_encode_then_attend(splits, lens):
    """vecinfer_decode_step == encode_kv(T=1) + attn_decode: the appended row's codes are the
    oracle's, bit for bit, and the output matches the oracle over the updated cache."""
    B = len(lens)
    n_cap = max(lens) + 5
    c = _attn_case(B, 8, 4, n_cap, lens, seed=60 + splits + len(lens))
    kn = synth.gen_keys(1, 8, 128, seed=70, batch=B)[:, 0]        # [B, H_kv, D]
    vn = synth.gen_values(1, 8, 128, seed=71, batch=B)[:, 0]
    wp = [n - 1 for n in lens]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens),
                          num_splits=splits, err_flags=err)
    assert int(err.item()) == 0
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]] = kk
            c["vc"][b, h, wp[b]] = vv
    assert np.array_equal(kcodes.cpu().numpy(), c["kc"].astype(np.uint8))
    assert np.array_equal(vcodes.cpu().numpy(), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


@pytest.mark.parametrize("B,N", [(1, 32768), (1, 196608), (64, 8192)])
def test_decode_step_fused_full_size_bench_config(B, N):
    """The bench's step at BASELINE configs[1] / [3] / [2] sizes: vecinfer_decode_step with the
    fused append at row N-1 (AUTO plan: split S = 18 with the owner's 512-token budget, or the
    stream partition at B = 64).  The appended codes equal the oracle's for every (b, h); the
    output of sampled units equals the oracle over the updated cache."""
    rng = np.random.default_rng(B + N)
    q = synth.gen_queries(B, 32, 8, 128, seed=91)
    kc = synth.gen_codes_torch((B, 8, N, 32), 8, seed=92, device=DEV)
    vc = synth.gen_codes_torch((B, 8, N, 32), 8, seed=93, device=DEV)
    kn = synth.gen_keys(1, 8, 128, seed=94, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=95, batch=B)[:, 0]
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    o, L = vi.decode_step(t_bf16(q), t_bf16(kn), t_bf16(vn), t_f32(CB["lambda"]), t_f32(CB["inv_lambda"]),
                          t_bf16(CB["ck_b2d4"]), t_bf16(CB["cv_b2d4"]), kc, vc, t_i32([N - 1] * B), t_i32([N] * B),
                          err_flags=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    o, L = o.cpu().numpy(), L.cpu().numpy()
    new_k = kc[:, :, N - 1].cpu().numpy()
    new_v = vc[:, :, N - 1].cpu().numpy()
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], CB["ck_b2d4"][h], CB["cv_b2d4"][h])
            assert np.array_equal(new_k[b, h], kk.astype(np.uint8)) and np.array_equal(new_v[b, h], vv.astype(np.uint8))
    for _ in range(3):
        b, h = int(rng.integers(B)), int(rng.integers(8))
        kk = kc[b, h].cpu().numpy().astype(np.int64)
        vv = vc[b, h].cpu().numpy().astype(np.int64)
        o_ref, L_ref = ref.attention_vq(q[b, 4 * h:4 * h + 4], CB["lambda"][h], CB["ck_b2d4"][h], CB["cv_b2d4"][h],
                                        kk, vv)
        _assert_close(o[b, 4 * h:4 * h + 4], L[b, 4 * h:4 * h + 4], o_ref, L_ref)


def test_decode_step_append_outside_attended_range():
    """write_pos beyond seq_len: the row is written (by split 0) but not attended."""
    c = _attn_case(1, 8, 4, 600, [500], seed=80)
    kn = synth.gen_keys(1, 8, 128, seed=81)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=82)[:, 0]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32([550]), t_i32([500]))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))      # old cache attended
    kk, _ = ref.encode_kv(kn[0, 3], vn[0, 3], CB["inv_lambda"][3], c["ck"][3], c["cv"][3])
    assert np.array_equal(kcodes[0, 3, 550].cpu().numpy(), kk.astype(np.uint8))


def test_decode_step_many_units_uses_separate_append():
    """320 units (>= #SMs): AUTO runs the stream kernel with the append fused; same result as the oracle."""
    B, n = 40, 64
    c = _attn_case(B, 8, 4, n + 2, [n] * B, seed=90)
    kn = synth.gen_keys(1, 8, 128, seed=91, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=92, batch=B)[:, 0]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32([n - 1] * B), t_i32([n] * B))
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, n - 1], c["vc"][b, h, n - 1] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), c["kc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


# ------------------------------------------- bit-width sweep (BASELINE configs[4]) + mixed K/V
CFGS = {4: vi.B1D4, 8: vi.B2D4, 16: vi.B4D4}
CBNAME = {4: "b1d4", 8: "b2d4", 16: "b4d4"}


def _bits_case(B, kb, vb, n_cap, lens, seed, G=4):
    """Random codes at the given widths; per-head codebooks (b1d4/b2d4) or the shared b4d4 one."""
    heads = np.arange(8)
    ck = CB[f"ck_{CBNAME[kb]}"]
    cv = CB[f"cv_{CBNAME[vb]}"]
    kc = synth.gen_codes(n_cap, 8, 32, kb, seed=seed, batch=B)
    vc = synth.gen_codes(n_cap, 8, 32, vb, seed=seed + 1, batch=B)
    q = synth.gen_queries(B, 8 * G, 8, 128, seed=seed + 2)
    return dict(q=q, lam=CB["lambda"][heads], ck=ck, cv=cv, kc=kc, vc=vc, seq_lens=np.asarray(lens), kb=kb, vb=vb)


def _run_gpu_bits(c, **kw):
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]),
                          t_u8(ref.pack_codes(c["kc"], c["kb"])), t_u8(ref.pack_codes(c["vc"], c["vb"])),
                          t_i32(c["seq_lens"]), kcfg=CFGS[c["kb"]], vcfg=CFGS[c["vb"]], **kw)
    return o.float().cpu().numpy(), L.cpu().numpy()


@pytest.mark.parametrize("kb,vb", [(4, 4), (16, 16), (8, 4), (4, 8), (16, 8), (8, 16), (4, 16), (16, 4)])
@pytest.mark.parametrize("splits", [0, 3])
def test_attn_bitwidths(kb, vb, splits):
    c = _bits_case(2, kb, vb, 800, [777, 100], seed=100 + kb + vb + splits)
    o, L = _run_gpu_bits(c, num_splits=splits)
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("kb,vb", [(4, 4), (8, 4), (4, 8), (16, 16), (16, 8), (8, 16), (16, 4)])
def test_decode_step_fused_bitwidths(kb, vb):
    """vecinfer_decode_step at every code width pair: 4/8-bit fuse the append into the attention
    launch, 16-bit (b4d4, 65 536-entry codebooks) run the centroid-split append launch first; the
    appended codes are the oracle's bit for bit and the output matches the oracle."""
    B, lens = 1, [1000]
    c = _bits_case(B, kb, vb, 1003, lens, seed=120 + kb * vb)
    kn = synth.gen_keys(1, 8, 128, seed=121, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=122, batch=B)[:, 0]
    kcodes = t_u8(ref.pack_codes(c["kc"], kb))
    vcodes = t_u8(ref.pack_codes(c["vc"], vb))
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32([999]), t_i32(lens),
                          kcfg=CFGS[kb], vcfg=CFGS[vb])
    for h in range(8):   # b4d4 books are shared by the heads ([65536, 4]), the others per head
        ckh = c["ck"] if c["ck"].ndim == 2 else c["ck"][h]
        cvh = c["cv"] if c["cv"].ndim == 2 else c["cv"][h]
        kk, vv = ref.encode_kv(kn[0, h], vn[0, h], CB["inv_lambda"][h], ckh, cvh)
        c["kc"][0, h, 999], c["vc"][0, h, 999] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), ref.pack_codes(c["kc"], kb))
    assert np.array_equal(vcodes.cpu().numpy(), ref.pack_codes(c["vc"], vb))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


def test_decode_step_b4d4_full_size_bench_config():
    """The bench's cfg5-b4d4 step at full size (B = 1, N = 65 536, 8 KV heads, shared 65 536-entry
    codebooks): vecinfer_decode_step appends row N-1 (16-bit search launch) and attends; the
    appended codes of all 8 heads are the oracle's bit for bit, and 3 heads' outputs match the oracle."""
    N, bits = 65536, 16
    kc = synth.gen_codes_torch((1, 8, N, 64), bits, seed=501, device=DEV)
    vc = synth.gen_codes_torch((1, 8, N, 64), bits, seed=502, device=DEV)
    q = synth.gen_queries(1, 32, 8, 128, seed=503)
    kn = synth.gen_keys(1, 8, 128, seed=504)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=505)[:, 0]
    ck, cv = CB["ck_b4d4"], CB["cv_b4d4"]
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    o, L = vi.decode_step(t_bf16(q), t_bf16(kn), t_bf16(vn), t_f32(CB["lambda"]), t_f32(CB["inv_lambda"]),
                          t_bf16(ck), t_bf16(cv), kc, vc, t_i32([N - 1]), t_i32([N]), kcfg=vi.B4D4, vcfg=vi.B4D4,
                          err_flags=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    o, L = o.cpu().numpy(), L.cpu().numpy()
    for h in range(8):
        kk, vv = ref.encode_kv(kn[0, h], vn[0, h], CB["inv_lambda"][h], ck, cv)
        assert np.array_equal(kc[0, h, N - 1].cpu().numpy(), ref.pack_codes(kk[None], bits)[0])
        assert np.array_equal(vc[0, h, N - 1].cpu().numpy(), ref.pack_codes(vv[None], bits)[0])
    for h in (0, 3, 7):
        kk = ref.unpack_codes(kc[0, h].cpu().numpy(), bits)
        vv = ref.unpack_codes(vc[0, h].cpu().numpy(), bits)
        o_ref, L_ref = ref.attention_vq(q[0, 4 * h:4 * h + 4], CB["lambda"][h], ck, cv, kk, vv)
        _assert_close(o[0, 4 * h:4 * h + 4], L[0, 4 * h:4 * h + 4], o_ref, L_ref)


@pytest.mark.parametrize("bits", [4, 16])
def test_cfg5_full_size_sampled_units(bits):
    """BASELINE configs[4] at full size (N = 65536, 8 KV heads) for b1d4 / b4d4, sampled units."""
    N = 65536
    rng = np.random.default_rng(bits)
    row = 32 * bits // 8
    kc = synth.gen_codes_torch((1, 8, N, row), bits, seed=bits, device=DEV)
    vc = synth.gen_codes_torch((1, 8, N, row), bits, seed=bits + 1, device=DEV)
    q = synth.gen_queries(1, 32, 8, 128, seed=bits + 2)
    ck, cv = CB[f"ck_{CBNAME[bits]}"], CB[f"cv_{CBNAME[bits]}"]
    o, L = vi.attn_decode(t_bf16(q), t_f32(CB["lambda"]), t_bf16(ck), t_bf16(cv), kc, vc, t_i32([N]),
                          kcfg=CFGS[bits], vcfg=CFGS[bits])
    o, L = o.cpu().numpy(), L.cpu().numpy()
    for h in rng.choice(8, size=2, replace=False):
        kk = ref.unpack_codes(kc[0, h].cpu().numpy(), bits)
        vv = ref.unpack_codes(vc[0, h].cpu().numpy(), bits)
        ckh = ck[h] if ck.ndim == 3 else ck
        cvh = cv[h] if cv.ndim == 3 else cv
        o_ref, L_ref = ref.attention_vq(q[0, 4 * h:4 * h + 4], CB["lambda"][h], ckh, cvh, kk, vv)
        _assert_close(o[0, 4 * h:4 * h + 4], L[0, 4 * h:4 * h + 4], o_ref, L_ref)


# ----------------------------------------------- residual window
def _res_case(B, n_q, r_lens, r_cap, seed):
    c = _attn_case(B, 8, 4, max(n_q) + 4, n_q, seed=seed)
    c["K_res"] = synth.gen_keys(r_cap, 8, 128, seed=seed + 7, batch=B).transpose(0, 2, 1, 3).copy()
    c["V_res"] = synth.gen_values(r_cap, 8, 128, seed=seed + 8, batch=B).transpose(0, 2, 1, 3).copy()
    c["res_lens"] = np.asarray(r_lens)
    return c


def _run_ref_res(c):
    return ref.attention_decode_batch(c["q"], c["lam"], c["ck"], c["cv"], c["kc"], c["vc"], c["seq_lens"],
                                      K_res=c["K_res"], V_res=c["V_res"], res_lens=c["res_lens"])


@pytest.mark.parametrize("splits", [0, 1, 3, 8, 18])
@pytest.mark.parametrize("n_q,r_lens", [([3000, 700], [128, 5]), ([0, 1000], [17, 0]), ([64, 64], [1, 256])])
def test_attn_residual_window(splits, n_q, r_lens):
    c = _res_case(2, n_q, r_lens, 256, seed=130 + splits)
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(c["kc"]),
                          t_u8(c["vc"]), t_i32(c["seq_lens"]), num_splits=splits, k_res=t_bf16(c["K_res"]),
                          v_res=t_bf16(c["V_res"]), res_lens=t_i32(c["res_lens"]))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref_res(c))


def test_decode_step_appends_to_residual():
    c = _res_case(2, [2000, 300], [40, 1], 128, seed=140)
    kn = synth.gen_keys(1, 8, 128, seed=141, batch=2)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=142, batch=2)[:, 0]
    kr, vr = t_bf16(c["K_res"]), t_bf16(c["V_res"])
    lens = np.array([41, 2])                       # the new token becomes row lens-1
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(c["kc"]), t_u8(c["vc"]), t_i32([0, 0]),
                          t_i32(c["seq_lens"]), k_res=kr, v_res=vr, res_lens=t_i32(lens), append_to_residual=True)
    for b in range(2):
        c["K_res"][b, :, lens[b] - 1] = kn[b]
        c["V_res"][b, :, lens[b] - 1] = vn[b]
    assert np.array_equal(kr.float().cpu().numpy(), c["K_res"]) and np.array_equal(vr.float().cpu().numpy(), c["V_res"])
    c["res_lens"] = lens
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref_res(c))


def test_vqkv_cache_protocol_replay():
    """Cache manager (residual R = 8; when an append brings the window to 16 rows,
    the oldest 8 are flushed before attending) over 40 decode steps vs the oracle replay: flushed
    tokens are the ORACLE's codes, the window is raw and never attended with more than 15 rows."""
    from paper_2510_06175_b200.cache import VQKVCache
    B, R, steps = 2, 8, 40
    cache = VQKVCache(B, 8, 256, t_f32(CB["lambda"]), t_f32(CB["inv_lambda"]), t_bf16(CB["ck_b2d4"]),
                      t_bf16(CB["cv_b2d4"]), residual=R)
    ks = synth.gen_keys(steps, 8, 128, seed=150, batch=B)          # [B, steps, H, D]
    vs = synth.gen_values(steps, 8, 128, seed=151, batch=B)
    qs = [synth.gen_queries(B, 32, 8, 128, seed=200 + i) for i in range(steps)]
    n_q = 0
    for i in range(steps):
        o, L = cache.step(t_bf16(qs[i]), t_bf16(ks[:, i]), t_bf16(vs[:, i]))
        n_tot = i + 1
        if n_tot - n_q == 2 * R:    # this append filled the window: the oldest R rows were flushed
            n_q += R
        kc = np.zeros((B, 8, max(n_q, 1), 32), np.int64)
        vc = np.zeros_like(kc)
        for b in range(B):
            for h in range(8):
                if n_q:
                    kk, vv = ref.encode_kv(ks[b, :n_q, h], vs[b, :n_q, h], CB["inv_lambda"][h], CB["ck_b2d4"][h],
                                           CB["cv_b2d4"][h])
                    kc[b, h, :n_q], vc[b, h, :n_q] = kk, vv
        o_ref, L_ref = ref.attention_decode_batch(
            qs[i], CB["lambda"], CB["ck_b2d4"], CB["cv_b2d4"], kc, vc, [n_q] * B,
            K_res=ks[:, n_q:n_tot].transpose(0, 2, 1, 3), V_res=vs[:, n_q:n_tot].transpose(0, 2, 1, 3),
            res_lens=[n_tot - n_q] * B)
        _assert_close(o.cpu().numpy(), L.cpu().numpy(), o_ref, L_ref)
    assert cache.n_q == n_q == 32 and cache.n_r == 8
    assert np.array_equal(cache.kc[:, :, :n_q].cpu().numpy(), kc.astype(np.uint8))
