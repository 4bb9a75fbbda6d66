"""The paper's other VQ configurations:
d8b8 (1-bit), d8b12 (1.5-bit), d4b10 (2.5-bit), d2b8 (4-bit) and the mixed K/V pairs of Table 3,
K-d4b10 / V-d8b12 (2-bit) and K-d8b12 / V-d8b8 (1.25-bit).

Codes are rows of one little-endian bit string (reading R11).  Encode must write exactly the
oracle's packed bytes (pinned transform + pinned distance, lowest index on ties); attention must
match the oracle within the usual 2e-3 bars, on the split kernel, for ragged lengths, split counts,
GQA groups, token ranges, paged pools and the residual window.
"""
import numpy as np
import pytest

import synth
from oracle import ref
from helpers import load_codebooks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402
from paper_2510_06175_b200._lib import VecInferError  # noqa: E402
from test_gpu_parity import _assert_close, t_bf16, t_f32, t_i32, t_u8  # noqa: E402

CB = load_codebooks()
FMT = {"d8b8": vi.D8B8, "d8b12": vi.D8B12, "d4b10": vi.D4B10, "d2b8": vi.D2B8, "d8b16": vi.D8B16}
PAIRS = [("d8b8", "d8b8"), ("d8b12", "d8b12"), ("d4b10", "d4b10"), ("d2b8", "d2b8"), ("d4b10", "d8b12"),
         ("d8b12", "d8b8"), ("d8b16", "d8b16")]


def _books(name, heads):
    ck, cv = CB[f"ck_{name}"], CB[f"cv_{name}"]
    if ck.ndim == 3:
        ck, cv = ck[heads], cv[heads]
    return ck, cv


def _case(kn, vn, B, Hkv, G, n_cap, lens, seed):
    heads = np.arange(Hkv)
    kcfg, vcfg = FMT[kn], FMT[vn]
    ck, _ = _books(kn, heads)
    _, cv = _books(vn, heads)
    kc = synth.gen_codes(n_cap, Hkv, kcfg.n_sub, kcfg.code_bits, seed=seed, batch=B)
    vc = synth.gen_codes(n_cap, Hkv, vcfg.n_sub, vcfg.code_bits, seed=seed + 1, batch=B)
    q = synth.gen_queries(B, Hkv * G, Hkv, 128, seed=seed + 2)
    return dict(q=q, lam=CB["lambda"][heads], ck=ck, cv=cv, kc=kc, vc=vc, seq_lens=np.asarray(lens), kcfg=kcfg,
                vcfg=vcfg)


def _run(c, kp=None, vp=None, **kw):
    kp = t_u8(ref.pack_codes(c["kc"], c["kcfg"].code_bits)) if kp is None else kp
    vp = t_u8(ref.pack_codes(c["vc"], c["vcfg"].code_bits)) if vp is None else vp
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), kp, vp,
                          t_i32(c["seq_lens"]), kcfg=c["kcfg"], vcfg=c["vcfg"], **kw)
    return o.float().cpu().numpy(), L.cpu().numpy()


def _ref(c, tok_begin=0, tok_end=None, **kw):
    return ref.attention_decode_batch(c["q"], c["lam"], c["ck"], c["cv"], c["kc"], c["vc"], c["seq_lens"],
                                      tok_begin, tok_end, **kw)


@pytest.mark.parametrize("name,T", [(n, t) for n in FMT for t in ((1, 300) if n != "d8b16" else (1, 12))])
def test_next2_encode_bit_exact(name, T):
    """Prefill (T = 300) and the 1-token append at ragged write positions: packed K and V rows
    equal the oracle's pack_codes(encode_kv(...)) byte for byte; untouched rows stay zero."""
    B, H = 2, 8
    cfg = FMT[name]
    k = synth.gen_keys(T, H, 128, seed=800 + T, batch=B)
    v = synth.gen_values(T, H, 128, seed=801 + T, batch=B)
    ck, cv = _books(name, np.arange(H))
    inv = CB["inv_lambda"]
    n_cap = T + 5
    kcodes = torch.zeros(B, H, n_cap, cfg.row_bytes, dtype=torch.uint8, device="cuda")
    vcodes = torch.zeros_like(kcodes)
    wp = np.array([0, 5], np.int32)
    cks = 0 if ck.ndim == 2 else None
    vi.encode_kv(t_bf16(k), t_bf16(v), t_f32(inv), t_bf16(ck), t_bf16(cv), kcodes, vcodes, t_i32(wp), cfg, cfg)
    want_k = np.zeros((B, H, n_cap, cfg.row_bytes), np.uint8)
    want_v = np.zeros_like(want_k)
    for b in range(B):
        for h in range(H):
            ckh = ck if ck.ndim == 2 else ck[h]
            cvh = cv if cv.ndim == 2 else cv[h]
            kk, vv = ref.encode_kv(k[b, :, h], v[b, :, h], inv[h], ckh, cvh)
            want_k[b, h, wp[b]:wp[b] + T] = ref.pack_codes(kk, cfg.code_bits)
            want_v[b, h, wp[b]:wp[b] + T] = ref.pack_codes(vv, cfg.code_bits)
    assert cks in (0, None)
    assert np.array_equal(kcodes.cpu().numpy(), want_k)
    assert np.array_equal(vcodes.cpu().numpy(), want_v)


@pytest.mark.parametrize("kn,vn", PAIRS)
@pytest.mark.parametrize("splits", [0, 1, 5])
def test_next2_attention(kn, vn, splits):
    c = _case(kn, vn, 2, 8, 4, 1500, [1500, 333], seed=810 + splits)
    o, L = _run(c, num_splits=splits)
    _assert_close(o, L, *_ref(c))


@pytest.mark.parametrize("kn,vn", [("d8b12", "d8b8"), ("d2b8", "d2b8")])
@pytest.mark.parametrize("G", [1, 7])
def test_next2_gqa_ranges_and_empty(kn, vn, G):
    """GQA groups 1 and 7 (two virtual heads), a token range, an empty sequence and a ragged
    one-token sequence."""
    c = _case(kn, vn, 3, 2, G, 700, [700, 0, 1], seed=820 + G)
    o, L = _run(c)
    _assert_close(o, L, *_ref(c))
    o, L = _run(c, tok_begin=64, tok_end=650, num_splits=3)
    _assert_close(o, L, *_ref(c, 64, 650))


def test_next2_paged_equals_contiguous():
    c = _case("d4b10", "d8b12", 2, 8, 4, 1024, [1024, 500], seed=830)
    kp = ref.pack_codes(c["kc"], 10).astype(np.uint8)
    vp = ref.pack_codes(c["vc"], 12).astype(np.uint8)
    ps, npb = 64, 1024 // 64
    perm = np.random.default_rng(831).permutation(2 * npb + 1)[:2 * npb].reshape(2, npb)
    kpool = np.zeros((2 * npb + 1, 8, ps, kp.shape[-1]), np.uint8)
    vpool = np.zeros((2 * npb + 1, 8, ps, vp.shape[-1]), np.uint8)
    for b in range(2):
        for i in range(npb):
            kpool[perm[b, i]] = kp[b, :, i * ps:(i + 1) * ps]
            vpool[perm[b, i]] = vp[b, :, i * ps:(i + 1) * ps]
    o_c, L_c = _run(c)
    o_p, L_p = _run(c, kp=t_u8(kpool), vp=t_u8(vpool), block_table=t_i32(perm.astype(np.int32)))
    assert np.array_equal(o_p, o_c) and np.array_equal(L_p, L_c)
    _assert_close(o_p, L_p, *_ref(c))


def test_next2_residual_window():
    c = _case("d8b12", "d8b12", 2, 8, 4, 900, [900, 40], seed=840)
    K_res = synth.gen_keys(64, 8, 128, seed=841, batch=2).transpose(0, 2, 1, 3).copy()
    V_res = synth.gen_values(64, 8, 128, seed=842, batch=2).transpose(0, 2, 1, 3).copy()
    r_lens = np.array([64, 9])
    o, L = _run(c, k_res=t_bf16(K_res), v_res=t_bf16(V_res), res_lens=t_i32(r_lens))
    _assert_close(o, L, *_ref(c, K_res=K_res, V_res=V_res, res_lens=r_lens))


@pytest.mark.parametrize("kn,vn,wp_off", [("d4b10", "d8b12", 1), ("d2b8", "d2b8", 1), ("d8b16", "d8b16", 1),
                                           ("d8b8", "d8b8", 1), ("d4b10", "d4b10", 1), ("d8b8", "d8b8", 40),
                                           ("d2b8", "d2b8", 33)])
def test_next2_decode_step(kn, vn, wp_off):
    """decode_step: books resident in the kernel's shared tables (d8b8, d2b8, d4b10, d8b12) append
    inside the attention launch (the owner split's 16-warp scan), d8b16 with the separate filter
    encode; the
    appended rows are the oracle's bit for bit, in the first or a middle tile of the owner split."""
    B, H = 2, 8
    lens = [600, 77]
    c = _case(kn, vn, B, H, 4, 610, lens, seed=850)
    kcfg, vcfg = c["kcfg"], c["vcfg"]
    kn_ = synth.gen_keys(1, H, 128, seed=851, batch=B)[:, 0]
    vn_ = synth.gen_values(1, H, 128, seed=852, batch=B)[:, 0]
    wp = [max(n - wp_off, 0) for n in lens]
    kcodes = t_u8(ref.pack_codes(c["kc"], kcfg.code_bits))
    vcodes = t_u8(ref.pack_codes(c["vc"], vcfg.code_bits))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn_), t_bf16(vn_), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens), kcfg=kcfg,
                          vcfg=vcfg, err_flags=err)
    assert int(err.item()) == 0
    fused = kn != "d8b16" and vn != "d8b16"
    # separate append: d8b12 / d8b16 streams through the tensor-core filter + exact selection (2
    # launches), any other stream through one generic launch, then the attention launch
    filt = [n in ("d8b12", "d8b16") for n in (kn, vn)]
    assert vi.decode_step_launches(B, H, 610, kcfg, vcfg) == (
        1 if fused else 1 + (2 if any(filt) else 0) + (0 if all(filt) else 1))
    for b in range(B):
        for h in range(H):
            ckh = c["ck"] if c["ck"].ndim == 2 else c["ck"][h]
            cvh = c["cv"] if c["cv"].ndim == 2 else c["cv"][h]
            kk, vv = ref.encode_kv(kn_[b, h], vn_[b, h], CB["inv_lambda"][h], ckh, cvh)
            c["kc"][b, h, wp[b]], c["vc"][b, h, wp[b]] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), ref.pack_codes(c["kc"], kcfg.code_bits))
    assert np.array_equal(vcodes.cpu().numpy(), ref.pack_codes(c["vc"], vcfg.code_bits))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_ref(c))


def test_next2_unsupported_fail_loudly():
    c = _case("d8b12", "d8b12", 1, 8, 4, 256, [256], seed=860)
    for algo in ("stream", "lut"):
        with pytest.raises(VecInferError):
            _run(c, algo=algo)
    c2 = _case("d8b8", "d8b12", 1, 8, 4, 256, [256], seed=861)   # no kernel for this pair
    with pytest.raises(VecInferError):
        _run(c2)


@pytest.mark.parametrize("kn,vn", [("d8b8", "d8b8"), ("d8b12", "d8b12"), ("d4b10", "d4b10"), ("d2b8", "d2b8"),
                                   ("d4b10", "d8b12"), ("d8b12", "d8b8")])
def test_next2_fused_append_many_steps(kn, vn):
    """48 consecutive fused decode steps (one launch each: the owner split's shared-table scan)
    append 48 x 8 token-heads; the cache afterwards equals vecinfer_encode_kv of the same tokens
    (the separate encoders) and the oracle's packed rows, byte for byte."""
    B, H, n_cap, T = 1, 8, 4096, 48
    kcfg, vcfg = FMT[kn], FMT[vn]
    assert vi.decode_step_launches(B, H, n_cap, kcfg, vcfg) == 1
    c = _case(kn, vn, B, H, 4, n_cap, [n_cap], seed=870)
    K = synth.gen_keys(T, H, 128, seed=871, batch=B)     # [B, T, H, D]
    V = synth.gen_values(T, H, 128, seed=872, batch=B)
    kcodes = t_u8(ref.pack_codes(c["kc"], kcfg.code_bits))
    vcodes = t_u8(ref.pack_codes(c["vc"], vcfg.code_bits))
    kref, vref = kcodes.clone(), vcodes.clone()
    q, lam, inv = t_bf16(c["q"]), t_f32(c["lam"]), t_f32(CB["inv_lambda"])
    ck, cv = t_bf16(c["ck"]), t_bf16(c["cv"])
    ws = vi.decode_step_workspace(B, 4 * H, H, n_cap, kcfg, vcfg)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    p0 = n_cap - T
    for t in range(T):
        vi.decode_step(q, t_bf16(K[:, t]), t_bf16(V[:, t]), lam, inv, ck, cv, kcodes, vcodes, t_i32([p0 + t]),
                       t_i32([p0 + t + 1]), kcfg=kcfg, vcfg=vcfg, workspace=ws, err_flags=err)
    vi.encode_kv(t_bf16(K), t_bf16(V), inv, ck, cv, kref, vref, t_i32([p0]), kcfg, vcfg)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert torch.equal(kcodes, kref) and torch.equal(vcodes, vref)
    for t in range(T):
        for h in range(H):
            ckh = c["ck"] if c["ck"].ndim == 2 else c["ck"][h]
            cvh = c["cv"] if c["cv"].ndim == 2 else c["cv"][h]
            c["kc"][0, h, p0 + t], c["vc"][0, h, p0 + t] = ref.encode_kv(K[0, t, h], V[0, t, h],
                                                                         CB["inv_lambda"][h], ckh, cvh)
    assert np.array_equal(kcodes.cpu().numpy(), ref.pack_codes(c["kc"], kcfg.code_bits))
    assert np.array_equal(vcodes.cpu().numpy(), ref.pack_codes(c["vc"], vcfg.code_bits))
