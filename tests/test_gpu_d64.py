"""head_dim 64 (the paper's Fig. 10 variant): 16 sub-vectors of 4 dims per
head.  Encode must match the oracle bit for bit (its pinned transform is written for any D: 64-point
integer Hadamard, 1/sqrt(64) = 0.125), attention must match the oracle within the usual 2e-3.
D = 64 runs the split kernel, with the residual window and the fused decode append (no stream /
LUT variant).
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
D = 64
CFG64 = {4: vi.VQConfig(64, 4, 4), 8: vi.VQConfig(64, 4, 8), 16: vi.VQConfig(64, 4, 16)}
NAME = {4: "b1d4", 8: "b2d4", 16: "b4d4"}
LAM, INV = CB["lambda"][:, :D].copy(), CB["inv_lambda"][:, :D].copy()


def _case(B, G, n_cap, lens, seed, bits=8, Hkv=8):
    ck, cv = CB[f"ck_{NAME[bits]}"], CB[f"cv_{NAME[bits]}"]
    kc = synth.gen_codes(n_cap, Hkv, D // 4, bits, seed=seed, batch=B)
    vc = synth.gen_codes(n_cap, Hkv, D // 4, bits, seed=seed + 1, batch=B)
    q = synth.gen_queries(B, Hkv * G, Hkv, D, seed=seed + 2)
    return dict(q=q, lam=LAM[:Hkv], ck=ck if ck.ndim == 2 else ck[:Hkv], cv=cv if cv.ndim == 2 else cv[:Hkv],
                kc=kc, vc=vc, seq_lens=np.asarray(lens), bits=bits)


def _run(c, **kw):
    b = c["bits"]
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]),
                          t_u8(ref.pack_codes(c["kc"], b)), t_u8(ref.pack_codes(c["vc"], b)), t_i32(c["seq_lens"]),
                          kcfg=CFG64[b], vcfg=CFG64[b], **kw)
    return o.float().cpu().numpy(), L.cpu().numpy()


def _ref(c, tok_begin=0, tok_end=None):
    return ref.attention_decode_batch(c["q"], c["lam"], c["ck"], c["cv"], c["kc"], c["vc"], c["seq_lens"],
                                      tok_begin, tok_end)


@pytest.mark.parametrize("bits", [4, 8, 16])
@pytest.mark.parametrize("T", [1, 300])
def test_d64_encode_bit_exact(bits, T):
    B, H = 2, 8
    k = synth.gen_keys(T, H, D, seed=600 + T, batch=B)
    v = synth.gen_values(T, H, D, seed=601 + T, batch=B)
    ck, cv = CB[f"ck_{NAME[bits]}"], CB[f"cv_{NAME[bits]}"]
    cfg = CFG64[bits]
    n_cap = T + 3
    kcodes = torch.zeros(B, H, n_cap, cfg.row_bytes, dtype=torch.uint8, device="cuda")
    vcodes = torch.zeros_like(kcodes)
    wp = np.array([0, 3], np.int32)
    vi.encode_kv(t_bf16(k), t_bf16(v), t_f32(INV), t_bf16(ck), t_bf16(cv), kcodes, vcodes, t_i32(wp), cfg, cfg)
    for b in range(B):
        for h in range(H):
            ckh = ck if ck.ndim == 2 else ck[h]
            cvh = cv if cv.ndim == 2 else cv[h]
            kk, vv = ref.encode_kv(k[b, :, h], v[b, :, h], INV[h], ckh, cvh)
            got_k = ref.unpack_codes(kcodes[b, h, wp[b]:wp[b] + T].cpu().numpy(), bits)
            got_v = ref.unpack_codes(vcodes[b, h, wp[b]:wp[b] + T].cpu().numpy(), bits)
            assert np.array_equal(got_k, kk) and np.array_equal(got_v, vv), (b, h)


@pytest.mark.parametrize("splits", [0, 1, 3, 16, 40])
@pytest.mark.parametrize("lens", [[2000, 17], [1, 4097]])
def test_d64_attention(splits, lens):
    c = _case(len(lens), 4, max(lens) + 2, lens, seed=610 + splits)
    o, L = _run(c, num_splits=splits)
    _assert_close(o, L, *_ref(c))


@pytest.mark.parametrize("G,bits", [(1, 8), (2, 4), (8, 8), (5, 16)])
def test_d64_gqa_and_bitwidths(G, bits):
    c = _case(2, G, 900, [900, 450], seed=620 + G + bits, bits=bits)
    o, L = _run(c)
    _assert_close(o, L, *_ref(c))


def test_d64_token_range_and_bf16():
    c = _case(2, 4, 1200, [1200, 700], seed=630)
    o, L = _run(c, tok_begin=100, tok_end=1000)
    _assert_close(o, L, *_ref(c, 100, 1000))
    of, Lf = _run(c, num_splits=3)
    ob, Lb = _run(c, num_splits=3, o_dtype=torch.bfloat16)
    assert np.array_equal(synth.round_to_bf16(of.astype(np.float32)), ob.astype(np.float32))


@pytest.mark.parametrize("bits,lens", [(8, [700, 64]), (4, [3000, 901]), (8, [40000])])
def test_d64_decode_step(bits, lens):
    """D = 64 decode step with the append fused into the attention launch (the owner split encodes
    the new token on 16 lanes: 64-point integer FWHT, 16 sub-vectors); appended codes are the
    oracle's bit for bit, the output matches the oracle."""
    B = len(lens)
    c = _case(B, 4, max(lens) + 10, lens, seed=640 + bits, bits=bits)
    kn = synth.gen_keys(1, 8, D, seed=641, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, D, seed=642, batch=B)[:, 0]
    wp = [n - 1 for n in lens]
    kcodes, vcodes = t_u8(ref.pack_codes(c["kc"], bits)), t_u8(ref.pack_codes(c["vc"], bits))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(INV), t_bf16(c["ck"]),
                          t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens), kcfg=CFG64[bits], vcfg=CFG64[bits],
                          err_flags=err)
    assert int(err.item()) == 0
    assert vi.decode_step_launches(B, 8, max(lens) + 10, CFG64[bits], CFG64[bits]) == 1
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], INV[h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]], c["vc"][b, h, wp[b]] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), ref.pack_codes(c["kc"], bits))
    assert np.array_equal(vcodes.cpu().numpy(), ref.pack_codes(c["vc"], bits))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_ref(c))


@pytest.mark.parametrize("splits", [0, 1, 3, 18])
@pytest.mark.parametrize("n_q,r_lens", [([3000, 700], [128, 5]), ([0, 1000], [17, 0])])
def test_d64_residual_window(splits, n_q, r_lens):
    """Full-precision residual window at D = 64 (raw bf16 rows of 64 elements)."""
    B = len(n_q)
    c = _case(B, 4, max(n_q) + 4, n_q, seed=660 + splits)
    K_res = synth.gen_keys(256, 8, D, seed=661, batch=B).transpose(0, 2, 1, 3).copy()
    V_res = synth.gen_values(256, 8, D, seed=662, batch=B).transpose(0, 2, 1, 3).copy()
    rl = np.asarray(r_lens)
    o, L = _run(c, num_splits=splits, k_res=t_bf16(K_res), v_res=t_bf16(V_res), res_lens=t_i32(rl))
    _assert_close(o, L, *ref.attention_decode_batch(c["q"], c["lam"], c["ck"], c["cv"], c["kc"], c["vc"],
                                                    c["seq_lens"], K_res=K_res, V_res=V_res, res_lens=rl))


def test_d64_decode_step_appends_to_residual():
    c = _case(2, 4, 2004, [2000, 300], seed=670)
    K_res = synth.gen_keys(128, 8, D, seed=671, batch=2).transpose(0, 2, 1, 3).copy()
    V_res = synth.gen_values(128, 8, D, seed=672, batch=2).transpose(0, 2, 1, 3).copy()
    kn = synth.gen_keys(1, 8, D, seed=673, batch=2)[:, 0]
    vn = synth.gen_values(1, 8, D, seed=674, batch=2)[:, 0]
    kr, vr = t_bf16(K_res), t_bf16(V_res)
    lens = np.array([41, 2])                       # the new token becomes row lens-1
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(INV), t_bf16(c["ck"]),
                          t_bf16(c["cv"]), t_u8(ref.pack_codes(c["kc"], 8)), t_u8(ref.pack_codes(c["vc"], 8)),
                          t_i32([0, 0]), t_i32(c["seq_lens"]), kcfg=CFG64[8], vcfg=CFG64[8], k_res=kr, v_res=vr,
                          res_lens=t_i32(lens), append_to_residual=True)
    for b in range(2):
        K_res[b, :, lens[b] - 1] = kn[b]
        V_res[b, :, lens[b] - 1] = vn[b]
    assert np.array_equal(kr.float().cpu().numpy(), K_res) and np.array_equal(vr.float().cpu().numpy(), V_res)
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *ref.attention_decode_batch(
        c["q"], c["lam"], c["ck"], c["cv"], c["kc"], c["vc"], c["seq_lens"], K_res=K_res, V_res=V_res,
        res_lens=lens))


@pytest.mark.parametrize("lens,splits", [([1, 17, 513], 0), ([4097, 0, 33], 0), ([2500, 2400, 2300], 3),
                                         ([3000, 1000, 7], 40)])   # 40 x 24 units > #SMs: persistent
def test_d64_stream_kernel(lens, splits):
    """D = 64 through the stream partition (pieces cut at 16-token boundaries, straddling warps,
    spin and last-arriver merges), bitwise reproducible, vs the oracle."""
    c = _case(len(lens), 4, max(lens) + 3, lens, seed=690 + splits + len(lens))
    o1, L1 = _run(c, algo="stream", num_splits=splits)
    o2, L2 = _run(c, algo="stream", num_splits=splits)
    assert np.array_equal(o1, o2) and np.array_equal(L1, L2)
    _assert_close(o1, L1, *_ref(c))


@pytest.mark.parametrize("G,bits", [(4, 8), (5, 8), (8, 4), (4, 16)])
def test_d64_stream_auto_batch_decode(G, bits):
    """B*H_kv >= #SMs: AUTO picks the stream kernel at D = 64 too (GQA 5 / 8: two virtual heads)."""
    B = 20
    lens = [300 + 37 * b for b in range(B)]
    c = _case(B, G, max(lens) + 1, lens, seed=700 + G + bits, bits=bits)
    assert vi.attn_kernel_kind(B, 8 * (2 if G > 4 else 1), max(lens) + 1) == "stream"
    o, L = _run(c)
    _assert_close(o, L, *_ref(c))


def test_d64_unsupported_paths_fail_loudly():
    c = _case(1, 4, 256, [256], seed=650)
    kr = torch.zeros(1, 8, 16, D, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(VecInferError):   # the D = 64 stream kernel has no residual window
        _run(c, algo="stream", k_res=kr, v_res=kr, res_lens=t_i32([4]))
    with pytest.raises(VecInferError):
        _run(c, algo="lut")
    with pytest.raises(VecInferError):   # K and V head dims must agree
        vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]),
                       t_u8(ref.pack_codes(c["kc"], 8)), t_u8(ref.pack_codes(c["vc"], 8)), t_i32(c["seq_lens"]),
                       kcfg=CFG64[8], vcfg=vi.B2D4)
