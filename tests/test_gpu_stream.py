"""GPU parity of the stream-partition attention kernel (attn_stream.cu) vs the CPU oracle.

The stream kernel cuts the B*H_kv units into pieces so that every CTA gets the same number of
tokens (units crossing CTA boundaries are split and merged in fixed piece order).  AUTO selects it
for B*H_kv >= #SMs; algo="stream" forces it at any size, which is how these tests reach the
straddling / tiny-piece / persistent (num_splits * units > #SMs) cases at small, oracle-friendly
shapes.  Same bars as test_gpu_parity: codes bit-exact, outputs <= 2e-3 row-relative, |dL| <= 2e-3.
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
from test_gpu_parity import (CFGS, _assert_close, _attn_case, _bits_case, _res_case, _run_gpu,  # noqa: E402
                             _run_gpu_bits, _run_ref, _run_ref_res, t_bf16, t_f32, t_i32, t_u8)

CB = load_codebooks()


@pytest.mark.parametrize("lens", [[1, 17, 513], [4097, 0, 33], [16, 16, 16], [2500, 2400, 2300]])
def test_stream_ragged_lengths(lens):
    """24 units over #SMs CTAs: most units split into many (often empty) pieces."""
    c = _attn_case(len(lens), 8, 4, max(lens) + 3, lens, seed=300 + sum(lens) % 97)
    o, L = _run_gpu(c, algo="stream")
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("splits", [1, 2, 3, 7, 40])   # 40 x 24 units > #SMs: persistent, last-arriver merge
def test_stream_fixed_pieces_and_determinism(splits):
    c = _attn_case(3, 8, 4, 3000, [2999, 1000, 7], seed=310 + splits)
    o1, L1 = _run_gpu(c, algo="stream", num_splits=splits)
    o2, L2 = _run_gpu(c, algo="stream", num_splits=splits)
    assert np.array_equal(o1, o2) and np.array_equal(L1, L2)
    _assert_close(o1, L1, *_run_ref(c))


def test_stream_repeated_calls_reuse_workspace():
    """The published-element region is consumed (zeroed) by the merge: back-to-back calls on one
    workspace with different inputs must not see stale pieces."""
    ws = vi.attn_workspace(2, 32, 8, 1500)
    for seed in (320, 321, 322):
        c = _attn_case(2, 8, 4, 1500, [1500, 900 + seed % 3], seed=seed)
        o, L = _run_gpu(c, algo="stream", workspace=ws)
        _assert_close(o, L, *_run_ref(c))


def test_workspace_reuse_across_groups_batches_and_splits():
    """One serving-sized workspace reused by calls that change G (2, 5: groups with padding head
    slots), B and the split plan, through both kernels with the publish/consume merges.  Only the
    real heads are published, so no padding element is left behind for a later call to take as a
    fresh piece.  Every call matches the oracle, and every call repeated at the end of
    the sequence on the same (now well-used) workspace is bitwise identical to its first run."""
    ws = vi.attn_workspace(6, 64, 8, 3000, 40)
    cases = [(5, 1, 12, "mma"), (2, 3, 5, "mma"), (5, 3, 0, "stream"), (2, 1, 7, "stream"), (5, 2, 3, "stream"),
             (2, 6, 0, "mma"), (5, 6, 12, "mma"), (2, 2, 0, "stream"), (5, 4, 18, "mma"), (5, 1, 0, "mma"), (2, 1, 20, "mma")]
    first = []
    for i, (G, B, splits, algo) in enumerate(cases):
        lens = [2900 - 411 * b for b in range(B)]
        c = _attn_case(B, 8, G, 3000, lens, seed=360 + i)
        o, L = _run_gpu(c, algo=algo, num_splits=splits, workspace=ws)
        _assert_close(o, L, *_run_ref(c))
        first.append((c, o, L))
    for (G, B, splits, algo), (c, o1, L1) in zip(cases, first):
        o2, L2 = _run_gpu(c, algo=algo, num_splits=splits, workspace=ws)
        assert np.array_equal(o1, o2) and np.array_equal(L1, L2), (G, B, splits, algo)


def test_workspace_left_zero_by_every_merge_path():
    """The workspace layout depends on each call's (B, H_kv, S), so one buffer reused by calls of
    different shapes sees every word in several roles; the contract (vecinfer.h) is that every
    launch leaves the WHOLE workspace zero.  Checked after each call for every merge path: split
    kernel spin merge, multi-wave last-CTA merge (fp32 partials), stream kernel spin and
    last-arriver merges, and the 16-bit decode-step append (its centroid-split minima and arrival
    counters live in the same buffer), with G = 5 padding slots."""
    ws = vi.decode_step_workspace(6, 40, 8, 3000, kcfg=vi.B4D4, vcfg=vi.B4D4, num_splits=40)
    cases = [(5, 1, 12, "mma"), (5, 4, 18, "mma"), (2, 3, 0, "stream"), (5, 3, 40, "stream"), (4, 6, 40, "mma"),
             (4, 2, 7, "stream")]
    for i, (G, B, splits, algo) in enumerate(cases):
        lens = [2900 - 411 * b for b in range(B)]
        c = _attn_case(B, 8, G, 3000, lens, seed=380 + i)
        o, L = _run_gpu(c, algo=algo, num_splits=splits, workspace=ws)
        torch.cuda.synchronize()
        assert int(ws.count_nonzero()) == 0, (G, B, splits, algo)
        _assert_close(o, L, *_run_ref(c))
    # 16-bit decode step (separate centroid-split append launch + attention) on the same buffer
    B, N = 2, 1003
    c = _bits_case(B, 16, 16, N, [1000, 700], seed=390)
    kn = synth.gen_keys(1, 8, 128, seed=391, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=392, batch=B)[:, 0]
    kcodes = t_u8(ref.pack_codes(c["kc"], 16))
    vcodes = t_u8(ref.pack_codes(c["vc"], 16))
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32([999, 699]), t_i32([1000, 700]),
                          kcfg=vi.B4D4, vcfg=vi.B4D4, workspace=ws)
    torch.cuda.synchronize()
    assert int(ws.count_nonzero()) == 0, "16-bit decode step"
    for b, p in ((0, 999), (1, 699)):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"], c["cv"])
            c["kc"][b, h, p], c["vc"][b, h, p] = kk, vv
    c["seq_lens"] = np.array([1000, 700], dtype=np.int32)
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


def test_stream_auto_many_units():
    """B*H_kv = 160 >= #SMs: AUTO picks the stream kernel (one unit per CTA plus a few split)."""
    lens = [300 + 37 * b for b in range(20)]
    lens[3] = 0
    c = _attn_case(20, 8, 4, max(lens) + 1, lens, seed=330)
    o, L = _run_gpu(c)
    _assert_close(o, L, *_run_ref(c))


def test_stream_gqa_groups_over_4():
    """G = 5 / 8 through the stream kernel (two virtual heads per KV head share one table)."""
    for G in (5, 8):
        c = _attn_case(3, 8, G, 1500, [1500, 77, 900], seed=345 + G)
        o, L = _run_gpu(c, algo="stream")
        _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("rng_", [(0, 500), (500, -1), (100, 101), (250, 250)])
def test_stream_token_ranges(rng_):
    a, e = rng_
    c = _attn_case(2, 8, 4, 1200, [1200, 700], seed=340)
    o, L = _run_gpu(c, algo="stream", tok_begin=a, tok_end=e)
    _assert_close(o, L, *_run_ref(c, a, None if e < 0 else e))


def test_stream_bf16_output_is_rounded_fp32():
    c = _attn_case(2, 8, 4, 900, [900, 333], seed=350)
    of, Lf = _run_gpu(c, algo="stream")
    ob, Lb = _run_gpu(c, algo="stream", o_dtype=torch.bfloat16)
    assert np.array_equal(synth.round_to_bf16(of.astype(np.float32)), ob.astype(np.float32))
    assert np.array_equal(Lf, Lb)


@pytest.mark.parametrize("kb,vb", [(4, 4), (16, 16), (8, 4), (16, 8)])
def test_stream_bitwidths(kb, vb):
    c = _bits_case(2, kb, vb, 800, [777, 100], seed=360 + kb + vb)
    o, L = _run_gpu_bits(c, algo="stream")
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("splits", [0, 3])
@pytest.mark.parametrize("n_q,r_lens", [([3000, 700], [128, 5]), ([0, 1000], [17, 0])])
def test_stream_residual_window(splits, n_q, r_lens):
    c = _res_case(2, n_q, r_lens, 256, seed=370 + splits)
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(c["kc"]),
                          t_u8(c["vc"]), t_i32(c["seq_lens"]), num_splits=splits, algo="stream",
                          k_res=t_bf16(c["K_res"]), v_res=t_bf16(c["V_res"]), res_lens=t_i32(c["res_lens"]))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref_res(c))


@pytest.mark.parametrize("splits", [0, 2])
@pytest.mark.parametrize("lens", [[2048], [1500, 37, 900], [33, 1]])
def test_stream_decode_step_fused(splits, lens):
    """Fused append in the stream kernel: the owner piece (the one holding write_pos) encodes the new
    token; its codes are the oracle's bit for bit and the output matches the oracle."""
    B = len(lens)
    n_cap = max(lens) + 5
    c = _attn_case(B, 8, 4, n_cap, lens, seed=380 + splits + len(lens))
    kn = synth.gen_keys(1, 8, 128, seed=381, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=382, batch=B)[:, 0]
    wp = [n - 1 for n in lens]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens),
                          num_splits=splits, algo="stream", err_flags=err)
    assert int(err.item()) == 0
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]] = kk
            c["vc"][b, h, wp[b]] = vv
    assert np.array_equal(kcodes.cpu().numpy(), c["kc"].astype(np.uint8))
    assert np.array_equal(vcodes.cpu().numpy(), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


def test_stream_decode_step_append_outside_range():
    """write_pos beyond seq_len: piece 0 of the unit writes the row, nobody attends it."""
    c = _attn_case(1, 8, 4, 600, [500], seed=390)
    kn = synth.gen_keys(1, 8, 128, seed=391)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=392)[:, 0]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32([550]), t_i32([500]),
                          algo="stream")
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))
    for h in range(8):
        kk, vv = ref.encode_kv(kn[0, h], vn[0, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
        assert np.array_equal(kcodes[0, h, 550].cpu().numpy(), kk.astype(np.uint8))
        assert np.array_equal(vcodes[0, h, 550].cpu().numpy(), vv.astype(np.uint8))


def test_stream_decode_step_many_units_b64():
    """BASELINE configs[2]'s batch shape (B = 64, 512 units) at a short length: AUTO picks the stream
    kernel with the append fused; every unit's appended codes checked."""
    B, n = 64, 96
    c = _attn_case(B, 8, 4, n + 2, [n] * B, seed=395)
    kn = synth.gen_keys(1, 8, 128, seed=396, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=397, batch=B)[:, 0]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32([n - 1] * B), t_i32([n] * B))
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, n - 1], c["vc"][b, h, n - 1] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), c["kc"].astype(np.uint8))
    assert np.array_equal(vcodes.cpu().numpy(), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))
