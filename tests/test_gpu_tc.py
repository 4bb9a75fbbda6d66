"""GPU parity of the tcgen05 score path (VECINFER_ATTN_DEQUANT_TC, attn_mma.cu TC=true) vs the oracle.

The split kernel with the score contraction s = q~ K^T (Alg. 1 l.11, Eq. 10) on the 5th-generation
tensor cores: 4-warp groups stage their gathered K^ tile in tensor memory, one thread issues
tcgen05.mma, the scores return through tcgen05.ld.  Same bars as test_gpu_parity: outputs <= 2e-3
row-relative, |dL| <= 2e-3, appended codes bit-exact.  Ragged tails, dummy group iterations
(warps of a group without a tile), multi-wave persistent grids, every split count, GQA groups,
residual windows and the fused decode append are covered.
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


@pytest.mark.parametrize("n", [1, 15, 31, 32, 33, 127, 128, 129, 511, 513, 2047, 4097])
@pytest.mark.parametrize("splits", [1, 3, 0])
def test_tc_ragged_lengths(n, splits):
    c = _attn_case(1, 8, 4, n + 5, [n], seed=700 + n % 97 + splits)
    o, L = _run_gpu(c, algo="tc", num_splits=splits)
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("splits", [2, 7, 18, 40])   # 40 x 24 units > #SMs: persistent multi-wave grid
def test_tc_splits_and_determinism(splits):
    c = _attn_case(3, 8, 4, 3000, [2999, 1000, 7], seed=710 + splits)
    o1, L1 = _run_gpu(c, algo="tc", num_splits=splits)
    o2, L2 = _run_gpu(c, algo="tc", num_splits=splits)
    assert np.array_equal(o1, o2) and np.array_equal(L1, L2)
    _assert_close(o1, L1, *_run_ref(c))


@pytest.mark.parametrize("G", [1, 2, 3, 4, 5, 8])
def test_tc_gqa_groups(G):
    c = _attn_case(2, 3, G, 900, [900, 450], seed=720 + G)
    o, L = _run_gpu(c, algo="tc")
    _assert_close(o, L, *_run_ref(c))


@pytest.mark.parametrize("kb,vb", [(4, 4), (4, 8), (8, 4), (8, 16), (4, 16)])
def test_tc_bitwidths(kb, vb):
    c = _bits_case(2, kb, vb, 800, [777, 100], seed=730 + kb + vb)
    o, L = _run_gpu_bits(c, algo="tc")
    _assert_close(o, L, *_run_ref(c))


def test_tc_cfg2_full_size_all_heads():
    """configs[1] shape (B = 1, N = 32768, 8 KV heads) through the TC kernel; every head vs the oracle."""
    N = 32768
    c = _attn_case(1, 8, 4, N, [N], seed=740)
    o, L = _run_gpu(c, algo="tc")
    _assert_close(o, L, *_run_ref(c))


def test_tc_matches_mma_path():
    """Both score paths on the same inputs agree far inside the tolerance (the scores differ only by
    the fp32 accumulation order of the 128-dim dot products)."""
    c = _attn_case(2, 8, 4, 5000, [5000, 2222], seed=750)
    o1, L1 = _run_gpu(c, algo="tc")
    o2, L2 = _run_gpu(c, algo="mma")
    assert np.abs(o1 - o2).max() <= 1e-4 * np.abs(o2).max() and np.abs(L1 - L2).max() <= 1e-4


@pytest.mark.parametrize("splits", [0, 3])
def test_tc_residual_window(splits):
    c = _res_case(2, [3000, 700], [128, 5], 256, seed=760 + splits)
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(c["kc"]),
                          t_u8(c["vc"]), t_i32(c["seq_lens"]), num_splits=splits, algo="tc",
                          k_res=t_bf16(c["K_res"]), v_res=t_bf16(c["V_res"]), res_lens=t_i32(c["res_lens"]))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref_res(c))


@pytest.mark.parametrize("wp_off", [1, 17, 40])   # appended row in the first, middle and a late tile
def test_tc_decode_step_fused_append(wp_off):
    lens = [2000, 777]
    B = len(lens)
    c = _attn_case(B, 8, 4, max(lens) + 2, lens, seed=770 + wp_off)
    kn = synth.gen_keys(1, 8, 128, seed=771, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=772, batch=B)[:, 0]
    wp = [n - wp_off for n in lens]
    kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens), algo="tc")
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]], c["vc"][b, h, wp[b]] = kk, vv
    assert np.array_equal(kcodes.cpu().numpy(), c["kc"].astype(np.uint8))
    assert np.array_equal(vcodes.cpu().numpy(), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


def test_tc_rejects_unsupported():
    c = _bits_case(1, 16, 8, 64, [64], seed=780)     # 16-bit K codebook: not in the shared table
    with pytest.raises(RuntimeError):
        _run_gpu_bits(c, algo="tc")
