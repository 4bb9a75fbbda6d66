"""Seeded random-configuration sweep of vecinfer_attn_decode against the CPU oracle.

Each case draws a combination the targeted tests cover only one axis at a time: batch, KV heads,
GQA group (1..8), head dim (64/128), K/V code widths (every 4th case a NEXT-2 format pair), ragged lengths (incl. 0), token ranges,
fixed or automatic splits, algorithm (auto / split / stream), paged or contiguous codes and a
residual window, then checks the output against attention_decode_batch (same 2e-3 bars).
"""
import os

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
from test_gpu_parity import _assert_close, t_bf16, t_f32, t_i32, t_u8  # noqa: E402

CB = load_codebooks()
NAME = {4: "b1d4", 8: "b2d4", 16: "b4d4"}
# NEXT-2 pairs (D = 128, split kernel): name -> (sub_dim, code_bits)
N2 = {"d8b8": (8, 8), "d8b12": (8, 12), "d4b10": (4, 10), "d2b8": (2, 8)}
N2_PAIRS = [("d8b8", "d8b8"), ("d8b12", "d8b12"), ("d4b10", "d4b10"), ("d2b8", "d2b8"), ("d4b10", "d8b12"),
            ("d8b12", "d8b8")]


def _paginate(codes, ps, rng):
    B, H, n_cap, row = codes.shape
    npb = n_cap // ps
    n_pages = B * npb + 1
    perm = rng.permutation(n_pages)[:B * npb].reshape(B, npb)
    pool = np.zeros((n_pages, H, ps, row), codes.dtype)
    for b in range(B):
        for i in range(npb):
            pool[perm[b, i]] = codes[b, :, i * ps:(i + 1) * ps]
    return pool, perm.astype(np.int32)


_FUZZ_BASE = int(os.environ.get("VECINFER_FUZZ_BASE", "700"))      # wider sweeps: set both variables
_FUZZ_CASES = int(os.environ.get("VECINFER_FUZZ_CASES", "64"))


@pytest.mark.parametrize("case", range(_FUZZ_CASES))
def test_random_configuration(case):
    rng = np.random.default_rng(_FUZZ_BASE + case)
    D = int(rng.choice([128, 128, 64]))
    B = int(rng.integers(1, 4))
    Hkv = int(rng.choice([1, 2, 8]))
    G = int(rng.integers(1, 9))
    kb, vb = int(rng.choice([4, 8, 8, 16])), int(rng.choice([4, 8, 8, 16]))
    paged = bool(rng.integers(0, 2))
    ps = 64
    n_cap = int(rng.integers(2, 40)) * 64
    lens = [int(rng.integers(0, n_cap + 1)) for _ in range(B)]
    algo = "auto"
    if D == 128 and not paged:
        algo = str(rng.choice(["auto", "mma", "stream"]))
    splits = int(rng.choice([0, 0, 1, 3, 7]))
    tok_begin = 32 * int(rng.integers(0, 4)) if rng.integers(0, 3) == 0 else 0
    tok_end = int(rng.integers(tok_begin, n_cap + 1)) if rng.integers(0, 3) == 0 else -1
    use_res = D == 128 and rng.integers(0, 3) == 0
    if case % 4 == 3:
        use_res = bool(rng.integers(0, 3) == 0)

    kname, vname = NAME[kb], NAME[vb]
    ksub = vsub = 4
    if case % 4 == 3:   # every 4th case: a NEXT-2 format pair (D = 128, split kernel)
        D = 128
        kname, vname = N2_PAIRS[int(rng.integers(0, len(N2_PAIRS)))]
        (ksub, kb), (vsub, vb) = N2[kname], N2[vname]
        algo = "auto" if algo == "stream" else algo
    heads = np.arange(Hkv)
    lam = CB["lambda"][heads, :D].copy()
    ck, cv = CB[f"ck_{kname}"], CB[f"cv_{vname}"]
    ck = ck if ck.ndim == 2 else ck[heads]
    cv = cv if cv.ndim == 2 else cv[heads]
    kc = synth.gen_codes(n_cap, Hkv, D // ksub, kb, seed=701 + case, batch=B)
    vc = synth.gen_codes(n_cap, Hkv, D // vsub, vb, seed=702 + case, batch=B)
    q = synth.gen_queries(B, Hkv * G, Hkv, D, seed=703 + case)
    kcfg, vcfg = vi.VQConfig(D, ksub, kb), vi.VQConfig(D, vsub, vb)
    kp, vp = ref.pack_codes(kc, kb), ref.pack_codes(vc, vb)
    kw = dict(num_splits=splits, algo=algo, tok_begin=tok_begin, tok_end=tok_end, kcfg=kcfg, vcfg=vcfg)
    if paged:   # the same page permutation for K and V
        kp, bt = _paginate(kp, ps, np.random.default_rng(900 + case))
        vp, _ = _paginate(vp, ps, np.random.default_rng(900 + case))
        kw["block_table"] = t_i32(bt)
    K_res = V_res = r_lens = None
    if use_res:
        r_cap = 32
        K_res = synth.gen_keys(r_cap, Hkv, D, seed=704 + case, batch=B).transpose(0, 2, 1, 3).copy()
        V_res = synth.gen_values(r_cap, Hkv, D, seed=705 + case, batch=B).transpose(0, 2, 1, 3).copy()
        r_lens = np.array([int(rng.integers(0, r_cap + 1)) for _ in range(B)])
        kw.update(k_res=t_bf16(K_res), v_res=t_bf16(V_res), res_lens=t_i32(r_lens))
    o, L = vi.attn_decode(t_bf16(q), t_f32(lam), t_bf16(ck), t_bf16(cv), t_u8(kp), t_u8(vp), t_i32(lens), **kw)
    o_ref, L_ref = ref.attention_decode_batch(q, lam, ck, cv, kc, vc, lens, tok_begin,
                                              None if tok_end < 0 else tok_end, K_res=K_res, V_res=V_res,
                                              res_lens=r_lens)
    _assert_close(o.float().cpu().numpy(), L.cpu().numpy(), o_ref, L_ref)
