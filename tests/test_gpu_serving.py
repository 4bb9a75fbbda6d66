"""Ragged batch over a shared page pool (cache.PagedVQCache; serving integration, SURVEY §8(f)
NEXT-4).  Sequences of different lengths are prefilled, decoded step by step (pages
allocated when a sequence crosses a page boundary), removed and replaced while others continue; at
every step the outputs match the ORACLE on the oracle-encoded codes of each sequence's tokens, and
the allocator never leaks or double-books a page."""
import numpy as np
import pytest

import synth
from oracle import ref
from helpers import load_codebooks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2510_06175_b200.cache import PagedVQCache  # noqa: E402
from test_gpu_parity import _assert_close, t_bf16, t_f32  # noqa: E402

CB = load_codebooks()


def _oracle_step(keys, vals, q):
    """Oracle attention of one sequence (keys / vals [n, H, D] raw) with query q [H_q, D]."""
    kc = np.zeros((1, 8, len(keys), 32), np.int64)
    vc = np.zeros_like(kc)
    for h in range(8):
        kk, vv = ref.encode_kv(keys[:, h], vals[:, h], CB["inv_lambda"][h], CB["ck_b2d4"][h], CB["cv_b2d4"][h])
        kc[0, h], vc[0, h] = kk, vv
    return ref.attention_decode_batch(q[None], CB["lambda"], CB["ck_b2d4"], CB["cv_b2d4"], kc, vc, [len(keys)])


@pytest.mark.parametrize("page_size", [32, 64])
def test_paged_serving_ragged_batch(page_size):
    rng = np.random.default_rng(900 + page_size)
    cache = PagedVQCache(4, 8, n_pages=64, page_size=page_size, max_len=512, lam=t_f32(CB["lambda"]),
                         inv_lambda=t_f32(CB["inv_lambda"]), ck=t_bf16(CB["ck_b2d4"]), cv=t_bf16(CB["cv_b2d4"]))
    toks = {}

    def add(s, T, seed):
        k = synth.gen_keys(T, 8, 128, seed=seed)[0]
        v = synth.gen_values(T, 8, 128, seed=seed + 1)[0]
        cache.add(s, t_bf16(k), t_bf16(v))
        toks[s] = [k, v]

    add(0, 95, 910)
    add(1, 31, 912)
    add(2, 200, 914)
    for step in range(40):
        if step == 12:                       # a sequence finishes; a new one takes its slot
            cache.remove(1)
            del toks[1]
            add(1, 64, 916)
        if step == 20:
            add(3, 1, 918)
        slots = sorted(toks)
        n = len(slots)
        q = synth.gen_queries(n, 32, 8, 128, seed=1000 + step)
        kn = synth.gen_keys(1, 8, 128, seed=2000 + step, batch=n)[:, 0]
        vn = synth.gen_values(1, 8, 128, seed=3000 + step, batch=n)[:, 0]
        o, L = cache.step(t_bf16(q), t_bf16(kn), t_bf16(vn), slots)
        o, L = o.cpu().numpy(), L.cpu().numpy()
        for i, s in enumerate(slots):
            toks[s][0] = np.concatenate([toks[s][0], kn[i][None]])
            toks[s][1] = np.concatenate([toks[s][1], vn[i][None]])
            if step % 7 == 0 or step == 39:
                _assert_close(o[i:i + 1], L[i:i + 1], *_oracle_step(toks[s][0], toks[s][1], q[i]))
        used = [p for s in range(4) for p in cache.bt_host[s]]
        assert len(used) == len(set(used)) and not set(used) & set(cache.free)
        assert len(used) + len(cache.free) == 64
        for s in slots:
            assert cache.lens[s] == len(toks[s][0]) and len(cache.bt_host[s]) == -(-cache.lens[s] // page_size)
