"""Sequence-sharded decode attention with the cross-GPU merge fused into the attention launch
(vecinfer_attn_decode_xr / vecinfer_decode_step_xr).

Single-process tests run the P ranks as concurrent launches on P streams of the one GPU, over P
in-process windows (XRankWindows.local); the two-process test runs two real ranks (gloo, CUDA IPC
windows) on the same device with the planner's full-size split count.  Every rank must hold
bitwise the same (o, lse), equal to the CPU oracle over the whole sequence (2e-3); the timeout
flag must stay clear.  Expected values come from the oracle only."""
import os
import socket

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
from paper_2510_06175_b200.sharding import XRankWindows, shard_range  # noqa: E402

DEV = torch.device("cuda", 0)
CB = load_codebooks()


def _case(B, n_cap, lens, seed):
    kc = synth.gen_codes(n_cap, 8, 32, 8, seed=seed, batch=B)
    vc = synth.gen_codes(n_cap, 8, 32, 8, seed=seed + 1, batch=B)
    q = synth.gen_queries(B, 32, 8, 128, seed=seed + 2)
    return dict(q=q, kc=kc, vc=vc, seq_lens=np.asarray(lens))


def _dev(c):
    return (torch.from_numpy(c["q"].astype(np.float32)).to(DEV).to(torch.bfloat16),
            torch.from_numpy(CB["lambda"]).to(DEV),
            torch.from_numpy(CB["ck_b2d4"]).to(DEV).to(torch.bfloat16),
            torch.from_numpy(CB["cv_b2d4"]).to(DEV).to(torch.bfloat16),
            torch.from_numpy(c["kc"].astype(np.uint8)).to(DEV),
            torch.from_numpy(c["vc"].astype(np.uint8)).to(DEV),
            torch.tensor(c["seq_lens"], dtype=torch.int32, device=DEV))


def _assert_oracle(o, L, c):
    o_ref, L_ref = ref.attention_decode_batch(c["q"], CB["lambda"], CB["ck_b2d4"], CB["cv_b2d4"], c["kc"], c["vc"],
                                              c["seq_lens"])
    err = row_rel_err(o, o_ref)
    assert err.max() <= TOL_O, f"max row rel err {err.max():.3e}"
    fin = np.isfinite(L_ref)
    assert np.array_equal(np.isfinite(L), fin)
    assert np.abs(L[fin] - L_ref[fin]).max() <= TOL_L
    assert np.all(o[~fin] == 0)


def _run_local(P, c, n_tok, iters=1, splits=2, o_dtype=torch.float32, q_seeds=None):
    """P ranks as concurrent launches on P streams; returns the outputs of every rank per iteration."""
    B = c["q"].shape[0]
    q, lam, ck, cv, kc, vc, seq = _dev(c)
    xrs = XRankWindows.local(P, B * 32, 128, DEV)
    streams = [torch.cuda.Stream(device=DEV) for _ in range(P)]
    ws = [vi.attn_workspace(B, 32, 8, n_tok, splits, device=DEV) for _ in range(P)]
    outs = []
    for it in range(iters):
        qi = q if q_seeds is None else torch.from_numpy(
            synth.gen_queries(B, 32, 8, 128, seed=q_seeds[it]).astype(np.float32)).to(DEV).to(torch.bfloat16)
        torch.cuda.synchronize()
        res = []
        for r in range(P):
            b, e = shard_range(n_tok, r, P)
            with torch.cuda.stream(streams[r]):
                res.append(vi.attn_decode(qi, lam, ck, cv, kc, vc, seq, tok_begin=b, tok_end=e, num_splits=splits,
                                          o_dtype=o_dtype, workspace=ws[r], xr=xrs[r]))
        torch.cuda.synchronize()
        outs.append([(o.float().cpu().numpy(), L.cpu().numpy()) for o, L in res])
    assert int(xrs[0].err.item()) == 0, "a peer partial timed out"
    return outs


@pytest.mark.parametrize("P,B,lens", [(2, 1, [5000]), (3, 2, [4000, 2900]), (4, 2, [6000, 777]), (2, 1, [40])])
def test_xr_local_ranks_vs_oracle(P, B, lens):
    """Fused cross-rank merge over P concurrent 'ranks': identical on every rank, oracle-exact."""
    n_cap = max(lens) + 3
    c = _case(B, n_cap, lens, seed=400 + P + B)
    outs = _run_local(P, c, max(lens))
    o0, L0 = outs[0][0]
    for o, L in outs[0][1:]:
        assert np.array_equal(o, o0) and np.array_equal(L, L0)
    _assert_oracle(o0, L0, c)


def test_xr_repeated_calls_both_parities():
    """Five calls through the same windows (slot parities alternate; consumed slots are zeroed) with a
    new query each time: every call is oracle-exact on every rank."""
    lens = [3000]
    c = _case(1, 3001, lens, seed=420)
    seeds = [421, 422, 423, 424, 425]
    outs = _run_local(3, c, 3000, iters=5, q_seeds=seeds)
    for it, s in enumerate(seeds):
        ci = dict(c, q=synth.gen_queries(1, 32, 8, 128, seed=s))
        o0, L0 = outs[it][0]
        for o, L in outs[it][1:]:
            assert np.array_equal(o, o0)
        _assert_oracle(o0, L0, ci)


def test_xr_bf16_output_and_empty_shard():
    """bf16 output; a rank whose shard is past one sequence's end contributes an empty partial."""
    lens = [2400, 700]
    c = _case(2, 2400, lens, seed=430)
    outs = _run_local(3, c, 2400, o_dtype=torch.bfloat16)   # rank 2 holds [1600, 2400): empty for b = 1
    o0, L0 = outs[0][0]
    for o, L in outs[0][1:]:
        assert np.array_equal(o, o0)
    o_ref, L_ref = ref.attention_decode_batch(c["q"], CB["lambda"], CB["ck_b2d4"], CB["cv_b2d4"], c["kc"], c["vc"],
                                              c["seq_lens"])
    assert row_rel_err(o0, o_ref).max() <= TOL_O + 4e-3   # bf16 output rounding (R13)
    assert np.abs(L0 - L_ref).max() <= TOL_L


def test_xr_decode_step_tail_rank_appends():
    """Bench pattern: every rank holds its own shard cache; the tail rank appends the new token
    (vecinfer_decode_step_xr), the others attend (vecinfer_attn_decode_xr); one launch per rank."""
    N, P = 4100, 2
    c = _case(1, N, [N], seed=440)
    kn = synth.gen_keys(1, 8, 128, seed=441, batch=1)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=442, batch=1)[:, 0]
    q, lam, ck, cv, _, _, _ = _dev(c)
    inv = torch.from_numpy(CB["inv_lambda"]).to(DEV)
    xrs = XRankWindows.local(P, 32, 128, DEV)
    streams = [torch.cuda.Stream(device=DEV) for _ in range(P)]
    shards = [shard_range(N, r, P) for r in range(P)]
    caches = [(torch.from_numpy(c["kc"][:, :, b:e].astype(np.uint8)).to(DEV).contiguous(),
               torch.from_numpy(c["vc"][:, :, b:e].astype(np.uint8)).to(DEV).contiguous()) for b, e in shards]
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    torch.cuda.synchronize()
    res = []
    for r, (b, e) in enumerate(shards):
        kc, vc = caches[r]
        seq = torch.tensor([e - b], dtype=torch.int32, device=DEV)
        with torch.cuda.stream(streams[r]):
            if r == P - 1:
                wp = torch.tensor([e - b - 1], dtype=torch.int32, device=DEV)
                res.append(vi.decode_step(q, torch.from_numpy(kn).to(DEV).to(torch.bfloat16),
                                          torch.from_numpy(vn).to(DEV).to(torch.bfloat16), lam, inv, ck, cv, kc, vc,
                                          wp, seq, num_splits=2, err_flags=err, xr=xrs[r]))
            else:
                res.append(vi.attn_decode(q, lam, ck, cv, kc, vc, seq, num_splits=2, xr=xrs[r]))
    torch.cuda.synchronize()
    assert int(err.item()) == 0 and int(xrs[0].err.item()) == 0
    for h in range(8):   # the appended row (last token of the sequence) is the oracle's encode
        kk, vv = ref.encode_kv(kn[0, h], vn[0, h], CB["inv_lambda"][h], CB["ck_b2d4"][h], CB["cv_b2d4"][h])
        c["kc"][0, h, N - 1], c["vc"][0, h, N - 1] = kk, vv
    assert np.array_equal(caches[-1][0][0, :, -1].cpu().numpy(), c["kc"][0, :, N - 1].astype(np.uint8))
    assert np.array_equal(caches[-1][1][0, :, -1].cpu().numpy(), c["vc"][0, :, N - 1].astype(np.uint8))
    o0, L0 = res[0][0].float().cpu().numpy(), res[0][1].cpu().numpy()
    assert np.array_equal(res[1][0].float().cpu().numpy(), o0)
    _assert_oracle(o0, L0, c)


def test_xr_rejects_unsupported():
    """Paged caches and grids that cannot be a single wave (B*H_kv*2 > #SMs) are refused loudly."""
    c = _case(1, 64, [64], seed=450)
    q, lam, ck, cv, kc, vc, seq = _dev(c)
    xr = XRankWindows.local(2, 32, 128, DEV)[0]
    bt = torch.zeros(1, 2, dtype=torch.int32, device=DEV)
    with pytest.raises(ValueError):
        vi.attn_decode(q, lam, ck, cv, kc.reshape(2, 8, 32, 32), vc.reshape(2, 8, 32, 32), seq, block_table=bt, xr=xr)
    B = 20   # 160 units x 2 splits > 148 SMs
    cb = _case(B, 64, [64] * B, seed=451)
    qb, lam, ck, cv, kcb, vcb, seqb = _dev(cb)
    xrb = XRankWindows.local(2, B * 32, 128, DEV)[0]
    with pytest.raises(RuntimeError, match="UNSUPPORTED"):
        vi.attn_decode(qb, lam, ck, cv, kcb, vcb, seqb, xr=xrb)


# ------------------------------------------------ two real ranks (processes) on the one device
def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, outq):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth as sy
        from helpers import load_codebooks as lcb
        from paper_2510_06175_b200 import vecinfer as v
        from paper_2510_06175_b200.sharding import XRankWindows as XW, shard_range as sr
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        cb = lcb()
        N = 20000   # planner's S (18 at this size per rank) -- the full single-wave configuration
        lam = torch.from_numpy(cb["lambda"]).to(dev)
        ck = torch.from_numpy(cb["ck_b2d4"]).to(dev).to(torch.bfloat16)
        cv = torch.from_numpy(cb["cv_b2d4"]).to(dev).to(torch.bfloat16)
        kc = sy.gen_codes_torch((1, 8, N, 32), 8, seed=15, device=dev)
        vc = sy.gen_codes_torch((1, 8, N, 32), 8, seed=16, device=dev)
        xr = XW(32, 128, dev)
        seq = torch.tensor([N], dtype=torch.int32, device=dev)
        b, e = sr(N, rank, world)
        outs = []
        for it in range(3):
            q = torch.from_numpy(sy.gen_queries(1, 32, 8, 128, seed=17 + it)).to(dev).to(torch.bfloat16)
            o, L = v.attn_decode(q, lam, ck, cv, kc, vc, seq, tok_begin=b, tok_end=e, xr=xr)
            torch.cuda.synchronize()
            outs.append((o.cpu().numpy(), L.cpu().numpy()))
        err = int(xr.err.item())
        inputs = (kc.cpu().numpy(), vc.cpu().numpy()) if rank == 0 else None
        xr.close()
        outq.put((rank, outs, err, inputs))
    finally:
        dist.destroy_process_group()


def test_xr_two_processes_full_split_plan():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, qu)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted((qu.get(timeout=300) for _ in ps), key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
    (_, outs0, err0, inputs), (_, outs1, err1, _) = res
    assert err0 == 0 and err1 == 0
    kc, vc = inputs
    for it in range(3):
        assert np.array_equal(outs0[it][0], outs1[it][0]) and np.array_equal(outs0[it][1], outs1[it][1])
        c = dict(q=synth.gen_queries(1, 32, 8, 128, seed=17 + it), kc=kc.astype(np.int64), vc=vc.astype(np.int64),
                 seq_lens=np.asarray([20000]))
        _assert_oracle(outs0[it][0], outs0[it][1], c)
