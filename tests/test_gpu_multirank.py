"""Sequence-sharded multi-rank decode attention on the GPU (BASELINE configs[3] pattern), with two
ranks sharing one device over gloo (the box has one GPU; NCCL refuses two ranks per device).
Each rank attends its token shard through vecinfer_attn_decode's tok_begin/tok_end hook, the
packed partials are all-gathered, and vecinfer_merge_lse merges them in rank order; every rank
must hold the same o, equal to the unsharded kernel bit-for-bit-close and to the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, outq):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from helpers import load_codebooks
        from paper_2510_06175_b200 import vecinfer as vi
        from paper_2510_06175_b200.sharding import gather_partials_packed, shard_range
        dev = torch.device("cuda", 0)
        cb = load_codebooks()
        N = 5000
        lam = torch.from_numpy(cb["lambda"]).to(dev)
        ck = torch.from_numpy(cb["ck_b2d4"]).to(dev).to(torch.bfloat16)
        cv = torch.from_numpy(cb["cv_b2d4"]).to(dev).to(torch.bfloat16)
        kc = synth.gen_codes_torch((1, 8, N, 32), 8, seed=5, device=dev)     # same seed on every rank
        vc = synth.gen_codes_torch((1, 8, N, 32), 8, seed=6, device=dev)
        q = torch.from_numpy(synth.gen_queries(1, 32, 8, 128, seed=7)).to(dev).to(torch.bfloat16)
        seq = torch.tensor([N], dtype=torch.int32, device=dev)
        b, e = shard_range(N, rank, world)
        o_p, l_p = vi.attn_decode(q, lam, ck, cv, kc, vc, seq, tok_begin=b, tok_end=e)
        o_all, l_all = gather_partials_packed(o_p.cpu(), l_p.cpu())            # gloo: host tensors
        o, lse = vi.merge_lse(o_all.to(dev).contiguous(), l_all.to(dev).contiguous())
        o_ref, l_ref = vi.attn_decode(q, lam, ck, cv, kc, vc, seq)
        torch.cuda.synchronize()
        outq.put((rank, o.cpu().numpy(), lse.cpu().numpy(), o_ref.cpu().numpy(), l_ref.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_sequence_sharded_two_ranks_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (_, o0, l0, oref, lref), (_, o1, l1, _, _) = res
    assert np.array_equal(o0, o1) and np.array_equal(l0, l1)        # identical on every rank
    rel = np.abs(o0 - oref).max(-1) / np.abs(oref).max(-1)
    assert rel.max() <= 2e-3 and np.abs(l0 - lref).max() <= 2e-3
