"""World-size-2 gloo tests of the multi-GPU host logic (sharding.py) on CPU.

The partials each rank contributes are computed by the ORACLE here (no GPU on this host); what is
under test is the host-side partition, the all-gather (rank order) and the packed exchange: the
merged result must equal the unsharded oracle attention.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q_):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_06175_b200.sharding import gather_partials, gather_partials_packed, shard_range, batch_shard
        rng = np.random.default_rng(0)
        N = 1000
        Ck = synth.gen_codebook(256, 4, seed=1)
        Cv = synth.gen_codebook(256, 4, seed=2)
        kc = rng.integers(0, 256, (N, 32))
        vc = rng.integers(0, 256, (N, 32))
        lam = np.exp(rng.uniform(-1, 1, 128))
        q = rng.standard_normal((4, 128))
        b, e = shard_range(N, rank, world)
        o, L = ref.attention_vq(q, lam, Ck, Cv, kc[b:e], vc[b:e])
        o_all, L_all = gather_partials(torch.tensor(o, dtype=torch.float32), torch.tensor(L, dtype=torch.float32))
        o_p, L_p = gather_partials_packed(torch.tensor(o, dtype=torch.float32), torch.tensor(L, dtype=torch.float32))
        mo, mL = ref.merge_lse(o_all.double().numpy(), L_all.double().numpy())
        want_o, want_L = ref.attention_vq(q, lam, Ck, Cv, kc, vc)
        ok = (np.abs(mo - want_o).max() < 1e-5 and np.abs(mL - want_L).max() < 1e-5
              and torch.equal(o_all, o_p) and torch.equal(L_all, L_p))
        # batch sharding: the union of the rank slices is the batch, disjoint
        sl = [batch_shard(64, r, world) for r in range(world)]
        ok = ok and sl[0][0] == 0 and sl[-1][1] == 64 and all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
        q_.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_sequence_sharded_gather_merge_world2():
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q_)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q_.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("n,world", [(196608, 8), (1000, 3), (5, 4), (0, 2)])
def test_shard_range_partition(n, world):
    from paper_2510_06175_b200.sharding import shard_range
    rs = [shard_range(n, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
    assert all(b % 32 == 0 for b, _ in rs if b < n)
