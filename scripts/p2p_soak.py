"""Soak test of the fused P2P exchange + merge (vecinfer_merge_lse_p2p): 2, 3 and 4 ranks sharing one
GPU, hundreds of exchanges through the same windows with fresh data each time; every 10th result is
compared bit for bit with vecinfer_merge_lse over all ranks' partials.

    python scripts/p2p_soak.py
"""
import os, socket, sys
import numpy as np
import torch, torch.distributed as dist, torch.multiprocessing as mp
ROOT = os.getcwd(); sys.path.insert(0, ROOT)

def _port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p

def rank_fn(rank, world, port, iters, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_06175_b200 import vecinfer as vi
    from paper_2510_06175_b200.sharding import P2PExchange
    dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
    B, HQ, D = 4, 32, 128
    ex = P2PExchange(B * HQ, D, dev)
    bad = 0
    for it in range(iters):
        parts = []
        for r in range(world):
            g = torch.Generator().manual_seed(100000 * it + r)
            parts.append((torch.randn(B, HQ, D, generator=g), torch.randn(B, HQ, generator=g) * 4))
        o_m, l_m = ex.merge(parts[rank][0].to(dev).contiguous(), parts[rank][1].to(dev).contiguous())
        if it % 10 == 0 or it == iters - 1:
            o_r, l_r = vi.merge_lse(torch.stack([p[0] for p in parts]).to(dev).contiguous(),
                                    torch.stack([p[1] for p in parts]).to(dev).contiguous())
            torch.cuda.synchronize()
            bad += int(not (torch.equal(o_m, o_r) and torch.equal(l_m, l_r)))
    torch.cuda.synchronize()
    err = int(ex.err.item())
    ex.close()
    outq.put((rank, bad, err))
    dist.destroy_process_group()

if __name__ == "__main__":
    for world, iters in ((2, 500), (3, 300), (4, 200)):
        ctx = mp.get_context("spawn"); q = ctx.Queue(); port = _port()
        ps = [ctx.Process(target=rank_fn, args=(r, world, port, iters, q)) for r in range(world)]
        for p in ps: p.start()
        res = [q.get(timeout=900) for _ in ps]
        for p in ps: p.join(timeout=60)
        print(f"world={world} iters={iters}: mismatches {[r[1] for r in sorted(res)]}, timeouts {[r[2] for r in sorted(res)]}", flush=True)
