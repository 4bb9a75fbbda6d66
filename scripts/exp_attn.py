"""Attention-kernel timing experiments (CUDA-graph replay of back-to-back launches, events).

    python scripts/exp_attn.py --case B,N,splits[,algo] ...
Prints µs per launch and GB/s on compressed bytes; rotates over enough cache copies to exceed L2.
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402


def _paginate(kc, ps, seed):
    """[B, H, N, row] -> random-permuted page pool [n_pages, H, ps, row] and block table [B, N/ps]."""
    B, H, N, row = kc.shape
    npb = N // ps
    g = torch.Generator(device="cpu").manual_seed(seed)
    perm = torch.randperm(B * npb, generator=g).to(kc.device)
    blocks = kc.view(B, H, npb, ps, row).permute(0, 2, 1, 3, 4).reshape(B * npb, H, ps, row)
    pool = torch.empty(blocks.shape, dtype=blocks.dtype, device=blocks.device)
    pool[perm] = blocks
    return pool, perm.view(B, npb).to(torch.int32)


FMTS = {"b2d4": (4, 8), "b1d4": (4, 4), "b4d4": (4, 16), "d8b8": (8, 8), "d8b12": (8, 12), "d4b10": (4, 10), "d2b8": (2, 8),
        "d8b16": (8, 16)}


def _book(name, side, dev):
    if name == "d8b16":   # product book from its frozen 8 x 4 levels
        z = np.load(os.path.join(ROOT, "data", "d8b16_levels.npz"))
        cb = synth.product_codebook(synth.bf16_from_bits(z[f"lv_d8b16_{side}"]))
        return torch.from_numpy(cb).to(dev).to(torch.bfloat16)
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz" if name in ("b2d4", "b1d4", "b4d4") else
                             "next2_codebooks.npz"))
    return torch.from_numpy(synth.bf16_from_bits(z[f"c{side}_{name}"])).to(dev).to(torch.bfloat16)


def run(B, N, splits, algo, reps=20, with_encode=False, paged=0, dh=128, fmt=("b2d4", "b2d4"), early=False):
    dev = torch.device("cuda", 0)
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    lam = torch.from_numpy(z["lambda"]).to(dev)
    ck, cv = _book(fmt[0], "k", dev), _book(fmt[1], "v", dev)
    kcfg, vcfg = vi.VQConfig(dh, *FMTS[fmt[0]]), vi.VQConfig(dh, *FMTS[fmt[1]])
    nbytes = B * 8 * N * (kcfg.row_bytes + vcfg.row_bytes)
    copies = max(1, int(np.ceil(400e6 / nbytes)))
    kcs = [synth.gen_codes_torch((B, 8, N, kcfg.row_bytes), 8, seed=2 * i, device=dev) for i in range(copies)]
    vcs = [synth.gen_codes_torch((B, 8, N, vcfg.row_bytes), 8, seed=2 * i + 1, device=dev) for i in range(copies)]
    cfg = kcfg
    if dh != 128:
        lam = lam[:, :dh].contiguous()
    bt = None
    if paged:
        pk = [_paginate(k, paged, 7 + i) for i, k in enumerate(kcs)]
        pv = [_paginate(v, paged, 7 + i) for i, v in enumerate(vcs)]
        kcs, vcs, bt = [p[0] for p in pk], [p[0] for p in pv], pk[0][1]   # same permutation for K and V
    q = torch.from_numpy(synth.gen_queries(B, 32, 8, dh, seed=3)).to(dev).to(torch.bfloat16)
    seq = torch.full((B,), N, dtype=torch.int32, device=dev)
    ws = [vi.attn_workspace(B, 32, 8, N, splits, device=dev) for _ in range(copies)]
    o = torch.empty(B, 32, dh, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, 32, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(copies):
            if algo != "none":
                vi.attn_decode(q, lam, ck, cv, kcs[i], vcs[i], seq, num_splits=splits, algo=algo, out=o, lse=lse,
                               workspace=ws[i], block_table=bt, kcfg=kcfg, vcfg=vcfg)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    n_l = max(copies, 8)
    inv = torch.from_numpy(z["inv_lambda"]).to(dev)[:, :dh].contiguous()
    kn = torch.from_numpy(synth.gen_keys(1, 8, dh, seed=4, batch=B)).to(dev).to(torch.bfloat16)
    vn = torch.from_numpy(synth.gen_values(1, 8, dh, seed=5, batch=B)).to(dev).to(torch.bfloat16)
    wp = torch.full((B,), N - 1, dtype=torch.int32, device=dev)
    with torch.cuda.stream(s):
        vi.encode_kv(kn, vn, inv, ck, cv, kcs[0], vcs[0], wp, kcfg, vcfg, block_table=bt)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(n_l):
            if with_encode == "fused":
                vi.decode_step(q, kn[:, 0], vn[:, 0], lam, inv, ck, cv, kcs[i % copies], vcs[i % copies], wp, seq,
                               num_splits=splits, out=o, lse=lse, workspace=ws[i % copies], kcfg=kcfg, vcfg=vcfg,
                               early_cache=early)
                continue
            if with_encode:
                vi.encode_kv(kn, vn, inv, ck, cv, kcs[i % copies], vcs[i % copies], wp, kcfg, vcfg, block_table=bt)
            if algo == "none":
                continue
            vi.attn_decode(q, lam, ck, cv, kcs[i % copies], vcs[i % copies], seq, num_splits=splits, algo=algo,
                           out=o, lse=lse, workspace=ws[i % copies], block_table=bt, kcfg=kcfg, vcfg=vcfg,
                           early_cache=early and not with_encode)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):      # CUDAGraph.replay() launches on the CURRENT stream
        g.replay()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * n_l)
    S = vi.attn_num_splits(B, 8, N, splits)
    try:
        V = vi.attn_num_ctas(B, 8, N, splits)
    except Exception:
        V = -1
    print(f"{'early ' if early else ''}{fmt[0]}/{fmt[1]} B={B:3d} N={N:7d} S={S:3d} V={V:4d} algo={algo:4s} enc={with_encode}: {us:8.2f} us/launch  {nbytes / us / 1e3:7.0f} GB/s  "
          f"({100 * nbytes / us / 1e3 / 6553.6:.1f}% of 6553.6)  cyc/token-head@1.9GHz/SM={us * 1.9e3 * 148 / (B * 8 * N):.2f}",
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append", required=True)
    ap.add_argument("--paged", type=int, default=0, help="page size of a random-permuted paged cache (0: contiguous)")
    ap.add_argument("--dh", type=int, default=128, help="head dim (128 or 64)")
    ap.add_argument("--early", action="store_true", help="VECINFER_ATTN_FLAG_EARLY_CACHE launches")
    ap.add_argument("--fmt", action="append", default=None, help="K,V formats, e.g. d8b12,d8b8 (default b2d4,b2d4)")
    args = ap.parse_args()
    for f in args.fmt or ["b2d4,b2d4"]:
        for c in args.case:
            p = c.split(",")
            run(int(p[0]), int(p[1]), int(p[2]), p[3] if len(p) > 3 else "mma", paged=args.paged, dh=args.dh,
                with_encode=(p[4] if p[4] == "fused" else True) if len(p) > 4 else False, fmt=tuple(f.split(",")),
                early=args.early)
    from paper_2510_06175_b200 import _lib
    lib = _lib.load()
    print("max active clusters (size: n):", {c: lib.vecinfer_debug_attn_max_clusters(c) for c in (2, 4, 8, 12, 16)})
