"""Profiling driver: a few eager decode-attention layer calls at a BASELINE config (for ncu).

    python scripts/prof_attn.py [--workload cfg2] [--iters 6] [--algo mma] [--splits 0] [--encode]
Random uniform codes (synth.gen_codes_torch), frozen codebooks; prints the per-launch event time.
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

CFG = {"cfg2": (1, 32768), "cfg3": (64, 8192), "cfg4": (1, 196608), "cfg1": (1, 1024),
       "steady": (18, 65536)}   # steady: 144 units of 65536 tokens, use --splits 1 --copies 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--algo", default="mma")
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--encode", action="store_true")
    ap.add_argument("--copies", type=int, default=8)
    args = ap.parse_args()
    B, N = CFG[args.workload]
    dev = torch.device("cuda", 0)
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    lam = torch.from_numpy(z["lambda"]).to(dev)
    inv = torch.from_numpy(z["inv_lambda"]).to(dev)
    ck = torch.from_numpy(synth.bf16_from_bits(z["ck_b2d4"])).to(dev).to(torch.bfloat16)
    cv = torch.from_numpy(synth.bf16_from_bits(z["cv_b2d4"])).to(dev).to(torch.bfloat16)
    C = args.copies
    kcs = [synth.gen_codes_torch((B, 8, N, 32), 8, seed=2 * i, device=dev) for i in range(C)]
    vcs = [synth.gen_codes_torch((B, 8, N, 32), 8, seed=2 * i + 1, device=dev) for i in range(C)]
    q = torch.from_numpy(synth.gen_queries(B, 32, 8, 128, seed=3)).to(dev).to(torch.bfloat16)
    kn = torch.from_numpy(synth.gen_keys(1, 8, 128, seed=4, batch=B)).to(dev).to(torch.bfloat16)
    vn = torch.from_numpy(synth.gen_values(1, 8, 128, seed=5, batch=B)).to(dev).to(torch.bfloat16)
    seq = torch.full((B,), N, dtype=torch.int32, device=dev)
    wp = torch.full((B,), N - 1, dtype=torch.int32, device=dev)
    ws = vi.attn_workspace(B, 32, 8, N, args.splits, device=dev)
    o = torch.empty(B, 32, 128, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, 32, dtype=torch.float32, device=dev)
    times = []
    for i in range(args.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if args.encode:
            vi.encode_kv(kn, vn, inv, ck, cv, kcs[i % C], vcs[i % C], wp)
        e0.record()
        vi.attn_decode(q, lam, ck, cv, kcs[i % C], vcs[i % C], seq, num_splits=args.splits, algo=args.algo, out=o,
                       lse=lse, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    nbytes = B * 8 * N * 64
    print(f"{args.workload} algo={args.algo} splits={vi.attn_num_splits(B, 8, N, args.splits)}: "
          f"per-launch us {['%.1f' % t for t in times]}, best {min(times):.1f} us = {nbytes / min(times) / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
