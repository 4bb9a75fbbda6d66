"""Where the end-to-end step time goes at cfg2 (B=1, N=32k, 32 layers of vecinfer_decode_step):
graph replays back to back (device time), the same with a host wait per step, and with the packed
H2D / D2H copies of bench.py's e2e path (4 chunks).  Prints ms per step for each.

    python scripts/exp_e2e.py [--chunks 4]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--steps", type=int, default=200)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L, B, N, H = 32, 1, 32768, 8
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    lam = torch.from_numpy(z["lambda"]).to(dev)
    inv = torch.from_numpy(z["inv_lambda"]).to(dev)
    ck = torch.from_numpy(synth.bf16_from_bits(z["ck_b2d4"])).to(dev).to(torch.bfloat16)
    cv = torch.from_numpy(synth.bf16_from_bits(z["cv_b2d4"])).to(dev).to(torch.bfloat16)
    kcs = [synth.gen_codes_torch((B, H, N, 32), 8, seed=2 * l, device=dev) for l in range(L)]
    vcs = [synth.gen_codes_torch((B, H, N, 32), 8, seed=2 * l + 1, device=dev) for l in range(L)]
    nq, nk = B * 32 * 128, B * H * 128
    h_in = torch.randn(L, nq + 2 * nk).to(torch.bfloat16).pin_memory()
    d_in = torch.empty_like(h_in, device=dev)
    q_d = [d_in[l, :nq].view(B, 32, 128) for l in range(L)]
    kn_d = [d_in[l, nq:nq + nk].view(B, H, 128) for l in range(L)]
    vn_d = [d_in[l, nq + nk:].view(B, H, 128) for l in range(L)]
    o = torch.empty(L, B, 32, 128, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(L, B, 32, dtype=torch.float32, device=dev)
    o_h = torch.empty(o.shape, dtype=o.dtype).pin_memory()
    ws = [vi.decode_step_workspace(B, 32, H, N, device=dev) for _ in range(L)]
    wp = torch.full((B,), N - 1, dtype=torch.int32, device=dev)
    sl = torch.full((B,), N, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream()
    cs_in, cs_out = torch.cuda.Stream(), torch.cuda.Stream()

    def layer(l):
        vi.decode_step(q_d[l], kn_d[l], vn_d[l], lam, inv, ck, cv, kcs[l], vcs[l], wp, sl, out=o[l], lse=lse[l],
                       workspace=ws[l], early_cache=True)

    def body(copies):
        cur = torch.cuda.current_stream()
        if not copies:
            for l in range(L):
                layer(l)
            return
        if args.chunks > 0:
            C = args.chunks
            hin = [(c * L // C, (c + 1) * L // C) for c in range(C)]
            hout = hin
        else:   # -1: inputs [0,1) + [1,L), outputs [0,L-1) + [L-1,L)
            hin, hout = [(0, 1), (1, L)], [(0, L - 1), (L - 1, L)]
        ev_in = [torch.cuda.Event() for _ in hin]
        cs_in.wait_stream(cur)
        cs_out.wait_stream(cur)
        with torch.cuda.stream(cs_in):
            for c, (a, b) in enumerate(hin):
                d_in[a:b].copy_(h_in[a:b], non_blocking=True)
                ev_in[c].record(cs_in)
        start_of = {a: c for c, (a, b) in enumerate(hin)}
        end_of = {b - 1: (a, b) for (a, b) in hout}
        for l in range(L):
            if l in start_of:
                cur.wait_event(ev_in[start_of[l]])
            layer(l)
            if l in end_of:
                a, b = end_of[l]
                ev = torch.cuda.Event()
                ev.record(cur)
                with torch.cuda.stream(cs_out):
                    cs_out.wait_event(ev)
                    o_h[a:b].copy_(o[a:b], non_blocking=True)
        cur.wait_stream(cs_in)
        cur.wait_stream(cs_out)

    graphs = {}
    with torch.cuda.stream(s):
        for copies in (False, True):
            body(copies)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                body(copies)
            graphs[copies] = g
    done = torch.cuda.Event()
    with torch.cuda.stream(s):
        for copies in (False, True):
            g = graphs[copies]
            for wait in (False, True):
                for _ in range(5):
                    g.replay()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(args.steps):
                    g.replay()
                    if wait:
                        done.record(s)
                        while not done.query():
                            pass
                e1.record(s)
                torch.cuda.synchronize()
                wall = (time.perf_counter() - t0) * 1e3 / args.steps
                print(f"copies={copies!s:5} host_wait={wait!s:5}: {e0.elapsed_time(e1) / args.steps:.4f} ms/step (events)"
                      f"  {wall:.4f} ms/step (wall)", flush=True)


if __name__ == "__main__":
    main()
