"""Per-CTA phase timeline of the attention kernel (profiling build libvecinfer_phase.so).

    python -m paper_2510_06175_b200.build --phase-timing
    VECINFER_LIB=paper_2510_06175_b200/libvecinfer_phase.so python scripts/phase_attn.py --case 1,32768,0
Stamps (globaltimer ns, thread 0 of each CTA): 0 start, 1 prologue done, 2 main loop done,
3 warp partials in smem, 5 split partial published (atomic done), 4 exit.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_06175_b200 import _lib, vecinfer as vi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append", required=True)
    ap.add_argument("--sm-mhz", type=float, default=1965.0, help="SM clock converting the cycle stamps")
    ap.add_argument("--per-cta", action="store_true")
    args = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    lam = torch.from_numpy(z["lambda"]).to(dev)
    ck = torch.from_numpy(synth.bf16_from_bits(z["ck_b2d4"])).to(dev).to(torch.bfloat16)
    cv = torch.from_numpy(synth.bf16_from_bits(z["cv_b2d4"])).to(dev).to(torch.bfloat16)
    for c in args.case:
        B, N, splits = map(int, c.split(",")[:3])
        algo = c.split(",")[3] if len(c.split(",")) > 3 else "auto"
        fused = len(c.split(",")) > 4 and c.split(",")[4] == "fused"   # decode_step with the fused append
        S = vi.attn_num_splits(B, 8, N, splits)
        nct = vi.attn_num_ctas(B, 8, N, splits) if algo != "stream" else 148
        buf = torch.zeros(nct * 32, dtype=torch.int64, device=dev)
        lib.vecinfer_debug_set_phase_buffer.argtypes = [ctypes.c_void_p]
        lib.vecinfer_debug_set_phase_buffer(ctypes.c_void_p(buf.data_ptr()))
        kc = synth.gen_codes_torch((B, 8, N, 32), 8, seed=1, device=dev)
        vc = synth.gen_codes_torch((B, 8, N, 32), 8, seed=2, device=dev)
        q = torch.from_numpy(synth.gen_queries(B, 32, 8, 128, seed=3)).to(dev).to(torch.bfloat16)
        seq = torch.full((B,), N, dtype=torch.int32, device=dev)
        ws = vi.attn_workspace(B, 32, 8, N, splits, device=dev)
        for _ in range(5):
            buf.zero_()
            if fused:
                inv = torch.from_numpy(z["inv_lambda"]).to(dev)
                kn = torch.from_numpy(synth.gen_keys(1, 8, 128, seed=4, batch=B)[:, 0]).to(dev).to(torch.bfloat16)
                vn = torch.from_numpy(synth.gen_values(1, 8, 128, seed=5, batch=B)[:, 0]).to(dev).to(torch.bfloat16)
                vi.decode_step(q, kn, vn, lam, inv, ck, cv, kc, vc, seq - 1, seq, num_splits=splits,
                               workspace=vi.decode_step_workspace(B, 32, 8, N, device=dev), algo=algo)
            else:
                vi.attn_decode(q, lam, ck, cv, kc, vc, seq, num_splits=splits, workspace=ws, algo=algo)
            torch.cuda.synchronize()
        both = buf.view(nct, 32).cpu().numpy().astype(np.float64)
        t, cyc = both[:, :16], both[:, 16:]
        t0 = t[:, 0].min()
        # within a CTA: SM cycles at the sampled clock (fine); the CTA's start: globaltimer (coarse)
        mhz = args.sm_mhz
        rel = np.where(t == 0, 0.0, (t[:, :1] - t0) / 1e3 + (cyc - cyc[:, :1]) / mhz)
        span = (t[:, 4].max() - t0) / 1e3
        print(f"B={B} N={N} S={S} CTAs={nct}: span {span:.2f} us")

        def st(x, name):
            print(f"   {name:32s} min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f} us")
        rel[t == 0] = np.nan   # stamps a CTA did not write (e.g. no deferred merge)

        def st(x, name):   # noqa: F811
            x = x[~np.isnan(x)]
            if x.size:
                print(f"   {name:32s} min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f} us  (n={x.size})")
        st(rel[:, 0], "CTA start (rel)")
        if np.isfinite(rel[:, 12]).any():   # stream kernel (attn_stream.cu) stamps
            st(rel[:, 6] - rel[:, 0], "prologue: fill+wait+segs")
            st(rel[:, 12] - rel[:, 6], "prologue: piece setup (loads)")
            st(rel[:, 11] - rel[:, 12], "prologue: q~ transform")
            st(rel[:, 1] - rel[:, 11], "prologue: encode + sync")
            st(rel[:, 13] - rel[:, 11], "  encode: transform (thread 0)")
            st(rel[:, 14] - rel[:, 13], "  encode: scan (thread 0)")
            st(rel[:, 10] - rel[:, 14], "  encode: barrier (slowest warp)")
            st(rel[:, 1] - rel[:, 10], "  encode: reduce + store + sync")
            st(rel[:, 2] - rel[:, 1], "main loop warp 0 (last round)")
            st(rel[:, 7] - rel[:, 2], "wait for slowest warp")
            st(rel[:, 9] - rel[:, 7], "combine + store")
            st(rel[:, 5] - rel[:, 3], "spin wait (deferred merges)")
            st(rel[:, 4] - rel[:, 5], "slice merge")
        else:                                # split kernel (attn_mma.cu) stamps
            st(rel[:, 1] - rel[:, 0], "prologue (fill+q~+sync)")
            st(rel[:, 9] - rel[:, 0], "  start -> after griddep wait")
            st(rel[:, 13] - rel[:, 9], "  wait -> seq_lens, 1st tile issued")
            st(rel[:, 14] - rel[:, 13], "  table store + q~ (warp 0)")
            st(rel[:, 1] - rel[:, 14], "  barrier (slowest warp)")
            st(rel[:, 2] - rel[:, 1], "main loop warp 0 (incl. bq)")
            st(rel[:, 3] - rel[:, 2], "warp partials -> smem + sync")
            st(rel[:, 8] - rel[:, 3], "combine + publish")
            st(rel[:, 10] - rel[:, 8], "merge loads + poll (all seen)")
            st(rel[:, 5] - rel[:, 10], "fold + output store")
            st(rel[:, 8], "publish done (rel)")
            st(rel[:, 4] - rel[:, 5], "slice merge")
        st(rel[:, 4], "CTA end (rel)")
        if args.per_cta and np.isfinite(rel[:, 12]).any():   # stream kernel: main loop vs segments per CTA
            U, V = B * 8, nct
            segs_per = np.array([((c * U + U - 1) // V) - ((c * U) // V) + 1 for c in range(nct)])
            ml = rel[:, 2] - rel[:, 1]
            end = rel[:, 4]
            for ns in sorted(set(segs_per.tolist())):
                sel = segs_per == ns
                print(f"   CTAs with {ns} segments ({(ns + 1) // 2} rounds): n={sel.sum()}, main loop mean {ml[sel].mean():.2f} "
                      f"max {ml[sel].max():.2f} us, end mean {end[sel].mean():.2f} max {end[sel].max():.2f} us")
        if args.per_cta and not np.isfinite(rel[:, 12]).any():   # per-CTA main loop vs SM id (is the spread systematic?)
            sm = both[:, 15].astype(int)
            ml = rel[:, 2] - rel[:, 1]
            order = np.argsort(ml)
            print("   slowest CTAs (cta, sm, main loop us):", [(int(i), int(sm[i]), round(float(ml[i]), 2)) for i in order[-8:]])
            print("   fastest CTAs (cta, sm, main loop us):", [(int(i), int(sm[i]), round(float(ml[i]), 2)) for i in order[:8]])
            # per GPC-ish groups: SM id // 18
            for g in range(0, 148, 37):
                sel = (sm >= g) & (sm < g + 37)
                if sel.any():
                    print(f"   SMs {g:3d}-{g + 36:3d}: main loop mean {ml[sel].mean():.2f} us over {sel.sum()} CTAs")

if __name__ == "__main__":
    main()
