"""Steady-state timing of the bulk prefill encode (vecinfer_encode_kv) after warm-up.

    python scripts/time_encode.py
Prints tokens/s (all 8 KV heads, K + V) per code width and chunk size, and the fraction of the
fp32 ALU roofline (pinned distance: 4 sub + 4 mul + 3 add per (sub-vector, centroid) pair)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402

dev = torch.device("cuda", 0)
z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
inv = torch.from_numpy(z["inv_lambda"]).to(dev)
for name, cfg, bits in (("b1d4", vi.B1D4, 4), ("b2d4", vi.B2D4, 8), ("b4d4", vi.B4D4, 16)):
    ck = torch.from_numpy(synth.bf16_from_bits(z[f"ck_{name}"])).to(dev).to(torch.bfloat16)
    cv = torch.from_numpy(synth.bf16_from_bits(z[f"cv_{name}"])).to(dev).to(torch.bfloat16)
    for T in ((4096, 32768) if bits < 16 else (1024,)):
        k = torch.from_numpy(synth.gen_keys(T, 8, 128, seed=1)).to(dev).to(torch.bfloat16)
        v = torch.from_numpy(synth.gen_values(T, 8, 128, seed=2)).to(dev).to(torch.bfloat16)
        kc = torch.empty(1, 8, T, cfg.row_bytes, dtype=torch.uint8, device=dev)
        vc = torch.empty_like(kc)
        wp = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = vi.encode_workspace(1, T, 8, cfg, cfg, device=dev)
        for _ in range(3):
            vi.encode_kv(k, v, inv, ck, cv, kc, vc, wp, cfg, cfg, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10 if bits < 16 else 3
        e0.record()
        for _ in range(n):
            vi.encode_kv(k, v, inv, ck, cv, kc, vc, wp, cfg, cfg, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3 / n
        evals = T * 8 * 2 * 32 * (1 << bits)
        frac = evals * 11 / s / (128 * 148 * 1.965e9)
        print(f"{name} T={T:6d}: {s * 1e6:9.1f} us  {T / s / 1e6:8.3f} M tokens/s  ALU frac {frac:.3f}", flush=True)
