"""Freeze the d8b16 codebooks (2 bits per element, 65 536 eight-dim centroids; Table 5's 2-bit row
P:624; codebook-size trade-off P:603-610) -- SURVEY §8(f) NEXT-2.

Harness script: calls ONLY oracle/ and synth/ and writes data/d8b16_levels.npz (frozen INPUTS of
the hot path, never expected values).  Reading R18 as for b4d4: Lloyd iterations at 65 536
centroids are beyond a CPU harness, so each book is a 4-level-per-dimension quantile product grid
(4^8 = 65 536 entries): per position t of the 8-dim sub-vector, the levels are the 1/8, 3/8, 5/8,
7/8 quantiles of that position over pinned-transformed calibration keys (K) or synthetic values
(V), rounded to bf16.  The book itself is synth.product_codebook(levels).  Codebook quality does
not enter parity.
Usage: python scripts/fit_codebooks_d8b16.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import ref  # noqa: E402

H_KV, D = 8, 128


def main():
    base = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    inv = base["inv_lambda"]
    kcal = synth.gen_calibration_keys(H_KV, D)
    rng = np.random.default_rng(816)
    sel = rng.choice(kcal.shape[0], size=2048, replace=False)
    xk = np.concatenate([ref.transform_key_pinned(kcal[sel, h, :], inv[h]) for h in range(H_KV)]).reshape(-1, 8)
    xv = synth.gen_values(2048, H_KV, D, seed=3816).reshape(-1, 8)
    qs = np.array([1, 3, 5, 7]) / 8.0
    lk = synth.round_to_bf16(np.quantile(xk.astype(np.float64), qs, axis=0).T.astype(np.float32))   # [8, 4]
    lv = synth.round_to_bf16(np.quantile(xv.astype(np.float64), qs, axis=0).T.astype(np.float32))
    path = os.path.join(ROOT, "data", "d8b16_levels.npz")
    np.savez(path, lv_d8b16_k=synth.bf16_bits(lk), lv_d8b16_v=synth.bf16_bits(lv))
    print(f"wrote {path}: K levels\n{lk}\nV levels\n{lv}")


if __name__ == "__main__":
    main()
