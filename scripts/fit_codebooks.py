"""Fit and freeze the synthetic Llama-3.1-8B-shaped smoothing factors and codebooks.

Harness script (offline step of the method): it calls ONLY oracle/ and
synth/ and writes data/llama8b_synth_codebooks.npz, which the tests and bench.py load as frozen
INPUTS (codebooks are inputs of the hot path, never expected values).

  * lambda, inv_lambda [8, 128] fp32: Eq. 4 on 256 x 512 synthetic calibration tokens.
  * C_k / C_v per KV head for b1d4 (16 x 4) and b2d4 (256 x 4): k-means++ + <= 30 Lloyd
    iterations on 2^18 sub-vectors; C_k on pinned-transformed keys, C_v on raw values
    (Eq. 8).  Centroids rounded to bf16.
  * b4d4 (65536 x 4), one codebook shared by all heads: 16-level per-dimension quantile product
    grid (reading R18; Lloyd at 65536 centroids is too slow for the harness and parity does not
    depend on codebook quality).
Usage: python scripts/fit_codebooks.py [--out data/llama8b_synth_codebooks.npz]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import ref  # noqa: E402

H_KV, D = 8, 128


def fit(X, n, seed):
    C, hist = ref.kmeans(X, n, max_iters=30, seed=seed)
    return synth.round_to_bf16(C.astype(np.float32)), hist


def quantile_grid(X, levels=16):
    qs = (np.arange(levels) + 0.5) / levels
    lv = np.quantile(X.reshape(-1), qs)            # pooled over the 4 sub-vector dims
    idx = np.arange(levels ** 4)
    cb = np.empty((levels ** 4, 4), dtype=np.float32)
    for t in range(4):
        cb[:, t] = lv[(idx // levels ** t) % levels]
    return synth.round_to_bf16(cb)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    ap.add_argument("--train-tokens", type=int, default=8192)
    args = ap.parse_args()
    t0 = time.time()
    kcal = synth.gen_calibration_keys(H_KV, D)                       # [131072, 8, 128]
    lam, inv = ref.calibrate_smooth(kcal)
    print(f"calibration {kcal.shape} -> lambda range [{lam.min():.3f}, {lam.max():.3f}]  {time.time()-t0:.1f}s")
    out = {"lambda": lam, "inv_lambda": inv}
    rng = np.random.default_rng(77)
    for bits, n in ((4, 16), (8, 256)):
        name = {4: "b1d4", 8: "b2d4"}[bits]
        cks, cvs = [], []
        for h in range(H_KV):
            sel = rng.choice(kcal.shape[0], size=args.train_tokens, replace=False)
            xk = ref.transform_key_pinned(kcal[sel, h, :], inv[h]).reshape(-1, 4)
            xv = synth.gen_values(args.train_tokens, 1, D, seed=3000 + h)[0, :, 0, :].reshape(-1, 4)
            ck, hk = fit(xk, n, seed=10 * h + 1)
            cv, hv = fit(xv, n, seed=10 * h + 2)
            cks.append(ck)
            cvs.append(cv)
            print(f"{name} head {h}: kmeans K obj {hk[0]:.4g}->{hk[-1]:.4g} ({len(hk)} it), "
                  f"V obj {hv[0]:.4g}->{hv[-1]:.4g} ({len(hv)} it)  {time.time()-t0:.1f}s")
        out[f"ck_{name}"] = synth.bf16_bits(np.stack(cks))
        out[f"cv_{name}"] = synth.bf16_bits(np.stack(cvs))
    sel = rng.choice(kcal.shape[0], size=args.train_tokens, replace=False)
    xk = np.concatenate([ref.transform_key_pinned(kcal[sel, h, :], inv[h]) for h in range(H_KV)])
    xv = synth.gen_values(args.train_tokens, H_KV, D, seed=3100)
    out["ck_b4d4"] = synth.bf16_bits(quantile_grid(xk))
    out["cv_b4d4"] = synth.bf16_bits(quantile_grid(xv))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savez_compressed(args.out, **out)
    print(f"wrote {args.out} ({os.path.getsize(args.out)/1024:.0f} KiB) in {time.time()-t0:.1f}s")


if __name__ == "__main__":
    main()
