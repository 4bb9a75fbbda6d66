"""Fit and freeze the codebooks of the paper's other VQ configurations:
d8b8 (1-bit), d8b12 (1.5-bit), d4b10 (2.5-bit), d2b8 (4-bit) -- P:338, 340, 478, 946, 993-999.

Harness script: calls ONLY oracle/ and synth/, reuses lambda / inv_lambda from
data/llama8b_synth_codebooks.npz and writes data/next2_codebooks.npz (frozen INPUTS of the hot
path, never expected values).  Keys on pinned-transformed keys, values raw (Eq. 8).
  * 256-entry books (d8b8, d2b8): one per KV head, k-means++ + <= 30 Lloyd iterations.
  * 1024 / 4096-entry books (d4b10, d8b12): one book shared by the heads, k-means++ + 8 Lloyd
    iterations on 2^16 sub-vectors (reading R18: codebook quality does not enter parity).
Usage: python scripts/fit_codebooks_next2.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import ref  # noqa: E402

H_KV, D = 8, 128


def main():
    t0 = time.time()
    base = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    inv = base["inv_lambda"]
    kcal = synth.gen_calibration_keys(H_KV, D)
    rng = np.random.default_rng(78)
    out = {}
    for name, d, n in (("d8b8", 8, 256), ("d2b8", 2, 256)):
        cks, cvs = [], []
        for h in range(H_KV):
            sel = rng.choice(kcal.shape[0], size=4096, replace=False)
            xk = ref.transform_key_pinned(kcal[sel, h, :], inv[h]).reshape(-1, d)
            xv = synth.gen_values(4096, 1, D, seed=3200 + h)[0, :, 0, :].reshape(-1, d)
            ck, hk = ref.kmeans(xk, n, max_iters=30, seed=20 * h + d)
            cv, hv = ref.kmeans(xv, n, max_iters=30, seed=20 * h + d + 1)
            cks.append(synth.round_to_bf16(ck.astype(np.float32)))
            cvs.append(synth.round_to_bf16(cv.astype(np.float32)))
            print(f"{name} head {h}: K {hk[0]:.4g}->{hk[-1]:.4g}, V {hv[0]:.4g}->{hv[-1]:.4g}  {time.time()-t0:.0f}s")
        out[f"ck_{name}"] = synth.bf16_bits(np.stack(cks))
        out[f"cv_{name}"] = synth.bf16_bits(np.stack(cvs))
    for name, d, n in (("d4b10", 4, 1024), ("d8b12", 8, 4096)):
        ntok = (1 << 16) * d // D
        sel = rng.choice(kcal.shape[0], size=ntok, replace=False)
        xk = np.concatenate([ref.transform_key_pinned(kcal[sel, h, :], inv[h]) for h in range(H_KV)]).reshape(-1, d)
        xk = xk[rng.choice(xk.shape[0], size=1 << 16, replace=False)]
        xv = synth.gen_values(ntok, H_KV, D, seed=3300).reshape(-1, d)[: 1 << 16]
        ck, hk = ref.kmeans(xk, n, max_iters=8, seed=d * 1000 + n)
        cv, hv = ref.kmeans(xv, n, max_iters=8, seed=d * 1000 + n + 1)
        out[f"ck_{name}"] = synth.bf16_bits(synth.round_to_bf16(ck.astype(np.float32)))
        out[f"cv_{name}"] = synth.bf16_bits(synth.round_to_bf16(cv.astype(np.float32)))
        print(f"{name}: K {hk[0]:.4g}->{hk[-1]:.4g}, V {hv[0]:.4g}->{hv[-1]:.4g}  {time.time()-t0:.0f}s")
    path = os.path.join(ROOT, "data", "next2_codebooks.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)/1024:.0f} KiB) in {time.time()-t0:.1f}s")


if __name__ == "__main__":
    main()
