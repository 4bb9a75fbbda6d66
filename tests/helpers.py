"""Shared test helpers: frozen synthetic codebooks and tolerance metrics (no method arithmetic)."""
import os

import numpy as np

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODEBOOKS = os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz")
CODEBOOKS_NEXT2 = os.path.join(ROOT, "data", "next2_codebooks.npz")   # d8b8, d8b12, d4b10, d2b8
LEVELS_D8B16 = os.path.join(ROOT, "data", "d8b16_levels.npz")          # 8 x 4 levels -> 65 536 x 8 book

# north_star: outputs within 2e-3 max-abs relative error (bf16 I/O, fp32 accumulation);
# measured per (b, h_q) row on the fp32 output (reading R13)
TOL_O = 2e-3
TOL_L = 2e-3


def load_codebooks():
    """dict with lambda, inv_lambda (fp32 [8,128]) and ck_/cv_ b1d4, b2d4 ([8,n,4]), b4d4 ([65536,4])
    as bf16-exact float32 arrays."""
    z = np.load(CODEBOOKS)
    out = {"lambda": z["lambda"], "inv_lambda": z["inv_lambda"]}
    for path in (CODEBOOKS, CODEBOOKS_NEXT2):
        if not os.path.exists(path):
            continue
        z = np.load(path)
        for k in z.files:
            if k.startswith("ck_") or k.startswith("cv_"):
                out[k] = synth.bf16_from_bits(z[k])
    if os.path.exists(LEVELS_D8B16):   # d8b16: shared product books from their stored levels
        z = np.load(LEVELS_D8B16)
        out["ck_d8b16"] = synth.product_codebook(synth.bf16_from_bits(z["lv_d8b16_k"]))
        out["cv_d8b16"] = synth.product_codebook(synth.bf16_from_bits(z["lv_d8b16_v"]))
    return out


def row_rel_err(o_gpu, o_ref):
    """max_i |o_gpu - o_ref| / max_i |o_ref| per row (last axis); rows with o_ref == 0 use abs error."""
    o_gpu = np.asarray(o_gpu, dtype=np.float64)
    o_ref = np.asarray(o_ref, dtype=np.float64)
    num = np.abs(o_gpu - o_ref).max(-1)
    den = np.abs(o_ref).max(-1)
    return np.where(den > 0, num / np.where(den > 0, den, 1), num)
