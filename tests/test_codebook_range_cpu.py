"""DESIGN.md reading R24: the kernels hold centroids as fp16 copies, so every codebook value must be
exactly representable in fp16.  Checks the committed codebooks (data/*.npz, bf16 bit patterns)
and the d8b16 product book built from its levels.  Plain NumPy: no library, no GPU."""
import os

import numpy as np

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bf16_bits_to_f32(bits):
    return (np.asarray(bits, dtype=np.uint32) << 16).view(np.float32)


def _fp16_exact(x):
    x = np.asarray(x, dtype=np.float32)
    with np.errstate(over="ignore"):   # out-of-range values become inf (and fail the comparison)
        return np.array_equal(x.astype(np.float16).astype(np.float32), x)


def test_fp16_exactness_rule():
    """The rule itself: bf16 values inside the fp16 normal range round-trip; outside do not."""
    ok = _bf16_bits_to_f32(np.array([0x0000, 0x3F80, 0xBF80, 0x477F, 0x3880, 0x4200]))   # 0, +-1, 65280, 2^-14, 32
    assert _fp16_exact(ok)
    assert not _fp16_exact(_bf16_bits_to_f32(np.array([0x4780])))   # 65536 > 65504
    assert not _fp16_exact(_bf16_bits_to_f32(np.array([0x3381])))   # 2^-24 * (1 + 1/128): subnormal, bits lost


def test_committed_codebooks_are_fp16_exact():
    for name in ("llama8b_synth_codebooks.npz", "next2_codebooks.npz"):
        z = np.load(os.path.join(ROOT, "data", name))
        for k in z.files:
            if k.startswith(("ck_", "cv_")):
                assert _fp16_exact(_bf16_bits_to_f32(z[k])), f"{name}:{k} has values outside fp16"


def test_d8b16_product_book_is_fp16_exact():
    z = np.load(os.path.join(ROOT, "data", "d8b16_levels.npz"))
    for side in ("k", "v"):
        book = synth.product_codebook(synth.bf16_from_bits(z[f"lv_d8b16_{side}"]))
        assert book.shape == (65536, 8)
        assert _fp16_exact(np.asarray(book, dtype=np.float32))
