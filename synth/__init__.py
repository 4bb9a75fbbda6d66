"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the VecInfer method (no smoothing, no Hadamard, no VQ,
no attention).  It only draws random tensors with the shapes and value structure of the
paper's workloads and rounds them to bf16 (the storage type of the KV cache, PAPER.md:143
"assuming 16-bit floating-point precision").

Recipe:
  * keys, KV head h: channel scales sigma[h,c] = exp(U[ln 0.5, ln 2]) (rng seed 1000+h),
    4 outlier channels per head (seeded indices) scaled x16, entries N(0, sigma^2).
    This reproduces the fixed-channel outliers of Llama-3.1-8B's key cache
    (Fig. 1a, "key cache outliers") without model weights.
  * values: N(0, 1).
  * queries: N(0, 1) * sigma_q[h], sigma_q = 2*sqrt(D)/||sigma[h]||_2 so that the
    attention score q.k/sqrt(D) has std ~2 (softmax neither flat nor one-hot).
  * calibration keys: an independent draw (seed 2000+h) of 256 x 512 tokens.
All tensors are float32 arrays whose values are exactly representable in bf16
(round-to-nearest-even), plus helpers to view them as raw bf16 bits.
"""
from __future__ import annotations

import numpy as np

N_OUTLIER_CHANNELS = 4
OUTLIER_SCALE = 16.0


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32 holding bf16 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    bits = x.view(np.uint32).astype(np.uint64)
    lsb = (bits >> np.uint64(16)) & np.uint64(1)
    rounded = ((bits + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    out = (rounded & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
    return out.reshape(x.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Raw bf16 bit patterns (uint16) of float32 values that are already bf16-exact."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32)
    if np.any(b & np.uint32(0xFFFF)):
        raise ValueError("values are not bf16-representable; call round_to_bf16 first")
    return (b >> np.uint32(16)).astype(np.uint16)


def bf16_from_bits(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def key_channel_profile(n_kv_heads: int, head_dim: int):
    """Per-(head, channel) std of the synthetic keys: log-uniform scales with 4 x16 outlier channels."""
    sigma = np.empty((n_kv_heads, head_dim), dtype=np.float64)
    outliers = np.empty((n_kv_heads, N_OUTLIER_CHANNELS), dtype=np.int64)
    for h in range(n_kv_heads):
        rng = np.random.default_rng(1000 + h)
        s = np.exp(rng.uniform(np.log(0.5), np.log(2.0), size=head_dim))
        idx = rng.choice(head_dim, size=N_OUTLIER_CHANNELS, replace=False)
        s[idx] *= OUTLIER_SCALE
        sigma[h] = s
        outliers[h] = np.sort(idx)
    return sigma, outliers


def gen_keys(n_tokens: int, n_kv_heads: int, head_dim: int, seed: int, batch: int = 1,
             laplace: bool = False) -> np.ndarray:
    """Keys [batch, n_tokens, n_kv_heads, head_dim] (bf16-exact float32) with channel outliers."""
    sigma, _ = key_channel_profile(n_kv_heads, head_dim)
    rng = np.random.default_rng(seed)
    shape = (batch, n_tokens, n_kv_heads, head_dim)
    if laplace:
        z = rng.laplace(0.0, 1.0 / np.sqrt(2.0), size=shape).astype(np.float32)
    else:
        z = rng.standard_normal(size=shape, dtype=np.float32)
    return round_to_bf16(z * sigma[None, None].astype(np.float32))


def gen_values(n_tokens: int, n_kv_heads: int, head_dim: int, seed: int, batch: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    z = rng.standard_normal(size=(batch, n_tokens, n_kv_heads, head_dim), dtype=np.float32)
    return round_to_bf16(z)


def gen_queries(batch: int, n_q_heads: int, n_kv_heads: int, head_dim: int, seed: int) -> np.ndarray:
    """Queries [batch, n_q_heads, head_dim]; query head i reads KV head i // (n_q_heads // n_kv_heads)."""
    sigma, _ = key_channel_profile(n_kv_heads, head_dim)
    group = n_q_heads // n_kv_heads
    sq = 2.0 * np.sqrt(head_dim) / np.linalg.norm(sigma, axis=1)        # [n_kv_heads]
    rng = np.random.default_rng(seed)
    z = rng.standard_normal(size=(batch, n_q_heads, head_dim), dtype=np.float32)
    scale = np.repeat(sq, group).astype(np.float32)[None, :, None]
    return round_to_bf16(z * scale)


def gen_calibration_keys(n_kv_heads: int, head_dim: int, n_samples: int = 256, sample_len: int = 512,
                         seed_base: int = 2000) -> np.ndarray:
    """Calibration keys [n_samples*sample_len, n_kv_heads, head_dim] (256 x 512 tokens)."""
    sigma, _ = key_channel_profile(n_kv_heads, head_dim)
    n = n_samples * sample_len
    out = np.empty((n, n_kv_heads, head_dim), dtype=np.float32)
    for h in range(n_kv_heads):
        rng = np.random.default_rng(seed_base + h)
        out[:, h, :] = rng.standard_normal(size=(n, head_dim), dtype=np.float32) * sigma[h].astype(np.float32)
    return round_to_bf16(out)


def gen_codes(n_tokens: int, n_kv_heads: int, n_sub: int, code_bits: int, seed: int, batch: int = 1) -> np.ndarray:
    """Uniform random code indices [batch, n_kv_heads, n_tokens, n_sub] (int64), for attention-only tests."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << code_bits, size=(batch, n_kv_heads, n_tokens, n_sub), dtype=np.int64)


def gen_codebook(n_entries: int, sub_dim: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """A random bf16-exact codebook [n_entries, sub_dim] (used where codebook quality is irrelevant)."""
    rng = np.random.default_rng(seed)
    return round_to_bf16(rng.standard_normal(size=(n_entries, sub_dim), dtype=np.float32) * np.float32(scale))


def grid_levels(n_levels: int, step: float = 0.5) -> np.ndarray:
    """Dyadic, symmetric per-dimension levels, e.g. 4 levels -> [-0.75, -0.25, 0.25, 0.75]."""
    return (np.arange(n_levels, dtype=np.float64) - (n_levels - 1) / 2.0) * step


def product_grid_codebook(n_levels: int, sub_dim: int = 4, step: float = 0.5) -> np.ndarray:
    """Product-grid codebook: entry index = sum_t digit_t * n_levels**t, coordinate t = levels[digit_t].

    Used by the closed-form nearest-neighbour pins: with dyadic levels the
    nearest centroid is the per-dimension nearest level, a property that holds independently of
    any search code.
    """
    lv = grid_levels(n_levels, step)
    n = n_levels ** sub_dim
    idx = np.arange(n)
    cb = np.empty((n, sub_dim), dtype=np.float32)
    for t in range(sub_dim):
        cb[:, t] = lv[(idx // n_levels ** t) % n_levels]
    return cb


def product_codebook(levels: np.ndarray) -> np.ndarray:
    """Product codebook from per-dimension levels [d, n]: entry j has coordinate t = levels[t][digit_t(j)],
    digit_t(j) = (j // n**t) % n (dimension 0 is the least significant digit).  Index expansion only
    (used to build the frozen 65 536-entry d8b16 books from their 8 x 4 stored levels)."""
    levels = np.asarray(levels, dtype=np.float32)
    d, n = levels.shape
    idx = np.arange(n ** d)
    cb = np.empty((n ** d, d), dtype=np.float32)
    for t in range(d):
        cb[:, t] = levels[t][(idx // n ** t) % n]
    return cb


def dyadic_points(n: int, sub_dim: int, n_levels: int, step: float, seed: int, denom: int = 8) -> np.ndarray:
    """Random dyadic points covering the grid range, including exact level midpoints (genuine ties)."""
    rng = np.random.default_rng(seed)
    lo = -(n_levels / 2.0) * step - step
    hi = (n_levels / 2.0) * step + step
    k = rng.integers(int(lo * denom), int(hi * denom) + 1, size=(n, sub_dim))
    return (k / denom).astype(np.float32)


def gen_codes_torch(shape, code_bits: int, seed: int, device="cuda"):
    """Uniform random PACKED code bytes (uint8) generated with torch's seeded RNG on `device`, for
    full-size (GiB-scale) attention workloads where a NumPy draw would dominate the run time.
    Every byte pattern is a valid code at 4/8/16 bits, so uniform bytes = uniform codes."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randint(0, 256, tuple(shape), dtype=torch.uint8, device=device, generator=g)
