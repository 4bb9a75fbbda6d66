"""CPU oracle for the VecInfer decode-attention hot path (arXiv 2510.06175).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import or execute anything under oracle/.  The product path
(paper_2510_06175_b200/) never imports it and shares no code, headers, constants or helpers
with it.

Plain, slow, obviously-correct NumPy, following the paper equation by equation:
  * fp64 for the attention path (Eq. 1, 3, 5-7, 10; Alg. 1 outputs),
  * pinned fp32 where an fp32 decision selects an integer (the VQ code, Eq. 2) -- both the
    oracle and the GPU take that decision in the same precision (readings R9, R10).
Every function cites the passage it follows (P:n = /root/reference/PAPER.md line n).

Parity status: every function below is pinned by tests/test_oracle_pins.py against closed
forms, worked examples, invariants or brute force, except `kmeans` (codebook quality needs the
paper's datasets) -- "parity unpinned" for kmeans' optimality; its determinism and the SPEC
worked examples are checked, and it only produces frozen *inputs*, never expected values.
"""
from __future__ import annotations

import math

import numpy as np

# --------------------------------------------------------------------------------------------
# Eq. 5: Walsh-Hadamard matrix, Sylvester recursion, natural order.
# --------------------------------------------------------------------------------------------


def hadamard_pm(D: int) -> np.ndarray:
    """Unnormalised +-1 Hadamard matrix H_pm with H_D = H_pm / sqrt(D) (Eq. 5).

    Built by the recursion [[H, H], [H, -H]] starting from H_1 = [1]; the per-level 1/sqrt(2)
    of Eq. 5 is collected into the single 1/sqrt(D) factor of `hadamard`.
    """
    if D < 1 or (D & (D - 1)) != 0:
        raise ValueError("D must be a power of two (Eq. 5 is defined for D = 2^k)")
    H = np.ones((1, 1), dtype=np.int64)
    while H.shape[0] < D:
        H = np.block([[H, H], [H, -H]])
    return H


def hadamard(D: int) -> np.ndarray:
    """Orthonormal H_D of Eq. 5 (H_D H_D^T = I), fp64."""
    return hadamard_pm(D).astype(np.float64) / math.sqrt(D)


# --------------------------------------------------------------------------------------------
# Eq. 4: smoothing factors from calibration keys.
# --------------------------------------------------------------------------------------------

EPS_FLOOR = np.float32(1e-6)   # SPEC S:91 degenerate-channel floor (reading R6)


def calibrate_smooth(k_cal: np.ndarray, eps: float = 1e-6):
    """lambda_i = sqrt(max |K_i|) per (KV head, channel), Eq. 4.

    k_cal: [n_tokens, n_kv_heads, D], bf16-valued.  Returns (lambda, inv_lambda) fp32
    [n_kv_heads, D] with lambda = max(RN32(sqrt(amax)), RN32(eps)) and inv_lambda = RN32(1/lambda)
    (reading R6: both sides multiply; keys by inv_lambda, queries by lambda).
    """
    k_cal = np.asarray(k_cal, dtype=np.float32)
    if k_cal.shape[0] == 0:
        raise ValueError("empty calibration set")
    amax = np.abs(k_cal).max(axis=0)                         # exact on bf16 values
    lam = np.sqrt(amax.astype(np.float32))                   # IEEE correctly-rounded fp32 sqrt
    lam = np.maximum(lam, np.float32(eps))
    inv = (np.float32(1.0) / lam).astype(np.float32)         # IEEE correctly-rounded fp32 divide
    return lam.astype(np.float32), inv


# --------------------------------------------------------------------------------------------
# Eq. 3 + Eq. 6 + Eq. 7: dual equivalent transformation.
# --------------------------------------------------------------------------------------------


def transform_query(q: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """q~ = q diag(lambda) H_D (Eq. 7 left factor), fp64.  q: [..., D], lam: [D]."""
    q = np.asarray(q, dtype=np.float64)
    D = q.shape[-1]
    return (q * np.asarray(lam, dtype=np.float64)) @ hadamard(D)


def transform_keys_exact(K: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """K~ = K diag(lambda)^-1 H_D (Eq. 7 right factor), fp64 (mathematical path)."""
    K = np.asarray(K, dtype=np.float64)
    D = K.shape[-1]
    return (K / np.asarray(lam, dtype=np.float64)) @ hadamard(D)


FIXED_POINT_BITS = 24          # reading R10: pinned exact fixed point, 2^-24 grid
RANGE_LIMIT = 2.0 ** 32        # |k * inv_lambda| must stay below 2^32 (int64 headroom)


def rn_float32_from_int(X: np.ndarray) -> np.ndarray:
    """Round int64 values to the nearest float32 (ties to even), one rounding."""
    return np.asarray(X, dtype=np.int64).astype(np.float32)


def transform_key_pinned(k: np.ndarray, inv_lam: np.ndarray) -> np.ndarray:
    """Key side of the dual transform, pinned so that codes are reproducible bit for bit.

    Mathematically x = (k diag(lambda)^-1) H_D (Eq. 3 then Eq. 6; S+H order).  The paper
    fixes no rounding, so (reading R10) the smoothed key is put on an exact 2^-24 fixed-point
    grid and rotated exactly in integers:
        A_l = rint_even(k_l * inv_lambda_l * 2^24)            (exact f64 product, < 53 bits)
        X_j = sum_l H_pm[l, j] * A_l                           (exact int64, O(D^2))
        x_j = RN32( RN32(X_j) * 2^-24 ) (*)32 RN32(1/sqrt(D))
    k: [..., D] bf16-valued; inv_lam: [D] fp32.  Returns float32 [..., D].
    """
    k = np.asarray(k, dtype=np.float32)
    D = k.shape[-1]
    prod = k.astype(np.float64) * np.asarray(inv_lam, dtype=np.float32).astype(np.float64)
    if np.any(np.abs(prod) >= RANGE_LIMIT):
        raise OverflowError("|k * inv_lambda| >= 2^32: outside the pinned fixed-point range")
    A = np.rint(prod * float(2 ** FIXED_POINT_BITS)).astype(np.int64)
    X = A @ hadamard_pm(D)                                          # exact integer product
    xs = rn_float32_from_int(X) * np.float32(2.0 ** -FIXED_POINT_BITS)
    inv_sqrt_d = np.float32(1.0 / math.sqrt(D))
    return (xs * inv_sqrt_d).astype(np.float32)


# --------------------------------------------------------------------------------------------
# Eq. 2: product vector quantisation, nearest centroid.
# --------------------------------------------------------------------------------------------


def vq_encode(x: np.ndarray, C: np.ndarray, chunk: int = 2048) -> np.ndarray:
    """Codes j* = argmin_j ||x_i - C_j||^2 per contiguous sub-vector (Eq. 2).

    x: [..., D] float32; C: [2^b, d] (bf16-valued).  Distance evaluated in fp32, every op
    round-to-nearest, no fused multiply-add, summed in the fixed order ((e0^2+e1^2)+e2^2)+e3^2
    (reading R9); ties -> lowest index (np.argmin returns the first minimum).
    Returns int64 codes [..., D/d].
    """
    x = np.asarray(x, dtype=np.float32)
    C = np.asarray(C, dtype=np.float32)
    n_ent, d = C.shape
    D = x.shape[-1]
    if D % d:
        raise ValueError("sub-vector dim must divide D")
    lead = x.shape[:-1]
    sub = x.reshape(-1, d)
    codes = np.empty(sub.shape[0], dtype=np.int64)
    step = max(1, chunk * 256 // n_ent)
    for s0 in range(0, sub.shape[0], step):
        blk = sub[s0:s0 + step]
        dist = None
        for t in range(d):
            e = blk[:, None, t] - C[None, :, t]            # fp32 RN subtract
            e2 = e * e                                       # fp32 RN multiply
            dist = e2 if dist is None else dist + e2         # fp32 RN add, left to right
        codes[s0:s0 + step] = np.argmin(dist, axis=1)
    return codes.reshape(*lead, D // d)


def vq_decode(codes: np.ndarray, C: np.ndarray) -> np.ndarray:
    """VQ^-1: concatenate the selected centroids (Eq. 10), fp64 [..., M*d]."""
    codes = np.asarray(codes, dtype=np.int64)
    C = np.asarray(C, dtype=np.float64)
    out = C[codes]                                            # [..., M, d]
    return out.reshape(*codes.shape[:-1], codes.shape[-1] * C.shape[1])


def encode_kv(k: np.ndarray, v: np.ndarray, inv_lam: np.ndarray, Ck: np.ndarray, Cv: np.ndarray):
    """Prefill (Eq. 8) / decode append (Eq. 9) for one KV head.

    K~_q = VQ(K diag(lambda)^-1 H_D, C_k) (pinned transform), V_q = VQ(V, C_v) (values are not
    transformed).  k, v: [..., D].  Returns (k_codes, v_codes) int64 [..., M].
    """
    x = transform_key_pinned(k, inv_lam)
    return vq_encode(x, Ck), vq_encode(np.asarray(v, dtype=np.float32), Cv)


# --------------------------------------------------------------------------------------------
# Eq. 1 / Eq. 10 and Alg. 1 outputs.
# --------------------------------------------------------------------------------------------


def attention_full(q: np.ndarray, K: np.ndarray, V: np.ndarray):
    """Eq. 1: s = q K^T / sqrt(D), p = softmax(s), o = p V; also L = logsumexp(s).  fp64.

    q: [G, D]; K, V: [N, D].  Empty N -> (o = 0, L = -inf) (SURVEY §8(b) empty-shard rule).
    """
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    G, D = q.shape
    if K.shape[0] == 0:
        return np.zeros((G, V.shape[1])), np.full(G, -np.inf)
    s = q @ K.T / math.sqrt(D)
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    ell = p.sum(axis=1, keepdims=True)
    o = (p @ V) / ell
    L = (m + np.log(ell))[:, 0]
    return o, L


def attention_vq(q: np.ndarray, lam: np.ndarray, Ck: np.ndarray, Cv: np.ndarray,
                 k_codes: np.ndarray, v_codes: np.ndarray):
    """Decode attention over the VQ cache, Eq. 10 with Alg. 1's (o, L).

    q: [G, D] raw query heads sharing one KV head (GQA, reading R15); lam: [D];
    k_codes, v_codes: [N, M].  q~ = q diag(lambda) H_D (Eq. 7); s = q~ VQ^-1(K~_q)^T / sqrt(D);
    o = softmax(s) VQ^-1(V_q); L = logsumexp(s) (natural log, reading R12).  fp64.
    """
    qt = transform_query(q, lam)
    Kh = vq_decode(k_codes, Ck)
    Vh = vq_decode(v_codes, Cv)
    return attention_full(qt, Kh, Vh)


def attention_vq_residual(q: np.ndarray, lam: np.ndarray, Ck: np.ndarray, Cv: np.ndarray,
                          k_codes: np.ndarray, v_codes: np.ndarray, K_res: np.ndarray, V_res: np.ndarray):
    """VQ cache plus a full-precision residual window ("the residual length for all methods
    is set to 128"): one softmax over the union of the quantised tokens and the residual tokens.
    Quantised scores use q~ and VQ^-1(K~_q) (Eq. 10); residual scores use the raw q and raw keys,
    equal to q~ k~^T by Eq. 7.  q: [G, D]; K_res, V_res: [R, D] (R may be 0).  fp64."""
    qt = transform_query(q, lam)
    Kh = vq_decode(k_codes, Ck)
    Vh = vq_decode(v_codes, Cv)
    D = q.shape[-1]
    q = np.asarray(q, dtype=np.float64)
    K_res = np.asarray(K_res, dtype=np.float64).reshape(-1, D)
    V_res = np.asarray(V_res, dtype=np.float64).reshape(-1, D)
    s = np.concatenate([qt @ Kh.T, q @ K_res.T], axis=1) / math.sqrt(D)
    V = np.concatenate([Vh, V_res], axis=0)
    if s.shape[1] == 0:
        return np.zeros((q.shape[0], D)), np.full(q.shape[0], -np.inf)
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    ell = p.sum(axis=1, keepdims=True)
    return (p @ V) / ell, (m + np.log(ell))[:, 0]


def build_lut(q_tilde: np.ndarray, Ck: np.ndarray) -> np.ndarray:
    """Alg. 1 line 4: q~' = reshape(q~, (M, D/M)); lut = q~' C_k^T  -> [M, 2^b] fp64."""
    q_tilde = np.asarray(q_tilde, dtype=np.float64)
    Ck = np.asarray(Ck, dtype=np.float64)
    d = Ck.shape[1]
    return q_tilde.reshape(-1, d) @ Ck.T


def merge_lse(o_parts: np.ndarray, L_parts: np.ndarray):
    """Merge split partials (o_s normalised, L_s) over axis 0: L = logsumexp_s L_s,
    o = sum_s exp(L_s - L) o_s (the online-softmax recurrence of P:745-757 applied to whole
    splits).  Partials with L_s = -inf carry zero weight; all -inf -> (0, -inf).
    """
    o_parts = np.asarray(o_parts, dtype=np.float64)
    L_parts = np.asarray(L_parts, dtype=np.float64)
    Lmax = L_parts.max(axis=0)
    finite = np.isfinite(Lmax)
    safe = np.where(finite, Lmax, 0.0)
    w = np.where(np.isfinite(L_parts), np.exp(L_parts - safe[None]), 0.0)
    tot = w.sum(axis=0)
    L = np.where(finite, safe + np.log(np.where(finite, tot, 1.0)), -np.inf)
    o = (w[..., None] * o_parts).sum(axis=0) / np.where(finite, tot, 1.0)[..., None]
    o = np.where(finite[..., None], o, 0.0)
    return o, L


def attention_decode_batch(q: np.ndarray, lam: np.ndarray, Ck: np.ndarray, Cv: np.ndarray,
                           k_codes: np.ndarray, v_codes: np.ndarray, seq_lens, tok_begin: int = 0,
                           tok_end: int | None = None, K_res=None, V_res=None, res_lens=None):
    """One decode-attention layer call over a batch (the §8(b) vecinfer_attn_decode contract).

    q: [B, H_q, D]; lam: [H_kv, D]; Ck/Cv: [H_kv, 2^b, d] (or [2^b, d] shared);
    k_codes/v_codes: [B, H_kv, n_cap, M]; token range [tok_begin, min(tok_end, seq_len)).
    Query head i reads KV head i // (H_q/H_kv) (GQA).  Optional residual window K_res/V_res
    [B, H_kv, R_cap, D] with res_lens [B] (attention_vq_residual).  Returns o [B, H_q, D], L [B, H_q].
    """
    B, Hq, D = q.shape
    Hkv = k_codes.shape[1]
    G = Hq // Hkv
    o = np.zeros((B, Hq, D))
    L = np.full((B, Hq), -np.inf)
    for b in range(B):
        n = int(seq_lens[b])
        e = n if tok_end is None else min(int(tok_end), n)
        s = min(int(tok_begin), e)
        for h in range(Hkv):
            ck = Ck[h] if np.ndim(Ck) == 3 else Ck
            cv = Cv[h] if np.ndim(Cv) == 3 else Cv
            if K_res is None:
                oo, LL = attention_vq(q[b, h * G:(h + 1) * G], lam[h], ck, cv,
                                      k_codes[b, h, s:e], v_codes[b, h, s:e])
            else:
                r = int(res_lens[b])
                oo, LL = attention_vq_residual(q[b, h * G:(h + 1) * G], lam[h], ck, cv, k_codes[b, h, s:e],
                                               v_codes[b, h, s:e], K_res[b, h, :r], V_res[b, h, :r])
            o[b, h * G:(h + 1) * G] = oo
            L[b, h * G:(h + 1) * G] = LL
    return o, L


# --------------------------------------------------------------------------------------------
# Code packing (reading R11) and byte accounting.
# --------------------------------------------------------------------------------------------


def pack_codes(codes: np.ndarray, code_bits: int) -> np.ndarray:
    """Token-major packed rows (reading R11): the M codes of a row form one little-endian bit
    string, code m in bits [m*b, (m+1)*b) (bit i of the row = bit i%8 of byte i//8).  For b = 8
    that is one byte per code, for b = 4 sub-vector 2i in the low nibble, for b = 16 little-endian
    u16; b = 10 / 12 (d4b10, d8b12: P:338, 340, 993-999) are the same rule.  Row length
    M*b/8 bytes.  codes: [..., M] -> uint8 [..., M*b/8]."""
    codes = np.asarray(codes, dtype=np.int64)
    if code_bits == 8:
        return codes.astype(np.uint8)
    if code_bits == 4:
        lo = codes[..., 0::2]
        hi = codes[..., 1::2]
        return (lo | (hi << 4)).astype(np.uint8)
    if code_bits == 16:
        u = codes.astype(np.uint16)
        return u.view(np.uint8).reshape(*codes.shape[:-1], codes.shape[-1] * 2)
    if code_bits not in (10, 12):
        raise ValueError("code_bits must be 4, 8, 10, 12 or 16")
    return pack_bitstream(codes, code_bits)


def pack_bitstream(codes: np.ndarray, code_bits: int) -> np.ndarray:
    """The R11 rule written bit by bit, for any b (pack_codes' 4/8/16-bit branches are its
    special cases; tests/test_oracle_pins.py checks that they agree)."""
    codes = np.asarray(codes, dtype=np.int64)
    M = codes.shape[-1]
    if (M * code_bits) % 8:
        raise ValueError("a row of codes must fill whole bytes")
    bits = np.zeros(codes.shape[:-1] + (M * code_bits,), dtype=np.uint8)
    for m in range(M):                      # bit t of code m -> row bit m*b + t
        for t in range(code_bits):
            bits[..., m * code_bits + t] = (codes[..., m] >> t) & 1
    out = np.zeros(codes.shape[:-1] + (M * code_bits // 8,), dtype=np.int64)
    for i in range(8):
        out |= bits[..., i::8].astype(np.int64) << i
    return out.astype(np.uint8)


def unpack_bitstream(packed: np.ndarray, code_bits: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    nbits = packed.shape[-1] * 8
    bits = np.zeros(packed.shape[:-1] + (nbits,), dtype=np.int64)
    for i in range(8):
        bits[..., i::8] = (packed >> i) & 1
    M = nbits // code_bits
    out = np.zeros(packed.shape[:-1] + (M,), dtype=np.int64)
    for m in range(M):
        for t in range(code_bits):
            out[..., m] |= bits[..., m * code_bits + t] << t
    return out


def unpack_codes(packed: np.ndarray, code_bits: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    if code_bits == 8:
        return packed.astype(np.int64)
    if code_bits == 4:
        lo = (packed & 0xF).astype(np.int64)
        hi = (packed >> 4).astype(np.int64)
        out = np.empty(packed.shape[:-1] + (packed.shape[-1] * 2,), dtype=np.int64)
        out[..., 0::2] = lo
        out[..., 1::2] = hi
        return out
    if code_bits == 16:
        return packed.view(np.uint16).astype(np.int64)
    if code_bits not in (10, 12):
        raise ValueError("code_bits must be 4, 8, 10, 12 or 16")
    return unpack_bitstream(packed, code_bits)


def codebook_bytes(sub_dim: int, code_bits: int) -> int:
    """2^b x d x 2 bytes."""
    return (1 << code_bits) * sub_dim * 2


def index_bytes_per_vector(head_dim: int, sub_dim: int, code_bits: int) -> float:
    """(d_h / d) x (b / 8) bytes per cached vector."""
    return (head_dim // sub_dim) * code_bits / 8.0


def avg_bits(sub_dim: int, code_bits: int) -> float:
    """b / d bits per element ("Avg. bit" column of Table 2, e.g. d4b8 -> 2)."""
    return code_bits / sub_dim


# --------------------------------------------------------------------------------------------
# Codebook fitting (harness only): K-means, <= 30 iterations.
# --------------------------------------------------------------------------------------------


def _sqdist(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    return (X * X).sum(1)[:, None] - 2.0 * X @ C.T + (C * C).sum(1)[None, :]


def kmeans(X: np.ndarray, n_clusters: int, max_iters: int = 30, seed: int = 0):
    """K-means with k-means++ seeding and Lloyd iterations ("maximum number of iterations
    set to 30"); empty clusters re-seeded at the current worst-distortion point.
    Returns (centroids fp64 [n_clusters, d], objective history)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    if n < n_clusters:
        raise ValueError("insufficient data for k-means")
    rng = np.random.default_rng(seed)
    C = np.empty((n_clusters, X.shape[1]))
    C[0] = X[rng.integers(n)]
    d2 = ((X - C[0]) ** 2).sum(1)
    for c in range(1, n_clusters):
        tot = d2.sum()
        if tot <= 0:
            C[c] = X[rng.integers(n)]
        else:
            C[c] = X[rng.choice(n, p=d2 / tot)]
        d2 = np.minimum(d2, ((X - C[c]) ** 2).sum(1))
    hist = []
    for _ in range(max_iters):
        assign = np.empty(n, dtype=np.int64)
        best = np.empty(n)
        for s0 in range(0, n, 65536):
            dd = _sqdist(X[s0:s0 + 65536], C)
            assign[s0:s0 + 65536] = dd.argmin(1)
            best[s0:s0 + 65536] = dd[np.arange(dd.shape[0]), assign[s0:s0 + 65536]]
        hist.append(float(np.maximum(best, 0).sum()))
        counts = np.bincount(assign, minlength=n_clusters)
        sums = np.zeros_like(C)
        np.add.at(sums, assign, X)
        newC = C.copy()
        nz = counts > 0
        newC[nz] = sums[nz] / counts[nz, None]
        order = np.argsort(-best, kind="stable")
        k = 0
        for c in np.nonzero(~nz)[0]:
            newC[c] = X[order[k]]
            k += 1
        if np.array_equal(newC, C):
            break
        C = newC
    return C, hist


def pinned_sqdist(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Pinned fp32 squared distance of Eq. 2 under reading R9 for every (point, centroid) pair:
    e_t = x_t - c_t, dist = ((e_0^2 + e_1^2) + e_2^2) + ..., every op an fp32 round-to-nearest op,
    no fused multiply-add.  X: [n, d], C: [k, d] -> fp32 [n, k]."""
    X = np.asarray(X, dtype=np.float32)
    C = np.asarray(C, dtype=np.float32)
    dist = None
    for t in range(X.shape[1]):
        e = X[:, None, t] - C[None, :, t]
        e2 = e * e
        dist = e2 if dist is None else dist + e2
    return dist


def kmeans_lloyd_step(X: np.ndarray, C: np.ndarray):
    """One Lloyd iteration of the codebook k-means ("K-means ... maximum number of
    iterations set to 30"), on fp32 points and fp32 centroids, in the order
    the algorithm states:

      1. assignment: a_i = argmin_j dist(x_i, C_j) with the pinned fp32 distance of Eq. 2 /
         reading R9 (the encoder's rule, so a fitted codebook and its encoder agree), ties to the
         lowest index; best_i = dist(x_i, C_{a_i});
      2. update: for every cluster with n_j > 0 points, C'_j = RN32(sum_{a_i = j} x_i / n_j), the
         sum and the division in fp64 (the exact mean up to one fp64 rounding each);
      3. empty clusters (n_j = 0, in increasing j) are re-seeded at the points of largest best_i
         (ties: lowest point index), one point per empty cluster.

    Returns (C' fp32 [k, d], assign int64 [n], best fp32 [n], counts int64 [k], objective =
    sum_i best_i in fp64).
    """
    X = np.asarray(X, dtype=np.float32)
    C = np.asarray(C, dtype=np.float32)
    n, k = X.shape[0], C.shape[0]
    assign = np.empty(n, dtype=np.int64)
    best = np.empty(n, dtype=np.float32)
    step = max(1, (1 << 22) // max(k, 1))
    for s0 in range(0, n, step):
        dd = pinned_sqdist(X[s0:s0 + step], C)
        a = np.argmin(dd, axis=1)                              # first minimum = lowest index
        assign[s0:s0 + step] = a
        best[s0:s0 + step] = dd[np.arange(dd.shape[0]), a]
    counts = np.bincount(assign, minlength=k)
    sums = np.zeros((k, X.shape[1]), dtype=np.float64)
    np.add.at(sums, assign, X.astype(np.float64))
    newC = C.copy()
    nz = counts > 0
    newC[nz] = (sums[nz] / counts[nz, None]).astype(np.float32)
    empty = np.nonzero(~nz)[0]
    if empty.size:
        order = np.argsort(-best.astype(np.float64), kind="stable")   # largest best first, ties lowest index
        for e_i, c in enumerate(empty):
            newC[c] = X[order[e_i]]
    return newC, assign, best, counts, float(best.astype(np.float64).sum())
