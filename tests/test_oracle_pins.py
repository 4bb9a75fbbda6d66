"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU needed).

Each test names the passage (P:n = PAPER.md line n, S:n = SPEC.md line n) and the kind of pin:
closed form, worked example, invariant, special case reducing to a textbook/library routine,
or brute force.  A plausible slip in the oracle (dropped term, sign, index, transposed operand,
wrong rounding) fails at least one of them.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.special

import synth
from oracle import ref


# ----------------------------------------------------------------------------- Hadamard, Eq. 5
@pytest.mark.parametrize("D", [1, 2, 4, 8, 16, 32, 64, 128, 256])
def test_hadamard_pm_orthogonality_exact(D):
    """H_pm H_pm^T = D I exactly in integers (BASELINE north_star 'H.H^T = nI')."""
    H = ref.hadamard_pm(D)
    assert H.dtype == np.int64
    assert np.array_equal(H @ H.T, D * np.eye(D, dtype=np.int64))
    Hn = ref.hadamard(D)
    assert np.max(np.abs(Hn @ Hn.T - np.eye(D))) <= 1e-12   # orthonormal H_D


@pytest.mark.parametrize("D", [2, 8, 128, 256])
def test_hadamard_matches_sylvester_closed_form(D):
    """Closed form of the Sylvester recursion: H_pm[i, j] = (-1)^popcount(i & j) (natural order)."""
    i = np.arange(D)[:, None]
    j = np.arange(D)[None, :]
    pop = np.vectorize(lambda v: bin(int(v)).count("1"))(i & j)
    assert np.array_equal(ref.hadamard_pm(D), np.where(pop % 2 == 0, 1, -1))


def test_hadamard_worked_examples(golden):
    assert np.array_equal(ref.hadamard(1), np.array(golden["hadamard_H1"]["value"]))
    assert np.allclose(ref.hadamard(2) * math.sqrt(2), golden["hadamard_H2_times_sqrt2"]["value"], atol=1e-15)
    assert np.allclose(ref.hadamard(4)[0], golden["hadamard_H4_row0"]["value"], atol=1e-15)
    D = golden["hadamard_entry_magnitude"]["D"]
    assert np.allclose(np.abs(ref.hadamard(D)), 1 / math.sqrt(D), atol=1e-15)


def test_hadamard_involution_and_norm():
    """H symmetric orthogonal => H(Hx) = x and ||xH|| = ||x|| (used by Lemma 1)."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((50, 128))
    H = ref.hadamard(128)
    assert np.array_equal(H, H.T)
    assert np.max(np.abs(x @ H @ H - x)) < 1e-12
    assert np.allclose(np.linalg.norm(x @ H, axis=1), np.linalg.norm(x, axis=1), rtol=1e-13)


def test_hadamard_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        ref.hadamard_pm(96)


# ---------------------------------------------------------------------------- smoothing, Eq. 4
def test_calibration_worked_examples(golden):
    ex = golden["calibration_example"]
    K = np.zeros((3, 1, 3), dtype=np.float32)
    K[:, 0, 0] = ex["channel"]                      # {-4, 1, 2} -> 2
    K[:, 0, 1] = 1.0                                # all ones -> 1
    K[:, 0, 2] = 0.0                                # zero channel -> eps
    lam, inv = ref.calibrate_smooth(K)
    assert lam[0, 0] == np.float32(ex["lambda"])
    assert lam[0, 1] == np.float32(golden["calibration_ones"]["lambda"])
    assert lam[0, 2] == np.float32(golden["calibration_zero"]["lambda_f32_of"])
    assert inv[0, 0] == np.float32(0.5) and inv[0, 1] == np.float32(1.0)
    with pytest.raises(ValueError):
        ref.calibrate_smooth(np.zeros((0, 1, 4), dtype=np.float32))


def test_calibration_max_identity():
    """max_n |K_nc / lambda_c| = sqrt(max_n |K_nc|) (direct algebra on Eq. 4)."""
    K = synth.gen_calibration_keys(2, 64, n_samples=4, sample_len=64)
    lam, _ = ref.calibrate_smooth(K)
    lhs = np.abs(K.astype(np.float64) / lam[None].astype(np.float64)).max(axis=0)
    rhs = np.sqrt(np.abs(K.astype(np.float64)).max(axis=0))
    assert np.allclose(lhs, rhs, rtol=1e-6)


def test_calibration_is_correctly_rounded_sqrt():
    """lambda = RN32(sqrt(amax)) exactly: check with exact rational arithmetic on a few values."""
    vals = np.array([2.0, 3.0, 0.0078125, 17.25, 1e-3], dtype=np.float32)
    vals = synth.round_to_bf16(vals)
    K = vals.reshape(1, 1, -1)
    lam, inv = ref.calibrate_smooth(K)
    for a, l in zip(vals, lam[0]):
        if a == 0:
            continue
        # l is RN32(sqrt(a)) iff (l - ulp/2)^2 <= a <= (l + ulp/2)^2
        lf = Fraction(float(l))
        ulp = Fraction(float(np.spacing(l)))
        assert (lf - ulp / 2) ** 2 <= Fraction(float(a)) <= (lf + ulp / 2) ** 2


# ------------------------------------------------------------- dual transform, Eq. 3, 6, 7
@pytest.mark.parametrize("seed", range(5))
def test_dual_transform_invariance_fp64(seed):
    """q~ K~^T = q K^T (Eq. 7) to <= 1e-10 relative in fp64 (north_star)."""
    rng = np.random.default_rng(seed)
    D = 128
    q = rng.standard_normal((4, D))
    K = synth.gen_keys(256, 1, D, seed=seed)[0, :, 0, :]
    lam = np.exp(rng.uniform(-2, 2, D))
    lhs = ref.transform_query(q, lam) @ ref.transform_keys_exact(K, lam).T
    rhs = q @ K.T.astype(np.float64)
    assert np.max(np.abs(lhs - rhs)) / np.max(np.abs(rhs)) <= 1e-10


def test_transform_special_cases():
    """lambda = 1 -> plain Hadamard; q = 0 -> 0."""
    rng = np.random.default_rng(3)
    K = rng.standard_normal((8, 64))
    assert np.allclose(ref.transform_keys_exact(K, np.ones(64)), K @ ref.hadamard(64), atol=1e-14)
    assert np.array_equal(ref.transform_query(np.zeros((1, 64)), np.ones(64)), np.zeros((1, 64)))


def test_lemma1_norm_identity():
    """Appendix H: per-row mean of K~^2 equals ||K_i / lambda||^2 / D exactly."""
    K = synth.gen_keys(64, 1, 128, seed=9, laplace=True)[0, :, 0, :].astype(np.float64)
    lam = np.exp(np.random.default_rng(9).uniform(-1, 1, 128))
    Kt = ref.transform_keys_exact(K, lam)
    assert np.allclose((Kt ** 2).mean(1), ((K / lam) ** 2).sum(1) / 128, rtol=1e-12)


def test_lemma1_spreads_outliers():
    """Lemma 1 conclusion: a single spike spreads over all D columns (|entry| -> 1/sqrt(D))."""
    K = np.zeros((1, 128))
    K[0, 17] = 100.0
    Kt = ref.transform_keys_exact(K, np.ones(128))
    assert np.allclose(np.abs(Kt), 100.0 / math.sqrt(128))


# ----------------------------------------------------------- pinned key transform (reading R10)
def _exact_rn_f32(n: int) -> float:
    """Correctly rounded (ties-to-even) int -> float32, by exact integer arithmetic."""
    if n == 0:
        return 0.0
    s = -1 if n < 0 else 1
    a = abs(n)
    e = a.bit_length() - 24
    if e <= 0:
        return float(s * a)
    q, r = divmod(a, 1 << e)
    half = 1 << (e - 1)
    if r > half or (r == half and (q & 1)):
        q += 1
    return float(s * q * (1 << e))


def test_int_to_float32_single_rounding():
    """RN32(int64) in the oracle is ONE rounding (a double rounding via f64 would differ here)."""
    cases = [(1 << 62) + (1 << 38) + 1, (1 << 40) + (1 << 16) + 1, -((1 << 55) + (1 << 31) + 1),
             (1 << 24) + 1, (1 << 24) + 3, 123456789012345, -98765432109876]
    rng = np.random.default_rng(0)
    cases += [int(v) for v in rng.integers(-(1 << 62), 1 << 62, size=2000)]
    X = np.array(cases, dtype=np.int64)
    got = ref.rn_float32_from_int(X)
    want = np.array([_exact_rn_f32(c) for c in cases], dtype=np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def _fwht_int(A):
    """Independent in-place integer butterfly (order-free because integer addition is exact)."""
    X = A.copy()
    D = X.shape[-1]
    h = 1
    while h < D:
        X = X.reshape(*X.shape[:-1], D // (2 * h), 2, h)
        a = X[..., 0, :].copy()
        b = X[..., 1, :].copy()
        X[..., 0, :] = a + b
        X[..., 1, :] = a - b
        X = X.reshape(*X.shape[:-3], D)
        h *= 2
    return X


def test_pinned_transform_integer_core_is_order_free():
    """A @ H_pm (O(n^2)) equals the butterfly FWHT bit for bit (pinned exactness, reading R10)."""
    rng = np.random.default_rng(2)
    A = rng.integers(-(1 << 40), 1 << 40, size=(500, 128), dtype=np.int64)
    assert np.array_equal(A @ ref.hadamard_pm(128), _fwht_int(A))


def test_pinned_transform_close_to_exact_transform():
    """Pinned x vs the exact real transform K diag(lambda)^-1 H: error within the fixed-point bound
    (64 half-units of 2^-24 over 128 addends, / sqrt(128)) plus three fp32 roundings."""
    K = synth.gen_keys(512, 1, 128, seed=4)[0, :, 0, :]
    lam, inv = ref.calibrate_smooth(K[:, None, :])
    x = ref.transform_key_pinned(K, inv[0]).astype(np.float64)
    exact = (K.astype(np.float64) * inv[0].astype(np.float64)) @ ref.hadamard(128)
    bound = 64 * 2.0 ** -24 / math.sqrt(128) + 4 * 2.0 ** -24 * np.abs(exact)
    assert np.all(np.abs(x - exact) <= bound + 1e-30)


def test_inv_sqrt_d_constant(golden):
    got = np.float32(1.0 / math.sqrt(128)).view(np.uint32)
    assert int(got) == int(golden["inv_sqrt_128_f32_bits"]["value"], 16)


def test_pinned_transform_range_guard():
    k = np.zeros((1, 128), dtype=np.float32)
    k[0, 0] = 2.0 ** 33
    with pytest.raises(OverflowError):
        ref.transform_key_pinned(k, np.ones(128, dtype=np.float32))


# ------------------------------------------------------------------------------ VQ, Eq. 2
def test_encode_worked_examples(golden):
    for key in ("encode_nearest", "encode_tie"):
        ex = golden[key]
        C = np.array(ex["centroids"], dtype=np.float32)
        assert ref.vq_encode(np.array([ex["x"]], dtype=np.float32), C)[0, 0] == ex["code"]


@pytest.mark.parametrize("n_levels", [2, 4, 16])
def test_encode_product_grid_closed_form(n_levels):
    """Product-grid codebook (2^4 / 4^4 / 16^4 entries): squared L2 is separable, so the nearest
    centroid is the per-dimension nearest level; with dyadic data every fp32 op is exact, ties are
    genuine, and the lowest index = the lowest digit in each tied dimension."""
    cb = synth.product_grid_codebook(n_levels, 4, step=0.5)
    n = 300 if n_levels == 16 else 3000
    X = synth.dyadic_points(n, 4, n_levels, 0.5, seed=n_levels)
    lv = synth.grid_levels(n_levels, 0.5)
    dist = np.abs(X[:, :, None].astype(np.float64) - lv[None, None, :])
    digit = np.argmin(dist, axis=2)                      # first (lowest) level on ties
    want = (digit * (n_levels ** np.arange(4))[None, :]).sum(1)
    got = ref.vq_encode(X.reshape(n, 4), cb)[:, 0]
    assert np.array_equal(got, want)
    # the test data really contains ties
    srt = np.sort(dist, axis=2)
    assert np.any(srt[:, :, 0] == srt[:, :, 1])


def test_encode_is_nearest_within_fp32_error():
    """For random data the chosen centroid's EXACT distance is within fp32 evaluation error of the
    exact minimum (Eq. 2 with the rounding of reading R9)."""
    rng = np.random.default_rng(5)
    C = synth.gen_codebook(256, 4, seed=6)
    X = rng.standard_normal((400, 4)).astype(np.float32)
    codes = ref.vq_encode(X, C)[:, 0]
    d = ((X[:, None, :].astype(np.float64) - C[None].astype(np.float64)) ** 2).sum(2)
    chosen = d[np.arange(400), codes]
    assert np.all(chosen <= d.min(1) * (1 + 8 * 2.0 ** -24) + 1e-30)


def test_encode_fixed_point_and_idempotence():
    """decode(encode(X)) = X when every sub-vector is a centroid; encode(decode(encode)) =
    encode."""
    C = synth.gen_codebook(256, 4, seed=7)
    codes = np.random.default_rng(8).integers(0, 256, size=(50, 32))
    X = ref.vq_decode(codes, C).astype(np.float32)
    c2 = ref.vq_encode(X, C)
    assert np.array_equal(ref.vq_decode(c2, C), X.astype(np.float64))
    Y = np.random.default_rng(9).standard_normal((50, 128)).astype(np.float32)
    e1 = ref.vq_encode(Y, C)
    assert np.array_equal(ref.vq_encode(ref.vq_decode(e1, C).astype(np.float32), C), e1)


def test_decode_examples():
    C = np.arange(8, dtype=np.float64).reshape(4, 2)
    assert np.array_equal(ref.vq_decode(np.array([[1, 0]]), C), [[2, 3, 0, 1]])
    assert np.array_equal(ref.vq_decode(np.zeros((2, 3), dtype=int), C), np.tile(C[0], (2, 3)))


def test_encode_kv_values_untransformed():
    """Eq. 8: values are VQ'd raw; keys after the dual transform."""
    k = synth.gen_keys(16, 1, 128, seed=1)[0, :, 0]
    v = synth.gen_values(16, 1, 128, seed=2)[0, :, 0]
    _, inv = ref.calibrate_smooth(k[:, None, :])
    C = synth.gen_codebook(256, 4, seed=3)
    kc, vc = ref.encode_kv(k, v, inv[0], C, C)
    assert np.array_equal(vc, ref.vq_encode(v, C))
    assert np.array_equal(kc, ref.vq_encode(ref.transform_key_pinned(k, inv[0]), C))


# ----------------------------------------------------------------- attention, Eq. 1 and Eq. 10
def test_attention_full_matches_library_softmax():
    """Eq. 1 special case: oracle softmax attention vs scipy.special.softmax / logsumexp."""
    rng = np.random.default_rng(10)
    q, K, V = rng.standard_normal((4, 128)), rng.standard_normal((300, 128)), rng.standard_normal((300, 128))
    o, L = ref.attention_full(q, K, V)
    s = q @ K.T / math.sqrt(128)
    assert np.allclose(o, scipy.special.softmax(s, axis=1) @ V, rtol=1e-12, atol=1e-14)
    assert np.allclose(L, scipy.special.logsumexp(s, axis=1), rtol=1e-14)


def test_attention_special_cases():
    """N = 1 -> o = v, L = s_1; identical keys -> mean of V, L = s + ln N;
    two equal scores -> (v1 + v2)/2; empty -> (0, -inf)."""
    rng = np.random.default_rng(11)
    q = rng.standard_normal((2, 64))
    k = rng.standard_normal((1, 64))
    v = rng.standard_normal((1, 64))
    o, L = ref.attention_full(q, k, v)
    assert np.allclose(o, np.repeat(v, 2, 0)) and np.allclose(L, (q @ k.T)[:, 0] / 8.0)
    K = np.repeat(k, 7, 0)
    V = rng.standard_normal((7, 64))
    o, L = ref.attention_full(q, K, V)
    assert np.allclose(o, V.mean(0)[None].repeat(2, 0)) and np.allclose(L, (q @ k.T)[:, 0] / 8 + math.log(7))
    o, L = ref.attention_full(q, np.zeros((0, 64)), np.zeros((0, 64)))
    assert np.all(o == 0) and np.all(np.isneginf(L))


def test_vq_attention_equals_full_precision_attention_on_reconstructed_keys():
    """Identity/exhaustive-codebook pin (north_star): when every transformed key
    sub-vector is a codebook entry, VQ attention (Eq. 10) equals Eq. 1 attention on the
    ORIGINAL keys K = K~ H^T diag(lambda), via the Eq. 7 invariance, to 1e-10."""
    rng = np.random.default_rng(12)
    D, N, G = 128, 200, 4
    Ck = synth.gen_codebook(256, 4, seed=13)
    Cv = synth.gen_codebook(256, 4, seed=14)
    kc = rng.integers(0, 256, (N, 32))
    vc = rng.integers(0, 256, (N, 32))
    lam = np.exp(rng.uniform(-1, 1, D))
    q = rng.standard_normal((G, D))
    K_orig = ref.vq_decode(kc, Ck) @ ref.hadamard(D).T * lam[None]      # invert Eq. 7's K~
    V = ref.vq_decode(vc, Cv)
    o1, L1 = ref.attention_vq(q, lam, Ck, Cv, kc, vc)
    o2, L2 = ref.attention_full(q, K_orig, V)
    assert np.max(np.abs(o1 - o2)) <= 1e-10 * np.max(np.abs(o2))
    assert np.max(np.abs(L1 - L2)) <= 1e-10 * np.max(np.abs(L2))


def test_lut_identity_and_example(golden):
    """Alg. 1 l.4: lut example and sum_m lut[m][code_m] = q~ . decode(codes)."""
    ex = golden["lut_example"]
    lut = ref.build_lut(np.array(ex["q_tilde"], dtype=float), np.array(ex["centroids"], dtype=float))
    assert np.allclose(lut[0], ex["lut"])
    rng = np.random.default_rng(15)
    C = synth.gen_codebook(256, 4, seed=16)
    qt = rng.standard_normal(128)
    codes = rng.integers(0, 256, (10, 32))
    lut = ref.build_lut(qt, C)
    s_lut = lut[np.arange(32)[None, :], codes].sum(1)
    assert np.allclose(s_lut, ref.vq_decode(codes, C) @ qt, rtol=1e-12)


# ------------------------------------------------------------------------ split / LSE merge
def test_merge_identities():
    """single partial -> itself; two identical -> o, L + ln 2; -inf neutral;
    all -inf -> (0, -inf)."""
    rng = np.random.default_rng(17)
    o = rng.standard_normal((1, 3, 8))
    L = rng.standard_normal((1, 3))
    mo, mL = ref.merge_lse(o, L)
    assert np.allclose(mo, o[0]) and np.allclose(mL, L[0])
    mo, mL = ref.merge_lse(np.concatenate([o, o]), np.concatenate([L, L]))
    assert np.allclose(mo, o[0]) and np.allclose(mL, L[0] + math.log(2))
    mo, mL = ref.merge_lse(np.concatenate([o, 5 + o]), np.concatenate([L, np.full_like(L, -np.inf)]))
    assert np.allclose(mo, o[0]) and np.allclose(mL, L[0])
    mo, mL = ref.merge_lse(o, np.full_like(L, -np.inf))
    assert np.all(mo == 0) and np.all(np.isneginf(mL))


@pytest.mark.parametrize("cuts", [[0, 100, 300], [0, 1, 2, 299, 300], [0, 150, 150, 300]])
def test_split_merge_equals_unsplit(cuts):
    """Split-KV + merge = unsplit attention (exactness of the online-softmax recurrence,
    P:745-757), including an empty split."""
    rng = np.random.default_rng(18)
    q, K, V = rng.standard_normal((4, 64)), rng.standard_normal((300, 64)), rng.standard_normal((300, 64))
    parts = [ref.attention_full(q, K[a:b], V[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    mo, mL = ref.merge_lse(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]))
    o, L = ref.attention_full(q, K, V)
    assert np.allclose(mo, o, rtol=1e-12, atol=1e-14) and np.allclose(mL, L, rtol=1e-13)


def test_attention_decode_batch_gqa_and_ranges():
    """GQA (query head i -> KV head i // G) and shard ranges [begin, min(end, len))."""
    rng = np.random.default_rng(19)
    B, Hkv, G, n_cap = 2, 2, 4, 64
    Ck = np.stack([synth.gen_codebook(256, 4, seed=s) for s in (1, 2)])
    Cv = np.stack([synth.gen_codebook(256, 4, seed=s) for s in (3, 4)])
    kc = rng.integers(0, 256, (B, Hkv, n_cap, 32))
    vc = rng.integers(0, 256, (B, Hkv, n_cap, 32))
    lam = np.exp(rng.uniform(-1, 1, (Hkv, 128)))
    q = rng.standard_normal((B, Hkv * G, 128))
    lens = [40, 64]
    o, L = ref.attention_decode_batch(q, lam, Ck, Cv, kc, vc, lens)
    oo, LL = ref.attention_vq(q[1, 5:6], lam[1], Ck[1], Cv[1], kc[1, 1, :64], vc[1, 1, :64])
    assert np.allclose(o[1, 5], oo[0]) and np.isclose(L[1, 5], LL[0])
    parts = [ref.attention_decode_batch(q, lam, Ck, Cv, kc, vc, lens, a, b) for a, b in ((0, 30), (30, 1000))]
    mo, mL = ref.merge_lse(np.stack([parts[0][0], parts[1][0]]), np.stack([parts[0][1], parts[1][1]]))
    assert np.allclose(mo, o) and np.allclose(mL, L)


# ------------------------------------------------------------------------- byte accounting
def test_memory_formulas(golden):
    for key in ("memory_d4b8", "memory_d8b12"):
        ex = golden[key]
        assert ref.codebook_bytes(ex["sub_dim"], ex["code_bits"]) == ex["codebook_bytes"]
        assert ref.index_bytes_per_vector(ex["head_dim"], ex["sub_dim"], ex["code_bits"]) == ex["index_bytes"]
    ab = golden["avg_bits"]
    assert ref.avg_bits(4, 8) == ab["d4b8"] and ref.avg_bits(8, 12) == ab["d8b12"]
    assert (ref.avg_bits(8, 12) + ref.avg_bits(8, 8)) / 2 == ab["K_d8b12_V_d8b8"]


@pytest.mark.parametrize("bits", [4, 8, 16])
def test_pack_roundtrip_and_order(bits):
    rng = np.random.default_rng(bits)
    codes = rng.integers(0, 1 << bits, (3, 5, 32))
    packed = ref.pack_codes(codes, bits)
    assert packed.shape[-1] == 32 * bits // 8
    assert np.array_equal(ref.unpack_codes(packed, bits), codes)
    if bits == 4:
        assert packed[0, 0, 0] == codes[0, 0, 0] | (codes[0, 0, 1] << 4)
    if bits == 16:
        assert packed[0, 0, 0] == codes[0, 0, 0] & 0xFF and packed[0, 0, 1] == codes[0, 0, 0] >> 8


def test_pack_bitstream_hand_examples():
    """Reading R11 for non-byte-aligned codes, worked by hand: b = 10 codes 0x3FF, 0x001, 0x155,
    0x2AA occupy row bits 0-9, 10-19, 20-29, 30-39 -> bytes FF 07 50 95 AA; b = 12 codes 0xABC,
    0x123 -> the 24-bit value 0x123ABC little-endian -> BC 3A 12."""
    assert ref.pack_codes(np.array([[0x3FF, 0x001, 0x155, 0x2AA]]), 10).tolist() == [[0xFF, 0x07, 0x50, 0x95, 0xAA]]
    assert ref.pack_codes(np.array([[0xABC, 0x123]]), 12).tolist() == [[0xBC, 0x3A, 0x12]]
    assert ref.unpack_codes(np.array([[0xBC, 0x3A, 0x12]], np.uint8), 12).tolist() == [[0xABC, 0x123]]


@pytest.mark.parametrize("bits", [4, 8, 16])
def test_pack_byte_widths_are_the_bitstream(bits):
    """The 4/8/16-bit branches of pack_codes (written separately) are special cases of the
    bit-by-bit rule (same bytes both ways)."""
    codes = np.random.default_rng(40 + bits).integers(0, 1 << bits, (4, 32))
    assert np.array_equal(ref.pack_codes(codes, bits), ref.pack_bitstream(codes, bits))
    assert np.array_equal(ref.unpack_bitstream(ref.pack_codes(codes, bits), bits), codes)


@pytest.mark.parametrize("sub_dim,bits", [(4, 10), (8, 12), (8, 8), (2, 8), (8, 16)])
def test_pack_roundtrip_next2_formats(sub_dim, bits):
    """d4b10 / d8b12 / d8b8 / d2b8 rows: M = 128/d codes, M*b/8 bytes
    (P:143), lossless."""
    M = 128 // sub_dim
    codes = np.random.default_rng(sub_dim * bits).integers(0, 1 << bits, (3, 2, M))
    packed = ref.pack_codes(codes, bits)
    assert packed.shape[-1] == ref.index_bytes_per_vector(128, sub_dim, bits)
    assert np.array_equal(ref.unpack_codes(packed, bits), codes)
    extremes = np.full((1, M), (1 << bits) - 1)
    assert np.all(ref.pack_codes(extremes, bits) == 0xFF) and np.all(ref.pack_codes(0 * extremes, bits) == 0)


@pytest.mark.parametrize("sub_dim,n_levels", [(8, 2), (2, 16), (8, 3), (8, 4)])
def test_encode_product_grid_other_sub_dims(sub_dim, n_levels):
    """Eq. 2 with d = 8 (2^8, 3^8 = 6561 and 4^8 = 65 536 entries: the d8b16 size) and
    d = 2 (16^2): the separable closed form of test_encode_product_grid_closed_form at the other
    sub-vector sizes."""
    cb = synth.product_grid_codebook(n_levels, sub_dim, step=0.5)
    n = 400
    X = synth.dyadic_points(n, sub_dim, n_levels, 0.5, seed=sub_dim * 7 + n_levels)
    lv = synth.grid_levels(n_levels, 0.5)
    dist = np.abs(X[:, :, None].astype(np.float64) - lv[None, None, :])
    digit = np.argmin(dist, axis=2)
    want = (digit * (n_levels ** np.arange(sub_dim))[None, :]).sum(1)
    got = ref.vq_encode(X.reshape(n, sub_dim), cb)[:, 0]
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dk,nk,dv,nv", [(8, 4096, 8, 256), (4, 1024, 2, 256), (8, 65536, 8, 65536)])
def test_vq_attention_identity_other_formats(dk, nk, dv, nv):
    """The exhaustive-codebook identity pin at K-d8b12 / V-d8b8 and K-d4b10 / V-d2b8 (Table 3
    mixed configurations): Eq. 10 over codes = Eq. 1 over the reconstructed keys."""
    rng = np.random.default_rng(dk * 100 + dv)
    D, N, G = 128, 150, 4
    Ck = synth.gen_codebook(nk, dk, seed=15)
    Cv = synth.gen_codebook(nv, dv, seed=16)
    kc = rng.integers(0, nk, (N, D // dk))
    vc = rng.integers(0, nv, (N, D // dv))
    lam = np.exp(rng.uniform(-1, 1, D))
    q = rng.standard_normal((G, D))
    K_orig = ref.vq_decode(kc, Ck) @ ref.hadamard(D).T * lam[None]
    o1, L1 = ref.attention_vq(q, lam, Ck, Cv, kc, vc)
    o2, L2 = ref.attention_full(q, K_orig, ref.vq_decode(vc, Cv))
    assert np.max(np.abs(o1 - o2)) <= 1e-10 * np.max(np.abs(o2))
    assert np.max(np.abs(L1 - L2)) <= 1e-10 * np.max(np.abs(L2))


# ------------------------------------------------------------------------- k-means (harness)
def test_kmeans_examples(golden):
    ex = golden["kmeans_example"]
    C, hist = ref.kmeans(np.array(ex["points"], dtype=float), 2, seed=0)
    got = sorted(map(tuple, np.round(C, 9)))
    assert got == sorted(map(tuple, ex["centroids"]))
    C2, _ = ref.kmeans(np.array([[0, 0], [10, 10]], dtype=float), 2, seed=1)
    assert sorted(map(tuple, C2)) == [(0, 0), (10, 10)]
    X = np.random.default_rng(0).standard_normal((2000, 4))
    Ca, ha = ref.kmeans(X, 16, seed=3)
    Cb, hb = ref.kmeans(X, 16, seed=3)
    assert np.array_equal(Ca, Cb)                                  # deterministic
    assert all(b <= a + 1e-9 for a, b in zip(ha, ha[1:]))          # objective non-increasing
    assert len(ha) <= 30                                           # P:501 iteration cap


def test_kmeans_lloyd_step_worked_example(golden):
    """SPEC S:133 worked example through ONE pinned Lloyd step: from C0 = {(0,0), (10,10)}
    the points {(0,0), (0,1), (10,10), (10,11)} split 2/2 and the means are the brute-force optimal
    2-means {(0, 0.5), (10, 10.5)}; best distances 0, 1, 0, 1; objective 2."""
    ex = golden["kmeans_example"]
    X = np.array(ex["points"], dtype=np.float32)
    C, a, best, cnt, obj = ref.kmeans_lloyd_step(X, np.array([[0, 0], [10, 10]], dtype=np.float32))
    assert np.array_equal(C, np.array(ex["centroids"], dtype=np.float32))
    assert a.tolist() == [0, 0, 1, 1] and cnt.tolist() == [2, 2]
    assert best.tolist() == [0.0, 1.0, 0.0, 1.0] and obj == 2.0


def test_kmeans_lloyd_step_reseeds_empty_clusters():
    """an empty cluster is re-seeded at the point of largest distortion, ties to the
    lowest point index; several empty clusters (increasing index) take successive worst points.
    Hand-worked: best = [0, 1, 0, 1, 4] -> empty clusters 2, 3 take points 4 (best 4) and 1 (best 1,
    lower index than point 3)."""
    X = np.array([[0, 0], [0, 1], [10, 10], [10, 11], [0, -2]], dtype=np.float32)
    C0 = np.array([[0, 0], [10, 10], [500, 500], [-500, 9]], dtype=np.float32)
    C, a, best, cnt, _ = ref.kmeans_lloyd_step(X, C0)
    assert best.tolist() == [0.0, 1.0, 0.0, 1.0, 4.0] and cnt.tolist() == [3, 2, 0, 0]
    assert np.array_equal(C[0], np.array([0, -1 / 3], dtype=np.float32))   # RN32 of the exact mean
    assert np.array_equal(C[2], X[4]) and np.array_equal(C[3], X[1])


def test_kmeans_lloyd_step_exact_means_and_ties():
    """Closed form: points c_j + delta with the deltas of each cluster summing to zero (dyadic, so
    every op is exact) -> C' = the generating centres exactly; a point at the exact midpoint of two
    centroids (a genuine tie of the pinned distance) goes to the lower index."""
    rng = np.random.default_rng(5)
    centres = (rng.integers(-40, 40, size=(16, 4)) * 8).astype(np.float32)
    deltas = rng.integers(-3, 4, size=(16, 6, 4)).astype(np.float32) * 0.25
    deltas -= deltas.mean(axis=1, keepdims=True)                             # zero-sum per cluster
    X = (centres[:, None, :] + deltas).reshape(-1, 4).astype(np.float32)
    assert np.all(np.abs(X - (centres[:, None, :] + deltas).reshape(-1, 4)) == 0)
    C, a, _, cnt, _ = ref.kmeans_lloyd_step(X, centres)
    assert np.array_equal(cnt, np.full(16, 6)) and np.array_equal(C, centres)
    assert np.array_equal(a, np.repeat(np.arange(16), 6))
    tie = np.array([[1.0, 0, 0, 0]], dtype=np.float32)
    for C2 in (np.array([[0, 0, 0, 0], [2, 0, 0, 0]], np.float32), np.array([[2, 0, 0, 0], [0, 0, 0, 0]], np.float32)):
        _, a2, b2, _, _ = ref.kmeans_lloyd_step(np.repeat(tie, 2, 0), C2)
        assert a2.tolist() == [0, 0] and b2.tolist() == [1.0, 1.0]


def test_kmeans_lloyd_step_fixed_point_and_descent():
    """Invariants of Lloyd's algorithm: a codebook holding every distinct point is a fixed point
    with objective 0; iterating from any start never increases the objective (up to fp32 rounding
    of the pinned distances, 1e-6 relative)."""
    rng = np.random.default_rng(9)
    pts = rng.standard_normal((32, 4)).astype(np.float32)
    X = np.repeat(pts, 3, axis=0)
    C, _, _, _, obj = ref.kmeans_lloyd_step(X, pts)
    assert np.array_equal(C, pts) and obj == 0.0
    X = rng.standard_normal((3000, 4)).astype(np.float32)
    C = X[rng.choice(3000, 64, replace=False)].copy()
    objs = []
    for _ in range(8):
        C, _, _, _, obj = ref.kmeans_lloyd_step(X, C)
        objs.append(obj)
    assert all(b <= a * (1 + 1e-6) for a, b in zip(objs, objs[1:]))


# ------------------------------------------------------------ residual window (NEXT-1)
def test_residual_window_special_cases():
    """Residual-window attention: empty residual == Eq. 10 VQ attention; empty VQ part == Eq. 1 on
    the residual; and in general == the LSE merge of the two separate attentions (exact algebra)."""
    rng = np.random.default_rng(40)
    Ck = synth.gen_codebook(256, 4, seed=41)
    Cv = synth.gen_codebook(256, 4, seed=42)
    kc, vc = rng.integers(0, 256, (300, 32)), rng.integers(0, 256, (300, 32))
    lam = np.exp(rng.uniform(-1, 1, 128))
    q = rng.standard_normal((4, 128))
    Kr, Vr = rng.standard_normal((77, 128)), rng.standard_normal((77, 128))
    o0, L0 = ref.attention_vq_residual(q, lam, Ck, Cv, kc, vc, Kr[:0], Vr[:0])
    o1, L1 = ref.attention_vq(q, lam, Ck, Cv, kc, vc)
    assert np.allclose(o0, o1, rtol=1e-12) and np.allclose(L0, L1, rtol=1e-12)
    o0, L0 = ref.attention_vq_residual(q, lam, Ck, Cv, kc[:0], vc[:0], Kr, Vr)
    o1, L1 = ref.attention_full(q, Kr, Vr)
    assert np.allclose(o0, o1, rtol=1e-12) and np.allclose(L0, L1, rtol=1e-12)
    o, L = ref.attention_vq_residual(q, lam, Ck, Cv, kc, vc, Kr, Vr)
    pa, pb = ref.attention_vq(q, lam, Ck, Cv, kc, vc), ref.attention_full(q, Kr, Vr)
    mo, mL = ref.merge_lse(np.stack([pa[0], pb[0]]), np.stack([pa[1], pb[1]]))
    assert np.allclose(o, mo, rtol=1e-12, atol=1e-14) and np.allclose(L, mL, rtol=1e-12)


def test_residual_window_equals_unquantised_keys_when_exact():
    """If the quantised tokens are exactly representable (codes decode to the transformed keys), the
    residual + VQ attention equals Eq. 1 over all ORIGINAL keys (invariance, Eq. 7)."""
    rng = np.random.default_rng(43)
    Ck = synth.gen_codebook(256, 4, seed=44)
    Cv = synth.gen_codebook(256, 4, seed=45)
    kc, vc = rng.integers(0, 256, (100, 32)), rng.integers(0, 256, (100, 32))
    lam = np.exp(rng.uniform(-1, 1, 128))
    q = rng.standard_normal((4, 128))
    Kq = ref.vq_decode(kc, Ck) @ ref.hadamard(128).T * lam[None]
    Kr, Vr = rng.standard_normal((20, 128)), rng.standard_normal((20, 128))
    o, L = ref.attention_vq_residual(q, lam, Ck, Cv, kc, vc, Kr, Vr)
    o2, L2 = ref.attention_full(q, np.concatenate([Kq, Kr]), np.concatenate([ref.vq_decode(vc, Cv), Vr]))
    assert np.allclose(o, o2, rtol=1e-10, atol=1e-12) and np.allclose(L, L2, rtol=1e-10)
