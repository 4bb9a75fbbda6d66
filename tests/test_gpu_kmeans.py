"""GPU codebook k-means (NEXT-3) against the oracle's pinned Lloyd step.

One vecinfer_kmeans_step must reproduce oracle.kmeans_lloyd_step from the same fp32 centroids:
assignments and best distances bit-exact (the encoder's pinned fp32 distance, lowest index on
ties), counts exact, re-seeded empty clusters exact, and the updated centroids within one fp32 ulp
of RN32(exact mean) (the GPU sums each cluster exactly in int64 fixed point on a 2^-e grid, so
the step is bitwise reproducible run to run; the grid rounding is the only difference).  Inputs follow the
codebook-fitting recipe: pinned-transformed synthetic keys (C_k) and raw values (C_v) split into
d-dim sub-vectors, plus dyadic tie cases and forced empty clusters.
"""
import numpy as np
import pytest

import synth
from oracle import ref
from helpers import load_codebooks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402
from paper_2510_06175_b200._lib import VecInferError  # noqa: E402

DEV = torch.device("cuda", 0)
CB = load_codebooks()


def _subvectors(n_tok, d, which, seed):
    """Training sub-vectors of one KV head: pinned-transformed keys (C_k) or raw values (C_v)."""
    if which == "k":
        k = synth.gen_keys(n_tok, 8, 128, seed=seed)[0, :, 3]
        x = ref.transform_key_pinned(k, CB["inv_lambda"][3])
    else:
        x = synth.gen_values(n_tok, 8, 128, seed=seed)[0, :, 3].astype(np.float32)
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32).reshape(-1, d))


def _gpu_step(X, C):
    Xd = torch.from_numpy(X).to(DEV)
    Cd = torch.from_numpy(C).to(DEV)
    Cn, a, b, obj = vi.kmeans_step(Xd, Cd)
    torch.cuda.synchronize()
    return Cn.cpu().numpy(), a.cpu().numpy(), b.cpu().numpy(), float(obj.item())


def _check(X, C):
    Cg, ag, bg, og = _gpu_step(X, C)
    Cr, ar, br, cr, orf = ref.kmeans_lloyd_step(X, C)
    assert np.array_equal(ag, ar.astype(np.int32)), "assignments differ from the oracle"
    assert np.array_equal(bg.view(np.uint32), br.view(np.uint32)), "best distances differ"
    assert np.array_equal(np.bincount(ag, minlength=C.shape[0]), cr)
    ulp = np.spacing(np.abs(Cr).astype(np.float32))
    assert np.all(np.abs(Cg.astype(np.float64) - Cr) <= ulp), "centroids beyond one fp32 ulp"
    assert abs(og - orf) <= 1e-9 * max(1.0, abs(orf))
    return Cr, cr


@pytest.mark.parametrize("which", ["k", "v"])
@pytest.mark.parametrize("d,k", [(4, 256), (4, 16), (2, 256), (8, 256)])
def test_kmeans_step_matches_oracle(which, d, k):
    X = _subvectors(160, d, which, seed=11 + d)          # 160 tokens x 128/d sub-vectors
    rng = np.random.default_rng(d * 1000 + k)
    C = X[rng.choice(X.shape[0], k, replace=False)].copy()
    Cr, cr = _check(X, C)
    Cr2, _ = _check(X, Cr)                                # a second iteration from the oracle's C'


def test_kmeans_step_large_codebook_chunks():
    """k = 65536 (b4d4-sized): the centroids are staged through shared memory in chunks."""
    X = _subvectors(600, 4, "k", seed=3)                  # 19 200 + 51 200 sub-vectors >= k
    X = np.concatenate([X, _subvectors(1600, 4, "v", seed=4)])
    C = np.ascontiguousarray(CB["ck_b4d4"].astype(np.float32))       # [65536, 4] product grid
    _check(X, C)


def test_kmeans_step_ties_and_empty_clusters():
    """Genuine ties of the pinned distance (dyadic midpoints) go to the lower index; far-away
    centroids get no points and are re-seeded at the worst points (ties: lowest point index)."""
    rng = np.random.default_rng(2)
    grid = (rng.integers(-8, 8, size=(4000, 4)) * 0.5).astype(np.float32)
    C = np.concatenate([(rng.integers(-4, 4, size=(60, 4)) * 1.0).astype(np.float32),
                        np.full((4, 4), 1000.0, np.float32) + np.arange(4, dtype=np.float32)[:, None]])
    Cr, cr = _check(grid, C)
    assert (cr == 0).sum() >= 4


def test_kmeans_fit_descends_like_the_oracle():
    """Lloyd iterations (<= 30) from the same start: the objective never increases and the
    final objective matches the oracle's iterated steps within 1e-4 (trajectories may differ only
    through last-ulp centroid differences)."""
    X = _subvectors(256, 4, "k", seed=21)
    rng = np.random.default_rng(1)
    C0 = X[rng.choice(X.shape[0], 64, replace=False)].copy()
    Cg, hist = vi.kmeans_fit(torch.from_numpy(X).to(DEV), torch.from_numpy(C0).to(DEV), max_iters=12)
    assert all(b <= a * (1 + 1e-6) for a, b in zip(hist, hist[1:]))
    C, objs = C0, []
    for _ in range(len(hist)):
        C, _, _, _, o = ref.kmeans_lloyd_step(X, C)
        objs.append(o)
    assert abs(hist[-1] - objs[-1]) <= 1e-4 * objs[-1]


def test_kmeans_step_rejects_bad_arguments():
    X = torch.zeros(10, 4, device=DEV)
    with pytest.raises(VecInferError):
        vi.kmeans_step(X, torch.zeros(16, 4, device=DEV))        # n < k
    with pytest.raises(VecInferError):
        vi.kmeans_step(torch.zeros(40, 3, device=DEV), torch.zeros(4, 3, device=DEV))   # d = 3


@pytest.mark.parametrize("d,k", [(4, 256), (2, 256), (8, 4096)])
def test_kmeans_step_bitwise_reproducible(d, k):
    """SPEC S:128 / S:187 determinism: the same step twice gives bitwise identical centroids and
    objective (integer fixed-point sums; the atomics' landing order cannot change them)."""
    X = _subvectors(8192 * 8 // d, d, "k", seed=901)
    rng = np.random.default_rng(902)
    C = X[rng.choice(X.shape[0], size=k, replace=False)].copy()
    r1 = _gpu_step(X, C)
    r2 = _gpu_step(X, C)
    assert np.array_equal(r1[0].view(np.uint32), r2[0].view(np.uint32))
    assert np.array_equal(r1[1], r2[1]) and r1[3] == r2[3]
