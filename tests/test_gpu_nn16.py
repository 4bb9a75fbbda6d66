"""16-bit codebooks (65 536 entries): the tensor-core filter + exact selection of encode_kv.

The filter (mma.sync bf16 over a_j = ||c_j||^2 - 2 x.c_j) only decides WHICH 512-centroid chunks
are scanned with the pinned distance (R9); codes must stay bit-identical to the oracle's
full scan, lowest index on ties.  The cases target the filter's weak spots: near-ties (points a
hair from a centroid, so D_min << ||x||^2 and the ranking hangs on cancellation), exact
real-arithmetic ties between two centroids, inputs far outside the book's range, per-head books,
several passes of the workspace, head_dim 64, and the full-scan path kept behind
VECINFER_NN16_SCAN=1 as the A/B reference.
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
from test_gpu_parity import _encode_gpu, _encode_ref, t_bf16  # noqa: E402

CB = load_codebooks()
B4D4_64 = vi.VQConfig(64, 4, 16)


def _random_book(seed, n=65536, scale=1.0, heads=None):
    shape = (n, 4) if heads is None else (heads, n, 4)
    return synth.round_to_bf16(np.random.default_rng(seed).normal(0, scale, shape).astype(np.float32))


def test_nn16_per_head_books_several_passes():
    """Per-head K books (8 x 65 536 random bf16 centroids) and one shared V book; B*T*H = 520
    token-heads = two workspace passes (~512 token-heads each)."""
    H, T = 8, 65
    k = synth.gen_keys(T, H, 128, seed=1600)
    v = synth.gen_values(T, H, 128, seed=1601)
    ck = _random_book(1602, heads=H)
    cv = CB["cv_b4d4"]
    got = _encode_gpu(k, v, CB["inv_lambda"], ck, cv, T + 3, [3], vi.B4D4, vi.B4D4)
    want = _encode_ref(k, v, CB["inv_lambda"], ck, cv, T + 3, [3], vi.B4D4, vi.B4D4)
    assert np.array_equal(got[0], want[0]), "key codes differ"
    assert np.array_equal(got[1], want[1]), "value codes differ"


@pytest.mark.parametrize("eps", [0.0, 1e-7, 1e-5, 1e-3])
def test_nn16_points_next_to_centroids(eps):
    """Values = a centroid + eps noise (untransformed V path): D_min is ~eps^2 while ||x||^2 is
    O(1), the cancellation regime of a_j = ||c||^2 - 2 x.c.  eps = 0 gives exact hits (and the
    lowest index among duplicate centroids)."""
    cv = _random_book(1610)
    cv[7] = cv[40000]                                    # a duplicate centroid: lowest index wins
    rng = np.random.default_rng(1611)
    T = 6
    idx = rng.integers(0, 65536, size=(T, 32))
    idx[0, :4] = 40000
    pts = cv[idx].reshape(1, T, 1, 128) + eps * rng.standard_normal((1, T, 1, 128)).astype(np.float32)
    pts = synth.round_to_bf16(pts.astype(np.float32))
    k = np.zeros_like(pts)
    got = _encode_gpu(k, pts, np.ones((1, 128), np.float32), CB["ck_b4d4"], cv, T, [0], vi.B4D4, vi.B4D4)
    want = _encode_ref(k, pts, np.ones((1, 128), np.float32), CB["ck_b4d4"], cv, T, [0], vi.B4D4, vi.B4D4)
    assert np.array_equal(got[1], want[1])
    if eps == 0.0:
        codes = ref.unpack_codes(got[1][0, 0, 0], 16)
        assert codes[0] == 7                             # cv[7] == cv[40000]: the lower index


def test_nn16_midpoint_ties():
    """Points exactly halfway between two centroids that differ in one coordinate by a power of
    two: equal distances in real arithmetic; the pinned fp32 distance (or the index) decides."""
    cv = _random_book(1620)
    rng = np.random.default_rng(1621)
    T = 4
    pts = np.zeros((T * 32, 4), np.float32)
    for i in range(T * 32):
        j1 = int(rng.integers(0, 65536))
        j2 = int(rng.integers(0, 65536))
        c = cv[j1].copy()
        dim = int(rng.integers(0, 4))
        c[dim] = cv[j1, dim] + np.float32(0.25)       # a second centroid 0.25 away in one dimension
        cv[j2] = synth.round_to_bf16(c)
        pts[i] = (cv[j1].astype(np.float64) + cv[j2].astype(np.float64)) / 2
    pts = synth.round_to_bf16(pts.reshape(1, T, 1, 128))   # (the kernel reads bf16 inputs)
    k = np.zeros_like(pts)
    got = _encode_gpu(k, pts, np.ones((1, 128), np.float32), CB["ck_b4d4"], cv, T, [0], vi.B4D4, vi.B4D4)
    want = _encode_ref(k, pts, np.ones((1, 128), np.float32), CB["ck_b4d4"], cv, T, [0], vi.B4D4, vi.B4D4)
    assert np.array_equal(got[1], want[1])


@pytest.mark.parametrize("scale", [1e-3, 40.0])
def test_nn16_inputs_outside_the_book_range(scale):
    """Keys far larger / smaller than the centroids (the error bounds scale with ||x||_1 max|c|)."""
    T = 5
    k = synth.round_to_bf16((synth.gen_keys(T, 2, 128, seed=1630) * scale).astype(np.float32))
    v = synth.round_to_bf16((synth.gen_values(T, 2, 128, seed=1631) * scale).astype(np.float32))
    got = _encode_gpu(k, v, CB["inv_lambda"][:2], CB["ck_b4d4"], CB["cv_b4d4"], T, [0], vi.B4D4, vi.B4D4)
    want = _encode_ref(k, v, CB["inv_lambda"][:2], CB["ck_b4d4"], CB["cv_b4d4"], T, [0], vi.B4D4, vi.B4D4)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("kcfg,vcfg", [(vi.B4D4, vi.B2D4), (vi.B1D4, vi.B4D4)])
def test_nn16_mixed_with_small_books(kcfg, vcfg):
    T = 9
    k = synth.gen_keys(T, 3, 128, seed=1640, batch=2)
    v = synth.gen_values(T, 3, 128, seed=1641, batch=2)
    name = {4: "b1d4", 8: "b2d4", 16: "b4d4"}
    ck = CB[f"ck_{name[kcfg.code_bits]}"]
    cv = CB[f"cv_{name[vcfg.code_bits]}"]
    ck = ck if ck.ndim == 2 else ck[:3]
    cv = cv if cv.ndim == 2 else cv[:3]
    got = _encode_gpu(k, v, CB["inv_lambda"][:3], ck, cv, T + 2, [2, 0], kcfg, vcfg)
    want = _encode_ref(k, v, CB["inv_lambda"][:3], ck, cv, T + 2, [2, 0], kcfg, vcfg)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_nn16_head_dim_64():
    T = 7
    k = synth.gen_keys(T, 4, 64, seed=1650)
    v = synth.gen_values(T, 4, 64, seed=1651)
    inv = CB["inv_lambda"][:4, :64].copy()
    got = _encode_gpu(k, v, inv, CB["ck_b4d4"], CB["cv_b4d4"], T, [0], B4D4_64, B4D4_64)
    want = _encode_ref(k, v, inv, CB["ck_b4d4"], CB["cv_b4d4"], T, [0], B4D4_64, B4D4_64)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_nn16_workspace_left_zero():
    """The selection zeroes every (lo, hi) pair the filter wrote: a zero-filled workspace stays
    zero (decode_step places it next to the attention workspace, which must stay zero)."""
    T, H = 3, 8
    k = synth.gen_keys(T, H, 128, seed=1660)
    v = synth.gen_values(T, H, 128, seed=1661)
    ws = vi.encode_workspace(1, T, H, vi.B4D4, vi.B4D4, device="cuda").zero_()
    kc = torch.zeros(1, H, T, 64, dtype=torch.uint8, device="cuda")
    vc = torch.zeros_like(kc)
    vi.encode_kv(t_bf16(k), t_bf16(v), torch.from_numpy(CB["inv_lambda"]).cuda(), t_bf16(CB["ck_b4d4"]),
                 t_bf16(CB["cv_b4d4"]), kc, vc, torch.zeros(1, dtype=torch.int32, device="cuda"), vi.B4D4, vi.B4D4,
                 workspace=ws)
    torch.cuda.synchronize()
    assert int(ws.count_nonzero().item()) == 0


def test_nn16_tcgen05_filter_variant():
    """The opt-in tcgen05 filter (VECINFER_NN16_TC=1: A tile in shared memory, two TMEM accumulators,
    tcgen05.mma kind::f16 bf16 -> fp32) runs every case of this file to the same oracle codes.  The
    switch is read once per process, hence the subprocess."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, VECINFER_NN16_TC="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", os.path.join(here, "test_gpu_nn16.py"),
                        "-k", "not tcgen05"], env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ---- d = 8 books (NEXT-2 d8b12: 4096 entries, d8b16: 65 536 entries): K = 32 filter, two chained MMAs
def _random_book8(seed, n, heads=None, scale=1.0):
    shape = (n, 8) if heads is None else (heads, n, 8)
    return synth.round_to_bf16(np.random.default_rng(seed).normal(0, scale, shape).astype(np.float32))


def test_nn_d8b12_per_head_books_several_passes():
    """Per-head 4096 x 8 K books and a shared V book, 65 tokens x 8 heads = two passes."""
    H, T = 8, 65
    k = synth.gen_keys(T, H, 128, seed=1700)
    v = synth.gen_values(T, H, 128, seed=1701)
    ck = _random_book8(1702, 4096, heads=H)
    cv = _random_book8(1703, 4096)
    got = _encode_gpu(k, v, CB["inv_lambda"], ck, cv, T + 2, [2], vi.D8B12, vi.D8B12)
    want = _encode_ref(k, v, CB["inv_lambda"], ck, cv, T + 2, [2], vi.D8B12, vi.D8B12)
    assert np.array_equal(got[0], want[0]), "key codes differ"
    assert np.array_equal(got[1], want[1]), "value codes differ"


@pytest.mark.parametrize("eps", [0.0, 1e-6, 1e-3])
def test_nn_d8b16_points_next_to_centroids(eps):
    cv = _random_book8(1710, 65536)
    cv[9] = cv[50000]                                     # duplicate: the lower index wins
    rng = np.random.default_rng(1711)
    T = 4
    idx = rng.integers(0, 65536, size=(T, 16))
    idx[0, :2] = 50000
    pts = cv[idx].reshape(1, T, 1, 128) + eps * rng.standard_normal((1, T, 1, 128)).astype(np.float32)
    pts = synth.round_to_bf16(pts.astype(np.float32))
    k = np.zeros_like(pts)
    got = _encode_gpu(k, pts, np.ones((1, 128), np.float32), cv, cv, T, [0], vi.D8B16, vi.D8B16)
    want = _encode_ref(k, pts, np.ones((1, 128), np.float32), cv, cv, T, [0], vi.D8B16, vi.D8B16)
    assert np.array_equal(got[1], want[1])
    if eps == 0.0:
        assert ref.unpack_codes(got[1][0, 0, 0], 16)[0] == 9


@pytest.mark.parametrize("kn,vn", [("d8b12", "d8b8"), ("d4b10", "d8b12"), ("d8b16", "d8b16")])
def test_nn_d8_mixed_pairs(kn, vn):
    """The paper's mixed pairs: the d8b12 / d8b16 stream through the filter, the other (d8b8 / d4b10)
    through the generic scan in its own launch."""
    cfg = {"d8b8": vi.D8B8, "d8b12": vi.D8B12, "d4b10": vi.D4B10, "d8b16": vi.D8B16}
    T = 6
    k = synth.gen_keys(T, 3, 128, seed=1720, batch=2)
    v = synth.gen_values(T, 3, 128, seed=1721, batch=2)
    ck, cv = CB[f"ck_{kn}"], CB[f"cv_{vn}"]
    ck = ck if ck.ndim == 2 else ck[:3]
    cv = cv if cv.ndim == 2 else cv[:3]
    got = _encode_gpu(k, v, CB["inv_lambda"][:3], ck, cv, T + 1, [1, 0], cfg[kn], cfg[vn])
    want = _encode_ref(k, v, CB["inv_lambda"][:3], ck, cv, T + 1, [1, 0], cfg[kn], cfg[vn])
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("fmt", ["b4d4", "d8b16"])
def test_nn_filter_paged_pool(fmt):
    """The filter path writes through the block table: paged prefill + 1-token append land at the
    translated rows with the oracle's codes; spare pages stay untouched."""
    from test_gpu_paged import _unpaginate
    cfg = {"b4d4": vi.B4D4, "d8b16": vi.D8B16}[fmt]
    B, H, ps, npb = 2, 4, 32, 3
    n_cap = ps * npb
    rng = np.random.default_rng(1730)
    n_pages = B * npb + 2
    bt = rng.permutation(n_pages)[:B * npb].reshape(B, npb).astype(np.int32)
    kpool = torch.zeros(n_pages, H, ps, cfg.row_bytes, dtype=torch.uint8, device="cuda")
    vpool = torch.zeros_like(kpool)
    T = 7
    k = synth.gen_keys(T, H, 128, seed=1731, batch=B)
    v = synth.gen_values(T, H, 128, seed=1732, batch=B)
    inv, ck, cv = CB["inv_lambda"][:H], CB[f"ck_{fmt}"], CB[f"cv_{fmt}"]
    wp = np.array([0, 40], np.int32)
    vi.encode_kv(t_bf16(k), t_bf16(v), torch.from_numpy(inv).cuda(), t_bf16(ck), t_bf16(cv), kpool, vpool,
                 torch.from_numpy(wp).cuda(), cfg, cfg, block_table=torch.from_numpy(bt).cuda())
    kc = _unpaginate(kpool.cpu().numpy(), bt, ps)
    vc = _unpaginate(vpool.cpu().numpy(), bt, ps)
    exp_k = np.zeros((B, H, n_cap, cfg.row_bytes), np.uint8)
    exp_v = np.zeros_like(exp_k)
    for b in range(B):
        for h in range(H):
            kk, vv = ref.encode_kv(k[b, :, h], v[b, :, h], inv[h], ck, cv)
            exp_k[b, h, wp[b]:wp[b] + T] = ref.pack_codes(kk, cfg.code_bits)
            exp_v[b, h, wp[b]:wp[b] + T] = ref.pack_codes(vv, cfg.code_bits)
    assert np.array_equal(kc, exp_k) and np.array_equal(vc, exp_v)
    spare = np.setdiff1d(np.arange(n_pages), bt.ravel())
    assert not kpool[torch.from_numpy(spare).cuda().long()].any()


def test_nn16_filter_matches_the_full_scan_at_scale():
    """Cross-check at a size the oracle cannot brute-force in seconds (4096 token-heads x 2 streams x
    32 sub-vectors against 65 536 centroids, keys with outlier channels, values next to centroids):
    the tensor-core filter path and the full pinned scan (VECINFER_NN16_SCAN=1, the round-1 kernel)
    give identical codes.  (Parity against the oracle itself is pinned by the cases above.)"""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    script = f"""
import sys
sys.path.insert(0, {here!r})
import numpy as np, torch, synth
from helpers import load_codebooks
from paper_2510_06175_b200 import vecinfer as vi
CB = load_codebooks()
T, H = 512, 8
k = synth.gen_keys(T, H, 128, seed=1800)
cv = CB['cv_b4d4']
rng = np.random.default_rng(1801)
v = cv[rng.integers(0, 65536, size=(T * H * 32,))].reshape(1, T, H, 128)
v = synth.round_to_bf16((v + 1e-3 * rng.standard_normal(v.shape)).astype(np.float32))
t = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)
kc = torch.zeros(1, H, T, 64, dtype=torch.uint8, device='cuda')
vc = torch.zeros_like(kc)
vi.encode_kv(t(k), t(v), torch.from_numpy(CB['inv_lambda']).cuda(), t(CB['ck_b4d4']), t(cv), kc, vc,
             torch.zeros(1, dtype=torch.int32, device='cuda'), vi.B4D4, vi.B4D4)
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([kc.cpu().numpy().ravel(), vc.cpu().numpy().ravel()]))
"""
    outs = []
    for scan in ("0", "1"):
        path = os.path.join("/tmp", f"nn16_xcheck_{scan}_{os.getpid()}.npy")
        env = dict(os.environ, VECINFER_NN16_SCAN=scan)
        r = subprocess.run([sys.executable, "-c", script, path], env=env, cwd=os.path.dirname(here),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(np.load(path))
        os.remove(path)
    assert np.array_equal(outs[0], outs[1])
