"""Paged code caches (serving integration): page pools [n_pages, H_kv,
page_size, row] addressed through a block table, as a vLLM/SGLang-style allocator hands them out.

The pages of every sequence are a random permutation of the pool, so any addressing mistake moves
tokens.  Paged attention must equal contiguous attention BIT FOR BIT (same tokens, same split plan,
same arithmetic) and match the oracle; paged encode must write exactly the oracle's codes at the
translated rows; the fused and separate decode-step appends must land in the right page.
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
from test_gpu_parity import _assert_close, _attn_case, _run_gpu, _run_ref, t_bf16, t_f32, t_i32, t_u8  # noqa: E402

CB = load_codebooks()


def _paginate(codes, page_size, seed, spare=3):
    """contiguous [B, H, n_cap, row] -> (pool [n_pages, H, ps, row], block_table [B, n_cap/ps])."""
    B, H, n_cap, row = codes.shape
    npb = n_cap // page_size
    n_pages = B * npb + spare
    perm = np.random.default_rng(seed).permutation(n_pages)[:B * npb].reshape(B, npb)
    pool = np.zeros((n_pages, H, page_size, row), codes.dtype)
    for b in range(B):
        for i in range(npb):
            pool[perm[b, i]] = codes[b, :, i * page_size:(i + 1) * page_size]
    return pool, perm.astype(np.int32)


def _unpaginate(pool, bt, page_size):
    B, npb = bt.shape
    out = np.stack([np.concatenate([pool[bt[b, i]] for i in range(npb)], axis=1) for b in range(B)])
    return out   # [B, H, n_cap, row]


@pytest.mark.parametrize("page_size", [32, 64, 256])
@pytest.mark.parametrize("lens", [[2048], [1000, 31, 1999], [5, 2048]])
def test_paged_attention_equals_contiguous(page_size, lens):
    n_cap = 2048
    c = _attn_case(len(lens), 8, 4, n_cap, lens, seed=500 + page_size + len(lens))
    kpool, bt = _paginate(c["kc"].astype(np.uint8), page_size, seed=501)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), page_size, seed=501)
    o_c, L_c = _run_gpu(c)
    o_p, L_p = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(kpool),
                              t_u8(vpool), t_i32(c["seq_lens"]), block_table=t_i32(bt))
    o_p, L_p = o_p.cpu().numpy(), L_p.cpu().numpy()
    assert np.array_equal(o_p, o_c) and np.array_equal(L_p, L_c)
    _assert_close(o_p, L_p, *_run_ref(c))


@pytest.mark.parametrize("splits", [0, 3])
def test_paged_token_range_and_gqa5(splits):
    """Sharding hook (tok_begin multiple of 32) and a GQA group of 5 over a paged pool."""
    n_cap, ps = 1536, 64
    c = _attn_case(2, 8, 5, n_cap, [1536, 700], seed=510)
    kpool, bt = _paginate(c["kc"].astype(np.uint8), ps, seed=511)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), ps, seed=511)
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(kpool),
                          t_u8(vpool), t_i32(c["seq_lens"]), tok_begin=256, tok_end=1200, num_splits=splits,
                          block_table=t_i32(bt))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c, 256, 1200))


def test_paged_encode_prefill_and_append():
    """Bulk encode (T = 300) and a 1-token append into a paged pool: the codes at the translated
    rows are the oracle's, every other page is untouched."""
    B, H, ps, npb = 2, 8, 64, 8
    n_cap = ps * npb
    rng = np.random.default_rng(520)
    n_pages = B * npb + 2
    bt = rng.permutation(n_pages)[:B * npb].reshape(B, npb).astype(np.int32)
    kpool = torch.zeros(n_pages, H, ps, 32, dtype=torch.uint8, device="cuda")
    vpool = torch.zeros_like(kpool)
    T = 300
    k = synth.gen_keys(T, 8, 128, seed=521, batch=B)
    v = synth.gen_values(T, 8, 128, seed=522, batch=B)
    inv, ck, cv = CB["inv_lambda"], CB["ck_b2d4"], CB["cv_b2d4"]
    wp = np.array([0, 100], np.int32)
    vi.encode_kv(t_bf16(k), t_bf16(v), t_f32(inv), t_bf16(ck), t_bf16(cv), kpool, vpool, t_i32(wp),
                 block_table=t_i32(bt))
    kn = synth.gen_keys(1, 8, 128, seed=523, batch=B)
    vn = synth.gen_values(1, 8, 128, seed=524, batch=B)
    wp2 = np.array([300, 400], np.int32)
    vi.encode_kv(t_bf16(kn), t_bf16(vn), t_f32(inv), t_bf16(ck), t_bf16(cv), kpool, vpool, t_i32(wp2),
                 block_table=t_i32(bt))
    kc = _unpaginate(kpool.cpu().numpy(), bt, ps)
    vc = _unpaginate(vpool.cpu().numpy(), bt, ps)
    exp_k = np.zeros((B, H, n_cap, 32), np.uint8)
    exp_v = np.zeros_like(exp_k)
    for b in range(B):
        for h in range(H):
            kk, vv = ref.encode_kv(k[b, :, h], v[b, :, h], inv[h], ck[h], cv[h])
            exp_k[b, h, wp[b]:wp[b] + T], exp_v[b, h, wp[b]:wp[b] + T] = kk, vv
            kk, vv = ref.encode_kv(kn[b, :, h], vn[b, :, h], inv[h], ck[h], cv[h])
            exp_k[b, h, wp2[b]], exp_v[b, h, wp2[b]] = kk[0], vv[0]
    assert np.array_equal(kc, exp_k) and np.array_equal(vc, exp_v)
    spare = np.setdiff1d(np.arange(n_pages), bt.ravel())
    assert not kpool[torch.from_numpy(spare).cuda().long()].any()


@pytest.mark.parametrize("B", [2, 20])   # 2: fused single-wave append; 20 (160 units): separate append launch
def test_paged_decode_step(B):
    n_cap, ps = 512, 32
    lens = [n_cap - 7 - (b % 5) for b in range(B)]
    c = _attn_case(B, 8, 4, n_cap, lens, seed=530 + B)
    kpool, bt = _paginate(c["kc"].astype(np.uint8), ps, seed=531)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), ps, seed=531)
    kn = synth.gen_keys(1, 8, 128, seed=532, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=533, batch=B)[:, 0]
    wp = [n - 1 for n in lens]
    kp, vp = t_u8(kpool), t_u8(vpool)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kp, vp, t_i32(wp), t_i32(lens), err_flags=err,
                          block_table=t_i32(bt))
    assert int(err.item()) == 0
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]], c["vc"][b, h, wp[b]] = kk, vv
    assert np.array_equal(_unpaginate(kp.cpu().numpy(), bt, ps), c["kc"].astype(np.uint8))
    assert np.array_equal(_unpaginate(vp.cpu().numpy(), bt, ps), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))


def test_paged_rejects_bad_descriptors():
    c = _attn_case(1, 8, 4, 256, [256], seed=540)
    kpool, bt = _paginate(c["kc"].astype(np.uint8), 64, seed=541)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), 64, seed=541)
    args = (t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(kpool), t_u8(vpool),
            t_i32(c["seq_lens"]))
    with pytest.raises(VecInferError):
        vi.attn_decode(*args, block_table=t_i32(bt), tok_begin=16)          # range start not 32-aligned
    with pytest.raises(VecInferError):
        vi.attn_decode(*args, block_table=t_i32(bt), algo="lut")            # contiguous-only variant
    kbad = torch.zeros(kpool.shape[0], 8, 48, 32, dtype=torch.uint8, device="cuda")   # page_size 48
    with pytest.raises(VecInferError):
        vi.attn_decode(args[0], args[1], args[2], args[3], kbad, kbad, args[6], block_table=t_i32(bt))


# ---------------------------------------------------------------- stream kernel over paged pools
@pytest.mark.parametrize("page_size", [32, 64])
@pytest.mark.parametrize("splits", [0, 3, 40])   # 0: one piece per CTA; 40 x 24 units > #SMs: persistent
def test_paged_stream_equals_contiguous(page_size, splits):
    """The stream partition cuts units at 16-token boundaries, so a 32-token tile's two sub-tiles
    can lie in different pages: each is translated separately.  Bit-equal to the contiguous stream
    kernel, and vs the oracle."""
    n_cap = 2048
    lens = [2048, 1000, 37]
    c = _attn_case(len(lens), 8, 4, n_cap, lens, seed=550 + page_size + splits)
    kpool, bt = _paginate(c["kc"].astype(np.uint8), page_size, seed=551)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), page_size, seed=551)
    o_c, L_c = _run_gpu(c, algo="stream", num_splits=splits)
    o_p, L_p = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(kpool),
                              t_u8(vpool), t_i32(c["seq_lens"]), block_table=t_i32(bt), algo="stream",
                              num_splits=splits)
    o_p, L_p = o_p.cpu().numpy(), L_p.cpu().numpy()
    assert np.array_equal(o_p, o_c) and np.array_equal(L_p, L_c)
    _assert_close(o_p, L_p, *_run_ref(c))


def test_paged_stream_auto_batch_decode_and_fused_append():
    """B*H_kv >= #SMs: AUTO runs the stream kernel on the paged pool, and decode_step fuses the append
    (owner pieces write the new codes at the translated rows)."""
    B, n_cap, ps = 20, 512, 64
    lens = [n_cap - 3 - (7 * b) % 40 for b in range(B)]
    c = _attn_case(B, 8, 4, n_cap, lens, seed=560)
    kpool, bt = _paginate(c["kc"].astype(np.uint8), ps, seed=561)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), ps, seed=561)
    assert vi.attn_kernel_kind(B, 8, n_cap) == "stream"
    o_p, L_p = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(kpool),
                              t_u8(vpool), t_i32(c["seq_lens"]), block_table=t_i32(bt))
    _assert_close(o_p.cpu().numpy(), L_p.cpu().numpy(), *_run_ref(c))
    kn = synth.gen_keys(1, 8, 128, seed=562, batch=B)[:, 0]
    vn = synth.gen_values(1, 8, 128, seed=563, batch=B)[:, 0]
    wp = [n - 1 for n in lens]
    kp, vp = t_u8(kpool), t_u8(vpool)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert vi.decode_step_launches(B, 8, n_cap) == 1
    o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                          t_bf16(c["ck"]), t_bf16(c["cv"]), kp, vp, t_i32(wp), t_i32(lens), err_flags=err,
                          block_table=t_i32(bt))
    assert int(err.item()) == 0
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]], c["vc"][b, h, wp[b]] = kk, vv
    assert np.array_equal(_unpaginate(kp.cpu().numpy(), bt, ps), c["kc"].astype(np.uint8))
    assert np.array_equal(_unpaginate(vp.cpu().numpy(), bt, ps), c["vc"].astype(np.uint8))
    _assert_close(o.cpu().numpy(), L.cpu().numpy(), *_run_ref(c))
