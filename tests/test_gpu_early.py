"""VECINFER_ATTN_FLAG_EARLY_CACHE (ABI v7): the split kernel reads seq_lens / write_pos / the block
table and issues its first code tile before the programmatic-dependent-launch wait.

The flag changes WHEN loads are issued, never what is computed: every result must equal the
flagless launch bit for bit and the oracle within the north_star bars.  The graph test chains
layers the way a model does -- layer l's q is layer l-1's output, written by the kernel right
before it -- so a q read before the wait would pick up a stale value and break bit-identity.
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
from test_gpu_parity import _assert_close, _attn_case, _run_ref, t_bf16, t_f32, t_i32, t_u8  # noqa: E402
from test_gpu_paged import _paginate  # noqa: E402

CB = load_codebooks()


def _attn(c, early, **kw):
    o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(c["kc"]),
                          t_u8(c["vc"]), t_i32(c["seq_lens"]), early_cache=early, **kw)
    return o.cpu().numpy(), L.cpu().numpy()


@pytest.mark.parametrize("splits", [0, 1, 3, 18])
@pytest.mark.parametrize("lens", [[4096], [3000, 17, 0], [33]])
def test_early_attention_equals_plain(splits, lens):
    c = _attn_case(len(lens), 8, 4, max(lens) + 40, lens, seed=900 + splits + len(lens))
    o0, L0 = _attn(c, False, num_splits=splits)
    o1, L1 = _attn(c, True, num_splits=splits)
    assert np.array_equal(o0, o1) and np.array_equal(L0, L1)
    _assert_close(o1, L1, *_run_ref(c))


@pytest.mark.parametrize("G", [2, 5])
def test_early_attention_gqa_and_token_range(G):
    c = _attn_case(2, 8, G, 2500, [2500, 1200], seed=910 + G)
    o0, L0 = _attn(c, False, tok_begin=64, tok_end=2000)
    o1, L1 = _attn(c, True, tok_begin=64, tok_end=2000)
    assert np.array_equal(o0, o1) and np.array_equal(L0, L1)
    _assert_close(o1, L1, *_run_ref(c, 64, 2000))


def test_early_attention_paged():
    lens = [2048, 700]
    c = _attn_case(2, 8, 4, 2048, lens, seed=920)
    kpool, bt = _paginate(c["kc"].astype(np.uint8), 64, seed=921)
    vpool, _ = _paginate(c["vc"].astype(np.uint8), 64, seed=921)
    outs = []
    for early in (False, True):
        o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(kpool),
                              t_u8(vpool), t_i32(lens), block_table=t_i32(bt), num_splits=5, algo="mma",
                              early_cache=early)
        outs.append((o.cpu().numpy(), L.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    _assert_close(*outs[1], *_run_ref(c))


@pytest.mark.parametrize("lens", [[2048] * 20, [3000, 17, 0, 1500, 999]])
def test_early_stream_kernel(lens):
    """The stream partition (forced, and AUTO at B * H_kv >= #SMs) with the flag: bit-identical."""
    c = _attn_case(len(lens), 8, 4, max(lens) + 16, lens, seed=960 + len(lens))
    algo = "auto" if len(lens) >= 19 else "stream"
    if algo == "auto":
        assert vi.attn_kernel_kind(len(lens), 8, max(lens) + 16) == "stream"
    o0, L0 = _attn(c, False, algo=algo)
    o1, L1 = _attn(c, True, algo=algo)
    assert np.array_equal(o0, o1) and np.array_equal(L0, L1)
    _assert_close(o1, L1, *_run_ref(c))


@pytest.mark.parametrize("splits,lens", [(0, [1500, 37]), (3, [1500, 37]), (0, [600] * 20)])   # B = 20: stream
def test_early_decode_step_fused_append(splits, lens):
    """decode_step with the flag: the appended codes are the oracle's; output == flagless launch."""
    B = len(lens)
    res = []
    for early in (False, True):
        c = _attn_case(B, 8, 4, max(lens) + 5, lens, seed=930 + splits)
        kn = synth.gen_keys(1, 8, 128, seed=931, batch=B)[:, 0]
        vn = synth.gen_values(1, 8, 128, seed=932, batch=B)[:, 0]
        wp = [n - 1 for n in lens]
        kcodes, vcodes = t_u8(c["kc"]), t_u8(c["vc"])
        o, L = vi.decode_step(t_bf16(c["q"]), t_bf16(kn), t_bf16(vn), t_f32(c["lam"]), t_f32(CB["inv_lambda"]),
                              t_bf16(c["ck"]), t_bf16(c["cv"]), kcodes, vcodes, t_i32(wp), t_i32(lens),
                              num_splits=splits, early_cache=early)
        res.append((o.cpu().numpy(), L.cpu().numpy(), kcodes.cpu().numpy(), vcodes.cpu().numpy()))
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)
    for b in range(B):
        for h in range(8):
            kk, vv = ref.encode_kv(kn[b, h], vn[b, h], CB["inv_lambda"][h], c["ck"][h], c["cv"][h])
            c["kc"][b, h, wp[b]] = kk
            c["vc"][b, h, wp[b]] = vv
    assert np.array_equal(res[1][2], c["kc"].astype(np.uint8)) and np.array_equal(res[1][3], c["vc"].astype(np.uint8))
    _assert_close(res[1][0], res[1][1], *_run_ref(c))


def _chain(n_layers, early, N, graph):
    """n_layers decode steps back to back; layer l's q = layer l-1's bf16 output (written by the
    kernel launched right before it), each layer with its own cache; returns every layer's o."""
    dev = "cuda"
    B, Hkv = 1, 8
    q0 = t_bf16(synth.gen_queries(B, 32, 8, 128, seed=941))
    kcs = [synth.gen_codes_torch((B, Hkv, N, 32), 8, seed=950 + 2 * l, device=dev) for l in range(n_layers)]
    vcs = [synth.gen_codes_torch((B, Hkv, N, 32), 8, seed=951 + 2 * l, device=dev) for l in range(n_layers)]
    kn = t_bf16(synth.gen_keys(1, 8, 128, seed=942, batch=B)[:, 0])
    vn = t_bf16(synth.gen_values(1, 8, 128, seed=943, batch=B)[:, 0])
    lam, inv = t_f32(CB["lambda"]), t_f32(CB["inv_lambda"])
    ck, cv = t_bf16(CB["ck_b2d4"]), t_bf16(CB["cv_b2d4"])
    wp, sl = t_i32([N - 1]), t_i32([N])
    # bf16 outputs feed the next layer's q; the last layer writes fp32 (checked against the oracle)
    outs = [torch.zeros(B, 32, 128, dtype=torch.bfloat16 if l < n_layers - 1 else torch.float32, device=dev)
            for l in range(n_layers)]
    lses = [torch.zeros(B, 32, dtype=torch.float32, device=dev) for _ in range(n_layers)]
    ws = [vi.decode_step_workspace(B, 32, Hkv, N, device=dev) for _ in range(n_layers)]
    s = torch.cuda.Stream()

    def run():
        for l in range(n_layers):
            q = q0 if l == 0 else outs[l - 1]
            vi.decode_step(q, kn, vn, lam, inv, ck, cv, kcs[l], vcs[l], wp, sl, out=outs[l], lse=lses[l],
                           workspace=ws[l], early_cache=early)

    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        if graph:
            run()   # warm-up (lazy attributes) outside the capture
            torch.cuda.synchronize()
            for o in outs:
                o.zero_()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                run()
            for _ in range(3):   # replays recompute the same chain (the append rewrites row N-1)
                g.replay()
        else:
            run()
    torch.cuda.synchronize()
    return ([o.float().cpu().numpy() for o in outs], [x.cpu().numpy() for x in lses],
            [k.cpu().numpy() for k in kcs], [v.cpu().numpy() for v in vcs], q0.float().cpu().numpy(),
            kn.float().cpu().numpy(), vn.float().cpu().numpy())


@pytest.mark.parametrize("N", [32768, 4000])
def test_early_layer_chain_in_graph(N):
    """A graph of 8 back-to-back decode steps (PDL) whose q is the previous step's output: with the
    flag, every layer equals the eager flagless chain bit for bit, and the last layer matches the
    oracle on its own (GPU-produced) input."""
    L = 8
    ref_o, ref_l, *_ = _chain(L, False, N, graph=False)
    o, lse, kcs, vcs, q0, kn, vn = _chain(L, True, N, graph=True)
    for l in range(L):
        assert np.array_equal(o[l], ref_o[l]) and np.array_equal(lse[l], ref_l[l]), f"layer {l}"
    q_last = o[L - 2].reshape(1, 32, 128)
    for h in (0, 5):
        kk = kcs[L - 1][0, h].astype(np.int64)
        vv = vcs[L - 1][0, h].astype(np.int64)
        o_ref, L_ref = ref.attention_vq(q_last[0, 4 * h:4 * h + 4], CB["lambda"][h], CB["ck_b2d4"][h],
                                        CB["cv_b2d4"][h], kk, vv)
        _assert_close(o[L - 1][0, 4 * h:4 * h + 4], lse[L - 1][0, 4 * h:4 * h + 4], o_ref, L_ref)


def test_early_persistent_grid_residual_and_d64():
    """Pre-wait reads on the paths with extra state: a persistent multi-item split grid (forced 40
    splits x 16 units > #SMs: only the first item reads before the wait), a residual window (read
    after the wait), and head_dim 64."""
    lens = [3000, 2500]
    c = _attn_case(2, 8, 4, 3000, lens, seed=970)
    o0, L0 = _attn(c, False, num_splits=40)
    o1, L1 = _attn(c, True, num_splits=40)
    assert np.array_equal(o0, o1) and np.array_equal(L0, L1)
    _assert_close(o1, L1, *_run_ref(c))
    # residual window rows next to the codes
    B, R = 2, 24
    kr = t_bf16(synth.gen_keys(R, 8, 128, seed=971, batch=B).transpose(0, 2, 1, 3))
    vr = t_bf16(synth.gen_values(R, 8, 128, seed=972, batch=B).transpose(0, 2, 1, 3))
    rl = t_i32([R, 5])
    outs = []
    for early in (False, True):
        o, L = vi.attn_decode(t_bf16(c["q"]), t_f32(c["lam"]), t_bf16(c["ck"]), t_bf16(c["cv"]), t_u8(c["kc"]),
                              t_u8(c["vc"]), t_i32(c["seq_lens"]), k_res=kr, v_res=vr, res_lens=rl, num_splits=3,
                              early_cache=early)
        outs.append((o.cpu().numpy(), L.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    # head_dim 64 (split kernel and the D = 64 stream partition)
    c64 = vi.VQConfig(64, 4, 8)
    kc64 = synth.gen_codes_torch((20, 8, 1500, 16), 8, seed=973, device="cuda")
    vc64 = synth.gen_codes_torch((20, 8, 1500, 16), 8, seed=974, device="cuda")
    q64 = t_bf16(synth.gen_queries(20, 32, 8, 64, seed=975))
    lam64 = t_f32(CB["lambda"][:, :64])
    seq = t_i32([1500 - 7 * i for i in range(20)])
    for algo in ("mma", "stream"):
        res = []
        for early in (False, True):
            o, L = vi.attn_decode(q64, lam64, t_bf16(c["ck"]), t_bf16(c["cv"]), kc64, vc64, seq, kcfg=c64, vcfg=c64,
                                  algo=algo, early_cache=early)
            res.append((o.cpu().numpy(), L.cpu().numpy()))
        assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1]), algo
