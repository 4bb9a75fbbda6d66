"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402

dev = torch.device("cuda", 0)
NN16_ONLY = "--nn16-only" in sys.argv   # (run under VECINFER_NN16_TC=1 for the tcgen05 filter)
z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
lam = torch.from_numpy(z["lambda"]).to(dev)
inv = torch.from_numpy(z["inv_lambda"]).to(dev)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
# 16-bit books (tensor-core filter + exact selection): per-head books over two passes, D = 64
ck16h = T(synth.round_to_bf16(np.random.default_rng(5).normal(0, 1, (8, 65536, 4)).astype(np.float32))).to(torch.bfloat16)
cv16s = T(synth.bf16_from_bits(z["cv_b4d4"])).to(torch.bfloat16)
k65 = T(synth.gen_keys(65, 8, 128, seed=6)).to(torch.bfloat16)
v65 = T(synth.gen_values(65, 8, 128, seed=7)).to(torch.bfloat16)
kc65 = torch.zeros(1, 8, 70, 64, dtype=torch.uint8, device=dev)
vc65 = torch.zeros_like(kc65)
vi.encode_kv(k65, v65, inv, ck16h, cv16s, kc65, vc65, torch.zeros(1, dtype=torch.int32, device=dev), vi.B4D4, vi.B4D4)
c16_64 = vi.VQConfig(64, 4, 16)
kc6 = torch.zeros(1, 4, 8, 32, dtype=torch.uint8, device=dev)
vi.encode_kv(k65[:, :7, :4, :64].contiguous(), v65[:, :7, :4, :64].contiguous(), inv[:4, :64].contiguous(), cv16s, cv16s,
             kc6, kc6.clone(), torch.zeros(1, dtype=torch.int32, device=dev), c16_64, c16_64)
if NN16_ONLY:
    torch.cuda.synchronize()
    print("sanitize smoke (16-bit encode only) done")
    sys.exit(0)
for name, cfg in (("b1d4", vi.B1D4), ("b2d4", vi.B2D4), ("b4d4", vi.B4D4)):
    ck = T(synth.bf16_from_bits(z[f"ck_{name}"])).to(torch.bfloat16)
    cv = T(synth.bf16_from_bits(z[f"cv_{name}"])).to(torch.bfloat16)
    B, N = 2, 300
    k = T(synth.gen_keys(N, 8, 128, seed=1, batch=B)).to(torch.bfloat16)
    v = T(synth.gen_values(N, 8, 128, seed=2, batch=B)).to(torch.bfloat16)
    kc = torch.zeros(B, 8, N + 4, cfg.row_bytes, dtype=torch.uint8, device=dev)
    vc = torch.zeros_like(kc)
    vi.encode_kv(k, v, inv, ck, cv, kc, vc, torch.zeros(B, dtype=torch.int32, device=dev), cfg, cfg)
    q = T(synth.gen_queries(B, 32, 8, 128, seed=3)).to(torch.bfloat16)
    seq = torch.tensor([N, N // 3], dtype=torch.int32, device=dev)
    for splits in (0, 1, 3, 8, 20):
        vi.attn_decode(q, lam, ck, cv, kc, vc, seq, num_splits=splits, kcfg=cfg, vcfg=cfg)
    # stream kernel: straddling pieces (auto), fixed pieces, persistent last-arriver merge (80 x 16 > #SMs)
    for splits in (0, 3, 80):
        vi.attn_decode(q, lam, ck, cv, kc, vc, seq, num_splits=splits, kcfg=cfg, vcfg=cfg, algo="stream")
    kn, vn = k[:, 0].contiguous(), v[:, 0].contiguous()
    vi.decode_step(q, kn, vn, lam, inv, ck, cv, kc, vc, torch.tensor([N, N // 3], dtype=torch.int32, device=dev),
                   seq + 1, kcfg=cfg, vcfg=cfg)
    vi.decode_step(q, kn, vn, lam, inv, ck, cv, kc, vc, torch.tensor([N, N // 3], dtype=torch.int32, device=dev),
                   seq + 1, kcfg=cfg, vcfg=cfg, algo="stream")
# ---- round-2 paths
ck = T(synth.bf16_from_bits(z["ck_b2d4"])).to(torch.bfloat16)
cv = T(synth.bf16_from_bits(z["cv_b2d4"])).to(torch.bfloat16)
B, N = 3, 700
kc = synth.gen_codes_torch((B, 8, N + 40, 32), 8, seed=11, device=dev)
vc = synth.gen_codes_torch((B, 8, N + 40, 32), 8, seed=12, device=dev)
q = T(synth.gen_queries(B, 32, 8, 128, seed=13)).to(torch.bfloat16)
seq = torch.tensor([N, 333, 31], dtype=torch.int32, device=dev)
kn = T(synth.gen_keys(1, 8, 128, seed=14, batch=B)[:, 0]).to(torch.bfloat16)
vn = T(synth.gen_values(1, 8, 128, seed=15, batch=B)[:, 0]).to(torch.bfloat16)
wp = seq - 1
# VECINFER_ATTN_FLAG_EARLY_CACHE: split, stream and fused decode step with the pre-wait cache reads
for splits in (0, 3):
    vi.attn_decode(q, lam, ck, cv, kc, vc, seq, num_splits=splits, early_cache=True)
vi.attn_decode(q, lam, ck, cv, kc, vc, seq, algo="stream", early_cache=True)
vi.decode_step(q, kn, vn, lam, inv, ck, cv, kc, vc, wp, seq, early_cache=True)
# tcgen05 score path (split / multi-wave persistent / fused append)
for splits in (0, 3, 60):
    vi.attn_decode(q, lam, ck, cv, kc, vc, seq, num_splits=splits, algo="tc")
vi.decode_step(q, kn, vn, lam, inv, ck, cv, kc, vc, wp, seq, algo="tc")
# paged stream kernel (16-token sub-tiles across pages) + paged fused append
ps = 32
npb = (N + 40 + ps - 1) // ps
pool_k = synth.gen_codes_torch((B * npb + 2, 8, ps, 32), 8, seed=16, device=dev)
pool_v = synth.gen_codes_torch((B * npb + 2, 8, ps, 32), 8, seed=17, device=dev)
bt = torch.randperm(B * npb + 2, device=dev)[:B * npb].view(B, npb).to(torch.int32)
for splits in (0, 3, 60):
    vi.attn_decode(q, lam, ck, cv, pool_k, pool_v, seq, num_splits=splits, algo="stream", block_table=bt)
vi.decode_step(q, kn, vn, lam, inv, ck, cv, pool_k, pool_v, wp, seq, algo="stream", block_table=bt)
# head_dim 64: residual window + fused append
c64 = vi.VQConfig(64, 4, 8)
kc64 = synth.gen_codes_torch((B, 8, N + 40, 16), 8, seed=18, device=dev)
vc64 = synth.gen_codes_torch((B, 8, N + 40, 16), 8, seed=19, device=dev)
q64 = T(synth.gen_queries(B, 32, 8, 64, seed=20)).to(torch.bfloat16)
kr = T(synth.gen_keys(64, 8, 64, seed=21, batch=B).transpose(0, 2, 1, 3)).to(torch.bfloat16)
vr = T(synth.gen_values(64, 8, 64, seed=22, batch=B).transpose(0, 2, 1, 3)).to(torch.bfloat16)
rl = torch.tensor([64, 9, 1], dtype=torch.int32, device=dev)
lam64, inv64 = lam[:, :64].contiguous(), inv[:, :64].contiguous()
vi.attn_decode(q64, lam64, ck, cv, kc64, vc64, seq, kcfg=c64, vcfg=c64, k_res=kr, v_res=vr, res_lens=rl)
kn64, vn64 = kn[..., :64].contiguous(), vn[..., :64].contiguous()
vi.decode_step(q64, kn64, vn64, lam64, inv64, ck, cv, kc64, vc64, wp, seq, kcfg=c64, vcfg=c64)
# NEXT-2: separate shared tables (d8b12, d4b10), fused generic append (d4b10, d2b8), d8b16
z2 = np.load(os.path.join(ROOT, "data", "next2_codebooks.npz"))
for name, cfg in (("d8b12", vi.D8B12), ("d4b10", vi.D4B10), ("d2b8", vi.D2B8)):
    ckn = T(synth.bf16_from_bits(z2[f"ck_{name}"])).to(torch.bfloat16)
    cvn = T(synth.bf16_from_bits(z2[f"cv_{name}"])).to(torch.bfloat16)
    kcn = synth.gen_codes_torch((B, 8, N + 40, cfg.row_bytes), 8, seed=23, device=dev)
    vcn = synth.gen_codes_torch((B, 8, N + 40, cfg.row_bytes), 8, seed=24, device=dev)
    vi.attn_decode(q, lam, ckn, cvn, kcn, vcn, seq, kcfg=cfg, vcfg=cfg, num_splits=3)
    vi.decode_step(q, kn, vn, lam, inv, ckn, cvn, kcn, vcn, wp, seq, kcfg=cfg, vcfg=cfg)
zl = np.load(os.path.join(ROOT, "data", "d8b16_levels.npz"))
ck16 = T(synth.product_codebook(synth.bf16_from_bits(zl["lv_d8b16_k"]))).to(torch.bfloat16)
cv16 = T(synth.product_codebook(synth.bf16_from_bits(zl["lv_d8b16_v"]))).to(torch.bfloat16)
kc16 = synth.gen_codes_torch((1, 8, 200, 32), 8, seed=25, device=dev)
vc16 = synth.gen_codes_torch((1, 8, 200, 32), 8, seed=26, device=dev)
vi.decode_step(q[:1], kn[:1], vn[:1], lam, inv, ck16, cv16, kc16, vc16, torch.tensor([150], dtype=torch.int32, device=dev),
               torch.tensor([151], dtype=torch.int32, device=dev), kcfg=vi.D8B16, vcfg=vi.D8B16)
vi.calibrate_smooth(T(synth.gen_calibration_keys(8, 128, n_samples=1, sample_len=64)).to(torch.bfloat16))
vi.merge_lse(torch.randn(3, 2, 32, 128, device=dev), torch.randn(3, 2, 32, device=dev))
# codebook k-means (assign / finalize / re-seed: four far centroids get no points)
X = torch.randn(3000, 4, device=dev)
C = torch.cat([X[:60].clone(), torch.full((4, 4), 100.0, device=dev)])
vi.kmeans_step(X, C)
vi.kmeans_step(X[:, :2].contiguous(), C[:, :2].contiguous())
# fused peer-memory exchange + merge with one rank (own window only; automatic epochs, 2 parities)
import ctypes  # noqa: E402
from paper_2510_06175_b200 import _lib  # noqa: E402
lib = _lib.load()
w = ctypes.c_void_p()
h = (ctypes.c_char * 64)()
_lib.check("p2p_window_create", lib.vecinfer_p2p_window_create(lib.vecinfer_p2p_window_bytes(1, 64, 128),
                                                             ctypes.addressof(w), ctypes.addressof(h)))
wins = torch.tensor([w.value], dtype=torch.int64, device=dev)
o_l, l_l = torch.randn(2, 32, 128, device=dev), torch.randn(2, 32, device=dev)
o_m, l_m = torch.empty_like(o_l), torch.empty_like(l_l)
for _ in range(2):
    _lib.check("merge_lse_p2p", lib.vecinfer_merge_lse_p2p(o_l.data_ptr(), l_l.data_ptr(), wins.data_ptr(), 1, 0, 2, 32,
                                                           128, 0, o_m.data_ptr(), 1, l_m.data_ptr(), None, None))
torch.cuda.synchronize()
lib.vecinfer_p2p_window_destroy(w)
torch.cuda.synchronize()
print("sanitize smoke done")
