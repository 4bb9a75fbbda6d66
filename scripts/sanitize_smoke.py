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
z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
lam = torch.from_numpy(z["lambda"]).to(dev)
inv = torch.from_numpy(z["inv_lambda"]).to(dev)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
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
ck = T(synth.bf16_from_bits(z["ck_b2d4"])).to(torch.bfloat16)
vi.attn_decode(q, lam, ck, ck, kc[..., :32].contiguous() if kc.shape[-1] >= 32 else kc, vc[..., :32].contiguous(),
               seq, algo="lut") if False else None
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
