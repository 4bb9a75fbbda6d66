"""On-box context baselines for the paper's speedup claims.

The paper reports its fused VQ decode attention against full-precision attention ("vanilla full
attention" / SDPA / FlashAttention) and against dequantise-then-attend (P:150,
270-272).  Those comparison systems are out of scope as products; this script measures on-box
stand-ins so the ratios can be quoted for B200 as context:

  bf16 SDPA      torch.nn.functional.scaled_dot_product_attention (GQA), bf16 K/V cache
  bf16 flashinfer  flashinfer decode over the same bf16 cache (if it runs on this box)
  dequant+SDPA   gather C[codes] into a bf16 K~/V^ cache (torch indexing), then SDPA with q~
  vecinfer       vecinfer.attn_decode on the VQ codes (this repo's kernels)

Every variant is CUDA-graph captured over enough distinct caches to exceed L2 and timed with
events on the launching stream.  Library kernels here are baselines, not the product path.

    python scripts/context_baselines.py [--workloads cfg2,cfg3,cfg4] [--reps 20]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402

SHAPES = {"cfg2": (1, 32768), "cfg3": (64, 8192), "cfg4": (1, 196608)}
HQ, HKV, D = 32, 8, 128


def time_graph(fn, copies, reps, stream):
    with torch.cuda.stream(stream):
        for i in range(copies):   # warm-up / lazy init outside capture
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(copies):
            fn(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * copies)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="cfg2,cfg3,cfg4")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    lam = torch.from_numpy(z["lambda"]).to(dev)
    ck = torch.from_numpy(synth.bf16_from_bits(z["ck_b2d4"])).to(dev).to(torch.bfloat16)   # [8, 256, 4]
    cv = torch.from_numpy(synth.bf16_from_bits(z["cv_b2d4"])).to(dev).to(torch.bfloat16)
    stream = torch.cuda.Stream()
    out = []
    for w in args.workloads.split(","):
        B, N = SHAPES[w]
        code_bytes = B * HKV * N * 64
        bf16_bytes = B * HKV * N * D * 2 * 2
        copies_vq = max(2, int(np.ceil(400e6 / code_bytes)))
        copies_bf = max(2, int(np.ceil(400e6 / bf16_bytes)))
        q = torch.from_numpy(synth.gen_queries(B, HQ, HKV, D, seed=3)).to(dev).to(torch.bfloat16)
        seq = torch.full((B,), N, dtype=torch.int32, device=dev)
        res = {"workload": w, "B": B, "N": N, "code_bytes": code_bytes, "bf16_kv_bytes": bf16_bytes}

        # ---- vecinfer (VQ codes)
        kcs = [synth.gen_codes_torch((B, HKV, N, 32), 8, seed=2 * i, device=dev) for i in range(copies_vq)]
        vcs = [synth.gen_codes_torch((B, HKV, N, 32), 8, seed=2 * i + 1, device=dev) for i in range(copies_vq)]
        ws = [vi.attn_workspace(B, HQ, HKV, N, device=dev) for _ in range(copies_vq)]
        o = torch.empty(B, HQ, D, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(B, HQ, dtype=torch.float32, device=dev)
        res["vecinfer_us"] = time_graph(
            lambda i: vi.attn_decode(q, lam, ck, cv, kcs[i], vcs[i], seq, out=o, lse=lse, workspace=ws[i]),
            copies_vq, args.reps, stream)
        res["vecinfer_kernel"] = vi.attn_kernel_kind(B, HKV, N)

        # ---- dequantise-then-attend: K~ = C_k[codes] (transformed space, Eq. 7), V^ = C_v[codes]
        hidx = torch.arange(HKV, device=dev).view(1, HKV, 1, 1)
        kdq = torch.empty(B, HKV, N, D, dtype=torch.bfloat16, device=dev)
        vdq = torch.empty_like(kdq)
        qt = torch.empty(B, HQ, 1, D, dtype=torch.bfloat16, device=dev)
        Hm = torch.from_numpy((np.asarray(
            [[(-1) ** bin(i & j).count("1") for j in range(D)] for i in range(D)], dtype=np.float64) / np.sqrt(D))
            .astype(np.float32)).to(dev)

        def dequant_attend(i):
            kdq.copy_(ck[hidx, kcs[i].long()].reshape(B, HKV, N, D))
            vdq.copy_(cv[hidx, vcs[i].long()].reshape(B, HKV, N, D))
            qq = (q.float().view(B, HKV, HQ // HKV, D) * lam.view(1, HKV, 1, D)).reshape(B, HQ, D) @ Hm
            qt.copy_(qq.view(B, HQ, 1, D).to(torch.bfloat16))
            F.scaled_dot_product_attention(qt, kdq, vdq, enable_gqa=True)
        try:
            res["dequant_sdpa_us"] = time_graph(dequant_attend, min(copies_vq, 4), max(2, args.reps // 4), stream)
        except Exception as ex:   # noqa: BLE001
            res["dequant_sdpa_us"] = None
            res["dequant_sdpa_error"] = str(ex)[:200]
        del kdq, vdq
        torch.cuda.empty_cache()

        # ---- bf16 cache: SDPA and flashinfer
        del kcs, vcs
        torch.cuda.empty_cache()
        ks = [torch.randn(B, HKV, N, D, dtype=torch.bfloat16, device=dev) for _ in range(copies_bf)]
        vs = [torch.randn(B, HKV, N, D, dtype=torch.bfloat16, device=dev) for _ in range(copies_bf)]
        q4 = q.view(B, HQ, 1, D)
        try:
            res["bf16_sdpa_us"] = time_graph(lambda i: F.scaled_dot_product_attention(q4, ks[i], vs[i], enable_gqa=True),
                                             copies_bf, args.reps, stream)
        except Exception as ex:   # noqa: BLE001
            res["bf16_sdpa_us"] = None
            res["bf16_sdpa_error"] = str(ex)[:200]
        try:
            import flashinfer
            if B == 1:
                kn = [k[0].transpose(0, 1).contiguous() for k in ks]   # [N, H_kv, D] (NHD)
                vn = [v[0].transpose(0, 1).contiguous() for v in vs]
                res["bf16_flashinfer_us"] = time_graph(
                    lambda i: flashinfer.single_decode_with_kv_cache(q[0], kn[i], vn[i]), copies_bf, args.reps, stream)
            else:
                page = 16
                npg = N // page
                kv_layout = "HND"
                wsb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
                wrap = flashinfer.BatchDecodeWithPagedKVCacheWrapper(wsb, kv_layout, use_cuda_graph=True,
                                                                     paged_kv_indptr_buffer=torch.arange(B + 1, dtype=torch.int32, device=dev) * npg,
                                                                     paged_kv_indices_buffer=torch.arange(B * npg, dtype=torch.int32, device=dev),
                                                                     paged_kv_last_page_len_buffer=torch.full((B,), page, dtype=torch.int32, device=dev))
                wrap.plan(torch.arange(B + 1, dtype=torch.int32, device=dev) * npg,
                          torch.arange(B * npg, dtype=torch.int32, device=dev),
                          torch.full((B,), page, dtype=torch.int32, device=dev), HQ, HKV, D, page,
                          q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
                # paged HND view of the contiguous cache: [B*npg, H_kv, page, D]
                kp = [k.view(B, HKV, npg, page, D).permute(0, 2, 1, 3, 4).contiguous().view(B * npg, HKV, page, D) for k in ks]
                vp = [v.view(B, HKV, npg, page, D).permute(0, 2, 1, 3, 4).contiguous().view(B * npg, HKV, page, D) for v in vs]
                del ks, vs
                torch.cuda.empty_cache()
                res["bf16_flashinfer_us"] = time_graph(lambda i: wrap.run(q, (kp[i], vp[i])), copies_bf, args.reps, stream)
        except Exception as ex:   # noqa: BLE001
            res["bf16_flashinfer_us"] = None
            res["bf16_flashinfer_error"] = str(ex)[:300]
        for k in ("bf16_sdpa_us", "bf16_flashinfer_us", "dequant_sdpa_us"):
            if res.get(k):
                res["speedup_vs_" + k[:-3]] = res[k] / res["vecinfer_us"]
        res["vecinfer_GBps_codes"] = code_bytes / res["vecinfer_us"] / 1e3
        if res.get("bf16_flashinfer_us"):
            res["flashinfer_GBps_bf16"] = bf16_bytes / res["bf16_flashinfer_us"] / 1e3
        if res.get("bf16_sdpa_us"):
            res["sdpa_GBps_bf16"] = bf16_bytes / res["bf16_sdpa_us"] / 1e3
        print(json.dumps(res), flush=True)
        out.append(res)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
