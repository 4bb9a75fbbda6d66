"""Timing of the GPU codebook k-means (NEXT-3) against the CPU oracle's Lloyd step.

    python scripts/bench_kmeans.py [--iters 30]

Workloads (the codebook-fitting recipe of scripts/fit_codebooks.py, reading R18):
  * b2d4: 2^18 pinned-transformed key sub-vectors (d = 4), k = 256, up to 30 Lloyd iterations;
  * b4d4: 2^20 sub-vectors, k = 65 536 (one Lloyd step; Lloyd at this size is the reason the
    harness froze a quantile grid instead -- on the GPU it is one ~second-scale job per iteration).
The assignment is ALU-bound: per (point, centroid) pair d subtracts + d multiplies + (d - 1) adds
(pinned, no FMA) + compare/select; the reported peak is 128 fp32 lanes/clk/SM x 148 SMs x the
measured SM clock (B200_PROFILING.md unit counts).  The CPU oracle is timed on a bounded sample
(stated) on the host cores.  Prints one JSON line per workload.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2510_06175_b200 import vecinfer as vi  # noqa: E402


def key_subvectors(n_sub, seed):
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    n_tok = (n_sub + 31) // 32
    k = synth.gen_keys(n_tok, 8, 128, seed=seed)[0, :, 2]
    return np.ascontiguousarray(ref.transform_key_pinned(k, z["inv_lambda"][2]).astype(np.float32).reshape(-1, 4)[:n_sub])


def time_gpu_steps(X, C, iters):
    Xd, Cd = torch.from_numpy(X).cuda(), torch.from_numpy(C).cuda()
    Cn = torch.empty_like(Cd)
    ws = torch.empty(max(vi._lib.load().vecinfer_kmeans_workspace_bytes(C.shape[0], C.shape[1]), 256),
                     dtype=torch.uint8, device="cuda")
    vi.kmeans_step(Xd, Cd, Cn, ws)                     # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        vi.kmeans_step(Xd, Cd, Cn, ws)
        Cd, Cn = Cn, Cd
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / iters          # s per Lloyd step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    sm_mhz = 1965.0
    try:
        import pynvml
        pynvml.nvmlInit()
        sm_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM))
    except Exception:
        pass
    peak_lane_ops = 128 * 148 * sm_mhz * 1e6
    for name, n, k, iters in (("b2d4", 1 << 18, 256, args.iters), ("b4d4", 1 << 20, 65536, 2)):
        X = key_subvectors(n, seed=31)
        rng = np.random.default_rng(7)
        C = X[rng.choice(n, k, replace=False)].copy()
        t_gpu = time_gpu_steps(X, C, iters)
        evals = float(n) * k
        ops = evals * (4 + 4 + 3)                       # pinned d = 4 distance: fp32 lane ops
        # CPU oracle on a bounded sample: a prefix of the points, scaled per point
        if k <= 4096:          # the whole oracle step on a prefix of the points (n_cpu >= k)
            n_cpu = min(n, max(4 * k, int(2e7 // k)))
            t0 = time.perf_counter()
            ref.kmeans_lloyd_step(X[:n_cpu], C)
            sample = f"oracle kmeans_lloyd_step on {n_cpu} of {n} points, scaled linearly"
        else:                  # b4d4: the oracle's assignment (step 1, pinned distances) on a prefix
            n_cpu = 2048
            t0 = time.perf_counter()
            ref.pinned_sqdist(X[:n_cpu], C).argmin(1)
            sample = f"oracle step 1 (pinned-distance assignment) on {n_cpu} of {n} points, scaled linearly"
        t_cpu = (time.perf_counter() - t0) * n / n_cpu
        print(json.dumps({
            "workload": f"kmeans {name}: n={n} sub-vectors (d=4), k={k}", "metric": "s per Lloyd step",
            "gpu_s_per_step": t_gpu, "gpu_steps_timed": iters, "evals_per_s": evals / t_gpu,
            "roofline": {"bound": "alu", "achieved": ops / t_gpu / 1e12, "peak": peak_lane_ops / 1e12,
                         "unit": "T fp32 lane-ops/s", "frac": ops / t_gpu / peak_lane_ops,
                         "peak_source": f"128 fp32 lanes/clk/SM x 148 SMs x {sm_mhz:.0f} MHz"},
            "cpu_baseline": {"s_per_step": t_cpu, "kind": "oracle", "cores": os.cpu_count(),
                             "sample": sample},
            "gpu_vs_cpu": t_cpu / t_gpu}), flush=True)


if __name__ == "__main__":
    main()
