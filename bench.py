#!/usr/bin/env python
"""Benchmark of the VecInfer decode-attention hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2|cfg3|cfg4|cfg5-b1d4|...]
    python bench.py --impl reference ...      # the CPU oracle arm (test infrastructure, timed as-is)

One STEP = one decoded token through the attention of all 32 Llama-3.1-8B layers: per layer, the
new token's k, v are encoded into the VQ cache (vecinfer_encode_kv, Eq. 9) and the G=4-grouped
decode attention runs over the whole cache (vecinfer_attn_decode: query transform + fused
dequant-MMA attention + split LSE merge, Eq. 10 / Alg. 1).  Each layer owns its own code cache, so a
step streams 32 distinct caches (512 MiB at configs[1]) -- larger than the 126 MB L2, no flush
needed.  The step is captured in a CUDA graph (the launch-bound inner loop; 2 kernels/layer).
Timing: W untimed warm-up steps, then EXACTLY K steps bracketed by barrier + synchronize, CUDA
events on the launching stream, max over ranks.  value = compressed-KV bytes of all ranks / time.
The new token is written at row N-1 every step so every timed step does identical work.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VQ decode-attn µs/step & HBM GB/s (% peak), Llama-3.1-8B b2d4, 1–8×B200"
H_Q, H_KV, D, LAYERS = 32, 8, 128, 32

WORKLOADS = {
    # name: (batch, seq_len, kbits, vbits, description)
    "cfg1": (1, 1024, 8, 8, "configs[0]: 1 batch, seq 1024, b2d4 (all 8 KV heads)"),
    "cfg2": (1, 32768, 8, 8, "configs[1]: Llama-3.1-8B b2d4, batch 1, seq 32k, 1xB200"),
    "cfg3": (64, 8192, 8, 8, "configs[2]: Llama-3.1-8B b2d4, batch 64, seq 8k (per-rank batch slice at N>1)"),
    "cfg4": (1, 196608, 8, 8, "configs[3]: Llama-3.1-8B b2d4, batch 1, seq 196k (sequence-sharded at N>1)"),
    "cfg5-b1d4": (1, 65536, 4, 4, "configs[4]: bit-width sweep, b1d4 (16 centroids), seq 64k"),
    "cfg5-b2d4": (1, 65536, 8, 8, "configs[4]: bit-width sweep, b2d4 (256 centroids), seq 64k"),
    "cfg5-b4d4": (1, 65536, 16, 16, "configs[4]: bit-width sweep, b4d4 (65536 centroids, shared codebook), seq 64k"),
}
CB_NAME = {4: "b1d4", 8: "b2d4", 16: "b4d4"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_codebooks():
    import synth
    z = np.load(os.path.join(ROOT, "data", "llama8b_synth_codebooks.npz"))
    out = {"lambda": z["lambda"], "inv_lambda": z["inv_lambda"]}
    for k in z.files:
        if k[:3] in ("ck_", "cv_"):
            out[k] = synth.bf16_from_bits(z[k])
    return out


# ------------------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int, period_s: float = 0.002):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------ CPU oracle arm
def _oracle_worker(job):
    """One host process of the CPU oracle pool (BLAS limited to 1 thread in this process): draws its
    own seeded codes for the workload, then runs (b, h_kv) units -- the 1-token append encode and the
    decode-attention of the 4 grouped query heads over N tokens -- until `seconds` have elapsed.
    Returns (units, elapsed seconds)."""
    seconds, N, kbits, vbits, wid = job
    import synth
    from oracle import ref
    cb = load_codebooks()
    rng = np.random.default_rng(1000 + wid)
    kc = rng.integers(0, 1 << kbits, (N, 32))
    vc = rng.integers(0, 1 << vbits, (N, 32))
    ckn, cvn = f"ck_{CB_NAME[kbits]}", f"cv_{CB_NAME[vbits]}"

    def head_cb(name, h):
        return cb[name][h] if cb[name].ndim == 3 else cb[name]
    q = synth.gen_queries(1, H_Q, H_KV, D, seed=7)[0]
    knew = synth.gen_keys(1, H_KV, D, seed=7)[0, 0]
    vnew = synth.gen_values(1, H_KV, D, seed=8)[0, 0]
    units, t0 = 0, time.perf_counter()
    while True:
        h = (wid + units) % H_KV
        ref.encode_kv(knew[h], vnew[h], cb["inv_lambda"][h], head_cb(ckn, h), head_cb(cvn, h))
        ref.attention_vq(q[4 * h:4 * h + 4], cb["lambda"][h], head_cb(ckn, h), head_cb(cvn, h), kc, vc)
        units += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return units, el


def _oracle_pool_init():
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


class OraclePool:
    """The CPU oracle run as a process pool over (b, h_kv) units on all host cores (SURVEY.md
    §8(d).4): one single-threaded process per core, started (and warmed: imports, codebooks, code
    draw) once, then timed on bounded samples.  `cores` = processes actually used."""

    def __init__(self, procs: int | None = None):
        import concurrent.futures as cf
        import multiprocessing as mp
        self.procs = procs or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()) or 1
        self.ex = cf.ProcessPoolExecutor(self.procs, mp_context=mp.get_context("spawn"), initializer=_oracle_pool_init)

    def sample(self, seconds: float, N: int, kbits: int = 8, vbits: int = 8):
        """Every process runs units for `seconds`; returns (units, wall seconds = slowest process)."""
        res = list(self.ex.map(_oracle_worker, [(seconds, N, kbits, vbits, w) for w in range(self.procs)]))
        return sum(u for u, _ in res), max(e for _, e in res)

    def close(self):
        self.ex.shutdown()


def run_reference(args, rank, world):
    """--impl reference: the oracle timed on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    B, N, kbits, vbits, desc = WORKLOADS[args.workload]
    unit_bytes = N * (4 * kbits + 4 * vbits)
    pool = OraclePool()
    for _ in range(max(1, args.warmup)):
        pool.sample(0.0, N, kbits=kbits, vbits=vbits)     # spawn + imports + first unit, untimed
    units, secs = 0, 0.0
    for _ in range(args.steps):
        u, s = pool.sample(args.ref_step_seconds, N, kbits=kbits, vbits=vbits)
        units += u
        secs += s
    pool.close()
    threads = pool.procs
    gbs = units * unit_bytes / secs / 1e9
    step_ms = secs / max(args.steps, 1) * 1e3
    sample = (f"{units} (b,h_kv) units of N={N} tokens (4 grouped q-heads each, + 1-token append encode) "
              f"over {args.steps} steps of ~{args.ref_step_seconds}s, {threads} single-threaded oracle processes "
              f"(one per host core, NumPy fp64)")
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if (args.workload == "cfg4" and world > 1) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "desc": desc, "global_batch": B, "seq_len": N},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import synth
    from paper_2510_06175_b200 import vecinfer as vi
    from paper_2510_06175_b200.sharding import (P2PExchange, XRankWindows, batch_shard, gather_partials_packed,
                                                shard_range)

    dev = torch.device("cuda", local_rank if args.backend == "nccl" else local_rank % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    B_glob, N, kbits, vbits, desc = WORKLOADS[args.workload]
    seq_sharded = args.workload == "cfg4" and world > 1
    if args.workload == "cfg3" and world > 1:
        b0, b1 = batch_shard(B_glob, rank, world)
        B = b1 - b0
    else:
        B = B_glob
    tok0, tok1 = shard_range(N, rank, world) if seq_sharded else (0, N)
    L = args.layers
    cb = load_codebooks()
    lam = torch.from_numpy(cb["lambda"]).to(dev)
    inv = torch.from_numpy(cb["inv_lambda"]).to(dev)
    ck = torch.from_numpy(cb[f"ck_{CB_NAME[kbits]}"]).to(dev).to(torch.bfloat16)
    cv = torch.from_numpy(cb[f"cv_{CB_NAME[vbits]}"]).to(dev).to(torch.bfloat16)
    cfgs = {4: vi.B1D4, 8: vi.B2D4, 16: vi.B4D4}
    kcfg, vcfg = cfgs[kbits], cfgs[vbits]
    unit_bytes = 4 * kbits + 4 * vbits          # K + V code bytes per cached (token, KV head)

    # ---- prefill: bulk-encode synthetic keys/values of one layer (Eq. 8), replicate per layer
    n_local = tok1 - tok0
    t_gen = time.perf_counter()
    kc0 = torch.empty(B, H_KV, n_local, kcfg.row_bytes, dtype=torch.uint8, device=dev)
    vc0 = torch.empty(B, H_KV, n_local, vcfg.row_bytes, dtype=torch.uint8, device=dev)
    enc_ws = vi.encode_workspace(B, 4096, H_KV, kcfg, vcfg, device=dev)
    chunk = 4096
    # the synthetic rows of every chunk are generated and moved to the device first; the encode of
    # all chunks is then timed back to back after one warm-up launch (steady state, no host work
    # or first-launch module loading inside the events)
    chunks = []
    for c0 in range(0, n_local, chunk):
        c1 = min(c0 + chunk, n_local)
        k = torch.from_numpy(synth.gen_keys(c1 - c0, H_KV, D, seed=1000 * rank + c0, batch=B)).to(dev).to(torch.bfloat16)
        v = torch.from_numpy(synth.gen_values(c1 - c0, H_KV, D, seed=7 + 1000 * rank + c0, batch=B)).to(dev).to(torch.bfloat16)
        chunks.append((k, v, torch.full((B,), c0, dtype=torch.int32, device=dev)))
    vi.encode_kv(*chunks[0][:2], inv, ck, cv, kc0, vc0, chunks[0][2], kcfg, vcfg, workspace=enc_ws)   # warm-up
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for k, v, wp in chunks:
        vi.encode_kv(k, v, inv, ck, cv, kc0, vc0, wp, kcfg, vcfg, workspace=enc_ws)
    ev1.record()
    ev1.synchronize()
    prefill_ms = ev0.elapsed_time(ev1)
    del chunks
    prefill_tok_s = B * n_local / (prefill_ms / 1e3)
    # ALU roofline of the encode: the pinned distance costs 4 sub + 4 mul + 3 add per (sub-vector,
    # centroid) pair at 128 fp32 lanes/clk/SM (N2)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    # 4/8-bit books: the full pinned scan on the fp32 ALU; 16-bit books (65 536 entries): the
    # tensor-core filter bounds the encode -- one mma.sync m16n8k16 per 128 (sub-vector, centroid)
    # pairs at the measured 0.465 HMMA/clk/SM (profiles/r01_ubench_hmma_lds_hbm.txt); the exact
    # rescans of the selected chunks are counted as overhead
    pairs16 = sum(1 << b for b in (kbits, vbits) if b == 16)
    pairs_alu = sum(1 << b for b in (kbits, vbits) if b != 16)
    tok_t = H_KV * (D // 4) * (pairs_alu * 11 / (128 * n_sm * 1.965e9) + pairs16 / (128 * 0.465 * n_sm * 1.965e9))
    prefill_bound = "mma.sync filter (HMMA rate)" if pairs16 else "fp32 ALU (pinned distance)"
    prefill_alu_frac = prefill_tok_s * tok_t
    kcs = [kc0] + [kc0.clone() for _ in range(L - 1)]
    vcs = [vc0] + [vc0.clone() for _ in range(L - 1)]
    # cache layout seen by the kernels: rows [0, n_local) of this rank's shard
    R = args.residual if not seq_sharded else 0
    seq_lens = torch.full((B,), n_local - R, dtype=torch.int32, device=dev)
    if R:   # full-precision window: the newest R tokens as raw bf16 rows (per layer), kept at R rows
        kres = [torch.from_numpy(synth.gen_keys(R, H_KV, D, seed=500 + l, batch=B)).to(dev).to(torch.bfloat16)
                .permute(0, 2, 1, 3).contiguous() for l in range(L)]
        vres = [torch.from_numpy(synth.gen_values(R, H_KV, D, seed=600 + l, batch=B)).to(dev).to(torch.bfloat16)
                .permute(0, 2, 1, 3).contiguous() for l in range(L)]
        res_lens = torch.full((B,), R, dtype=torch.int32, device=dev)
    owns_tail = (not seq_sharded) or (tok1 == N)
    write_pos = torch.full((B,), n_local - 1, dtype=torch.int32, device=dev)
    q_all = torch.from_numpy(np.stack([synth.gen_queries(B, H_Q, H_KV, D, seed=50 + l) for l in range(L)])).to(dev).to(torch.bfloat16)
    kn_all = torch.from_numpy(np.stack([synth.gen_keys(1, H_KV, D, seed=90 + l, batch=B) for l in range(L)])).to(dev).to(torch.bfloat16)
    vn_all = torch.from_numpy(np.stack([synth.gen_values(1, H_KV, D, seed=91 + l, batch=B) for l in range(L)])).to(dev).to(torch.bfloat16)
    gen_s = time.perf_counter() - t_gen

    o_all = torch.empty(L, B, H_Q, D, dtype=torch.bfloat16, device=dev)
    lse_all = torch.empty(L, B, H_Q, dtype=torch.float32, device=dev)
    o_part = torch.empty(L, B, H_Q, D, dtype=torch.float32, device=dev) if seq_sharded else None
    S = vi.attn_num_splits(B, H_KV, n_local, 0)
    ws = [vi.decode_step_workspace(B, H_Q, H_KV, n_local, kcfg, vcfg, device=dev) for _ in range(L)]
    stream = torch.cuda.Stream(device=dev)

    fused = not args.unfused and not seq_sharded
    # launches of one vecinfer_decode_step (the library decides whether the append is fused)
    fused_launch = fused and vi.decode_step_launches(B, H_KV, n_local, kcfg, vcfg, residual_append=bool(R)) == 1
    kernel_kind = vi.attn_kernel_kind(B, H_KV, n_local)

    # VECINFER_ATTN_FLAG_EARLY_CACHE: seq_lens / write_pos and layer l's cache are never written by
    # the kernel right before layer l's launch (that is layer l-1's, or an H2D copy), so the split
    # kernel may read them and issue its first code tile before the PDL wait
    EC = not args.no_early_cache

    def layer(l, ev_pair=None):
        if fused and R:   # one launch: the new token goes to residual row R-1, attention over codes + window
            vi.decode_step(q_all[l], kn_all[l][:, 0], vn_all[l][:, 0], lam, inv, ck, cv, kcs[l], vcs[l], write_pos,
                           seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l], lse=lse_all[l], workspace=ws[l],
                           k_res=kres[l], v_res=vres[l], res_lens=res_lens, append_to_residual=True, early_cache=EC)
            return
        if fused:   # one launch: append-encode of the new token + attention (vecinfer_decode_step)
            vi.decode_step(q_all[l], kn_all[l][:, 0], vn_all[l][:, 0], lam, inv, ck, cv, kcs[l], vcs[l], write_pos,
                           seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l], lse=lse_all[l], workspace=ws[l],
                           early_cache=EC)
            return
        if owns_tail:
            vi.encode_kv(kn_all[l], vn_all[l], inv, ck, cv, kcs[l], vcs[l], write_pos, kcfg, vcfg, workspace=enc_ws)
        if ev_pair is not None:
            ev_pair[0].record()
        ec = EC and not owns_tail   # an encode_kv launched right before writes this layer's cache
        if seq_sharded and xrw is not None:   # attention + cross-rank merge in one launch
            vi.attn_decode(q_all[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l],
                           lse=lse_m[l], workspace=ws[l], early_cache=ec, xr=xrw)
        elif seq_sharded:
            vi.attn_decode(q_all[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_part[l],
                           lse=lse_all[l], workspace=ws[l], early_cache=ec)
        else:
            vi.attn_decode(q_all[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l],
                           lse=lse_all[l], workspace=ws[l], early_cache=ec)
        if ev_pair is not None:
            ev_pair[1].record()
        if seq_sharded and xrw is None:   # layer l's output feeds layer l+1: its partials are exchanged right away
            exchange_layer(l)

    # sequence-sharded exchange, once PER LAYER (16.1 KiB of partials per rank and layer at B = 1):
    # the fused peer-memory kernel (vecinfer_merge_lse_p2p: remote stores into every rank's IPC
    # window + flags + rank-order merge, one launch, graph-safe) or NCCL all-gather of the packed
    # partials + vecinfer_merge_lse (--exchange nccl; gloo through host copies for 1-GPU checks)
    p2p, p2p_fallback, xrw = None, None, None
    if seq_sharded and args.exchange == "xr":
        # the cross-rank merge fused INTO the attention launch (vecinfer_attn_decode_xr): each CTA
        # stores its rank-merged slice into every rank's window and merges the P partials itself; no
        # exchange launch at all.  Same IPC windows as P2PExchange; falls back to it if mapping fails.
        ok, why = 1, None
        try:
            xrw = XRankWindows(B * H_Q, D, dev)
        except Exception as ex:   # noqa: BLE001 -- reported in the line
            ok, why = 0, f"{type(ex).__name__}: {ex}"
        t_ok = torch.tensor([ok], dtype=torch.int32, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
        if int(t_ok.item()) == 0:
            if xrw is not None:
                xrw.close()
                xrw = None
            args.exchange = "p2p"
            p2p_fallback = why or "a peer rank could not map the fused-merge windows"
    if seq_sharded and args.exchange == "p2p":
        # the peer windows need CUDA IPC + peer access between the ranks' GPUs; if the platform
        # refuses (on every rank alike: the outcome is all-reduced), run the all-gather exchange
        ok, why = 1, None
        try:
            p2p = P2PExchange(B * H_Q, D, dev)
        except Exception as ex:   # noqa: BLE001 -- reported in the line
            ok, why = 0, f"{type(ex).__name__}: {ex}"
        t_ok = torch.tensor([ok], dtype=torch.int32, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
        if int(t_ok.item()) == 0:
            if p2p is not None:
                p2p.close()
                p2p = None
            args.exchange = "nccl"
            p2p_fallback = (p2p_fallback + "; " if p2p_fallback else "") + (why or "a peer rank could not map the P2P windows")
    lse_m = torch.empty(L, B, H_Q, dtype=torch.float32, device=dev) if seq_sharded else None

    def exchange_layer(l):
        if p2p is not None:
            p2p.merge(o_part[l], lse_all[l], out=o_all[l], lse=lse_m[l])
            return
        if args.backend == "gloo":
            o_g, l_g = gather_partials_packed(o_part[l].cpu(), lse_all[l].cpu())
            o_g, l_g = o_g.to(dev), l_g.to(dev)
        else:
            o_g, l_g = gather_partials_packed(o_part[l], lse_all[l])
        vi.merge_lse(o_g.contiguous(), l_g.contiguous(), o_dtype=torch.bfloat16, out=o_all[l], lse=lse_m[l])

    def step_eager(evs=None):
        for l in range(L):
            layer(l, None if evs is None else evs[l])

    # 16-bit append: one centroid-split search launch (finalised in-kernel) up to 4096 token-heads
    append_kernels = 2 if (max(kbits, vbits) == 16 and B * H_KV > 4096) else 1
    if fused:
        launches_per_step = L * vi.decode_step_launches(B, H_KV, n_local, kcfg, vcfg, residual_append=bool(R))
    else:
        # + one exchange per layer when sequence-sharded (the P2P kernel; NCCL's own kernels and
        # merge_lse with --exchange nccl: 1 of ours)
        launches_per_step = L * ((append_kernels if owns_tail else 0) + 1 + (1 if seq_sharded and xrw is None else 0))

    # ---- warm-up (eager) so lazy init/attributes happen outside capture
    with torch.cuda.stream(stream):
        for _ in range(2):
            step_eager()
    torch.cuda.synchronize(dev)

    # NCCL all-gather kept eager; the fused P2P exchange keeps its epoch on the device: graph-safe
    use_graph = not args.no_graph and (not seq_sharded or p2p is not None or xrw is not None)
    K, W = args.steps, args.warmup
    if use_graph:
        g_step = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step, stream=stream):
            step_eager()
        # attention-only graph (same caches, same launch configuration) for the kernel roofline
        g_attn = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_attn, stream=stream):
            for l in range(L):
                vi.attn_decode(q_all[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l],
                               lse=lse_all[l], workspace=ws[l], early_cache=EC)
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def run_steps(n):
        for _ in range(n):
            if use_graph:
                g_step.replay()
            else:
                step_eager()

    with torch.cuda.stream(stream):
        run_steps(W)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        with torch.cuda.stream(stream):
            t_start.record(stream)
            run_steps(K)
            t_end.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    elapsed_ms = t_start.elapsed_time(t_end)
    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    elapsed_ms_local = elapsed_ms
    elapsed_ms = max_over_ranks(elapsed_ms)

    # ---- dominant kernel (vecinfer_attn_decode) timed alone: K replays of the 32-layer attention
    # graph on the launching stream; per-launch time = total / (K * L) (inter-kernel gaps included)
    attn_ms = []
    if use_graph:
        with torch.cuda.stream(stream):
            g_attn.replay()
            for _ in range(K):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                g_attn.replay()
                a1.record(stream)
                attn_ms.append((a0, a1))
        torch.cuda.synchronize(dev)
        attn_ms = [a0.elapsed_time(a1) / L for a0, a1 in attn_ms]
    else:
        attn_ms = [elapsed_ms / (K * L)]

    # ---- end to end through the public API: pinned host inputs -> device, eager calls, D2H read
    # a layer's inputs (q | k_new | v_new, bf16) are one slot of a packed pinned host buffer and of
    # its device twin, so a chunk of layers is ONE host-to-device copy
    nq, nk, nv = q_all[0].numel(), kn_all[0].numel(), vn_all[0].numel()
    h_in = torch.cat([q_all.reshape(L, nq), kn_all.reshape(L, nk), vn_all.reshape(L, nv)], dim=1).cpu().pin_memory()
    d_in = torch.empty_like(h_in, device=dev)
    q_d = [d_in[l, :nq].view(q_all.shape[1:]) for l in range(L)]
    kn_d = [d_in[l, nq:nq + nk].view(kn_all.shape[1:]) for l in range(L)]
    vn_d = [d_in[l, nq + nk:].view(vn_all.shape[1:]) for l in range(L)]
    o_h = torch.empty(o_all.shape, dtype=o_all.dtype).pin_memory()

    def layer_e2e(l):
        if fused:
            vi.decode_step(q_d[l], kn_d[l][:, 0], vn_d[l][:, 0], lam, inv, ck, cv, kcs[l], vcs[l], write_pos,
                           seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l], lse=lse_all[l], workspace=ws[l],
                           early_cache=EC, **({"k_res": kres[l], "v_res": vres[l], "res_lens": res_lens,
                                               "append_to_residual": True} if R else {}))
            return
        if owns_tail:
            vi.encode_kv(kn_d[l], vn_d[l], inv, ck, cv, kcs[l], vcs[l], write_pos, kcfg, vcfg, workspace=enc_ws)
        ec = EC and not owns_tail
        if seq_sharded and xrw is not None:
            vi.attn_decode(q_d[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l],
                           lse=lse_m[l], workspace=ws[l], early_cache=ec, xr=xrw)
        elif seq_sharded:
            vi.attn_decode(q_d[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_part[l],
                           lse=lse_all[l], workspace=ws[l], early_cache=ec)
            exchange_layer(l)
        else:
            vi.attn_decode(q_d[l], lam, ck, cv, kcs[l], vcs[l], seq_lens, kcfg=kcfg, vcfg=vcfg, out=o_all[l],
                           lse=lse_all[l], workspace=ws[l], early_cache=ec)

    def layers_e2e():
        for l in range(L):
            layer_e2e(l)

    # Pipelined end-to-end step (graph path): the H2D copies of q / k_new / v_new are issued in
    # chunks of 8 layers on a copy stream, a chunk's launches wait only for its own inputs, and the
    # D2H of a chunk's o starts as soon as its last layer is done (third stream), so the PCIe
    # transfers overlap the attention of the other chunks.  Every step still copies all its inputs and reads back all
    # of o inside the timed region, and the host synchronises on the step's result.
    pipelined = use_graph and not seq_sharded
    cs_in = torch.cuda.Stream(device=dev) if pipelined else None
    cs_out = torch.cuda.Stream(device=dev) if pipelined else None

    # layer chunks, one packed copy each per direction.  Every chunk boundary is a cross-stream
    # dependency in the graph (the layer waits for its copy, the copy for its layer), which costs more
    # than the overlap gains when the copies are small: at cfg2 (12 KiB of inputs per layer) two
    # copies per direction, split so that only layer 0's inputs and layer 31's output are exposed, are
    # fastest (scripts/exp_e2e.py: 0.4353 ms/step vs 0.4375 for two halves, 0.440 with 1 chunk,
    # 0.443-0.463 with 4); large batches (>= 256 KiB per layer, e.g. cfg3) overlap more with 8 chunks
    if h_in[0].numel() * h_in.element_size() >= 256 * 1024 and L % 8 == 0:
        chunks_in = [(c * L // 8, (c + 1) * L // 8) for c in range(8)]
        chunks_out = chunks_in
    elif L > 1:   # small inputs: layer 0's own copy, then the rest; the last layer's output on its own
        chunks_in, chunks_out = [(0, 1), (1, L)], [(0, L - 1), (L - 1, L)]
    else:
        chunks_in = chunks_out = [(0, L)]

    def step_e2e_pipelined_body():
        ev_in = [torch.cuda.Event() for _ in chunks_in]
        cur = torch.cuda.current_stream(dev)
        cs_in.wait_stream(cur)
        cs_out.wait_stream(cur)
        with torch.cuda.stream(cs_in):
            for c, (a, b) in enumerate(chunks_in):
                d_in[a:b].copy_(h_in[a:b], non_blocking=True)
                ev_in[c].record(cs_in)
        first_of = {a: c for c, (a, b) in enumerate(chunks_in)}
        last_of = {b - 1: (a, b) for (a, b) in chunks_out}
        for l in range(L):
            if l in first_of:
                cur.wait_event(ev_in[first_of[l]])
            layer_e2e(l)
            if l in last_of:
                a, b = last_of[l]
                ev = torch.cuda.Event()
                ev.record(cur)
                with torch.cuda.stream(cs_out):
                    cs_out.wait_event(ev)
                    o_h[a:b].copy_(o_all[a:b], non_blocking=True)
        cur.wait_stream(cs_in)
        cur.wait_stream(cs_out)

    g_e2e = None
    if pipelined:   # the serving pattern: copies + the 32 layer calls captured once, replayed per token
        with torch.cuda.stream(stream):
            step_e2e_pipelined_body()
        torch.cuda.synchronize(dev)
        g_e2e = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_e2e, stream=stream):
            step_e2e_pipelined_body()

    done_ev = torch.cuda.Event()

    def step_e2e():
        if g_e2e is not None:
            g_e2e.replay()
        else:
            d_in.copy_(h_in, non_blocking=True)
            layers_e2e()
            o_h.copy_(o_all, non_blocking=True)
        # the host waits for the step's result (o in pinned host memory) by polling an event: a
        # serving loop spins here rather than sleeping in cudaStreamSynchronize
        done_ev.record(torch.cuda.current_stream(dev))
        while not done_ev.query():
            pass


    with torch.cuda.stream(stream):
        for _ in range(max(1, W)):
            step_e2e()
        barrier()
        e0 = time.perf_counter()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0e.record(stream)
        for _ in range(K):
            step_e2e()
        t1e.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = t0e.elapsed_time(t1e)
    e2e_ms = max_over_ranks(e2e_ms)
    # per-rank evidence (every rank's own device time, device identity and process group backend)
    rank_info = {"rank": rank, "step_ms": elapsed_ms_local / K, "device": torch.cuda.get_device_name(dev),
                 "pci_bus_id": torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(
                     torch.cuda.get_device_properties(dev), "pci_bus_id") else None, "cuda_device": dev.index}
    ranks = [rank_info]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, rank_info)
    p2p_err = int(p2p.err.item()) if p2p is not None else (int(xrw.err.item()) if xrw is not None else 0)
    h2d = h_in.numel() * h_in.element_size()   # q, k_new, v_new of every layer (packed slots)
    d2h = o_h.numel() * 2

    if rank != 0:
        return
    # ---- figures
    # K + V bytes per layer call: codes of the quantised tokens + raw bf16 rows of the residual window
    code_bytes_rank = B * H_KV * ((n_local - R) * unit_bytes + R * 2 * D * 2)
    total_bytes = code_bytes_rank * L * K * (world if not seq_sharded else 1)
    if seq_sharded:
        total_bytes = B * H_KV * N * unit_bytes * L * K
    value = total_bytes / (elapsed_ms / 1e3) / 1e9
    e2e_value = total_bytes / (e2e_ms / 1e3) / 1e9
    peak, peak_src = load_peaks()
    attn_avg_ms = float(np.mean(attn_ms))
    traffic, ncu = None, None
    for tp in (os.path.join(ROOT, "profiles", "r02", f"attn_{args.workload}_ncu.json"),
               os.path.join(ROOT, "profiles", "r01", f"attn_{args.workload}_traffic.json")):
        if os.path.exists(tp):   # committed ncu --set full capture of this launch (scripts/ncu_summary.py)
            with open(tp) as f:
                ncu = json.load(f)
            traffic = ncu["traffic_per_launch"]   # dram__bytes_read.sum + dram__bytes_write.sum per launch
            ncu["file"] = os.path.relpath(tp, ROOT)
            break
    achieved = code_bytes_rank / (attn_avg_ms / 1e3) / 1e9
    # the binding on-chip resource: the L1/shared LSU data pipe, one wavefront
    # per clock per SM; wavefronts per unit (shared gathers + global code loads) from the ncu capture
    # per-unit cost of the main loop from the steady-state capture (18 x 8 units of 65536 tokens, one
    # split: fixed per-launch work amortised away); the launch's own capture adds its fixed costs
    # (table fill, combine, merge polls) and is reported beside it
    lsu = None
    sp = os.path.join(ROOT, "profiles", "r02", "attn_steady_ncu.json")
    if kbits == 8 and vbits == 8 and os.path.exists(sp):
        with open(sp) as f:
            steady = json.load(f)
        sm_hz = (clk.summary()["sm_mhz"] or 1965.0) * 1e6
        n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
        w = steady["lsu_wavefronts_per_unit"]
        bound = n_sms * sm_hz / w * unit_bytes / 1e9
        lsu = {"wavefronts_per_unit": w, "shared_per_unit": steady["lsu_shared_wavefronts_per_unit"],
               "global_per_unit": steady["lsu_global_wavefronts_per_unit"], "bound_gbs": bound,
               "frac": achieved / bound, "steady_capture": os.path.relpath(sp, ROOT),
               "launch_wavefronts_per_unit": ncu.get("lsu_wavefronts_per_unit") if ncu else None,
               "launch_lsu_pipe_pct": ncu.get("lsu_pipe_pct") if ncu else None,
               "note": "LSU data-pipe ceiling = #SMs x SM clock x 1 wavefront/clk / main-loop wavefronts per unit "
                       "x bytes per unit (DESIGN.md section 5)"}
    gather = None
    if kbits == 16 and vbits == 16:   # b4d4: the codebook gathers run through L1/L2 (scripts/ubench_gather16.cu)
        clk_per_unit = 59.0           # measured gather bound, profiles/r02/ubench_gather16_b4d4.txt
        sm_hz = (clk.summary()["sm_mhz"] or 1965.0) * 1e6
        n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
        gbound = n_sms * sm_hz / clk_per_unit * unit_bytes / 1e9
        gather = {"bound_gbs": gbound, "frac": achieved / gbound, "clk_per_unit": clk_per_unit,
                  "source": "profiles/r02/ubench_gather16_b4d4.txt (random 8-B gathers from two 512 KiB books, "
                            "attention launch shape, codes streamed from HBM)"}
    step_ms = elapsed_ms / K
    cpu = None
    if not args.no_cpu_baseline:
        pool = OraclePool()
        pool.sample(0.0, N, kbits=kbits, vbits=vbits)        # warm the processes (untimed)
        units, secs = pool.sample(args.cpu_seconds, N, kbits=kbits, vbits=vbits)
        pool.close()
        cpu = {"value": units * N * unit_bytes / secs / 1e9, "unit": "GB/s", "cores": pool.procs, "kind": "oracle",
               "sample": f"{units} (b,h_kv) units x {N} tokens (4 grouped q-heads each + 1-token append encode) "
                         f"in {secs:.1f}s by {pool.procs} single-threaded oracle processes (process pool, one per "
                         f"host core; NumPy fp64)"}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong" if seq_sharded else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.workload, "desc": desc, "global_batch": B_glob, "seq_len": N,
                   "layers_per_step": L, "q_heads": H_Q, "kv_heads": H_KV, "head_dim": D, "codebook": f"K-{CB_NAME[kbits]}/V-{CB_NAME[vbits]}",
                   "parallelism": ("seq-shard" if seq_sharded else "dp") + str(world),
                   "exchange": ((("xr: cross-rank merge fused into the attention launch (vecinfer_attn_decode_xr)"
                                  if args.exchange == "xr" else "p2p-fused-merge" if args.exchange == "p2p" else
                                  f"{args.backend}-allgather+merge_lse") + ", per layer (32 exchanges per step)")
                                if seq_sharded else None),
                   "l2": f"inputs larger than L2: {L} distinct layer caches = {code_bytes_rank * L / 2**20:.0f} MiB/rank per step",
                   "num_splits": S, "attn_kernel": kernel_kind, "cuda_graph": use_graph, "residual_window": R, "fused_append": fused_launch, "early_cache": EC,
                   "dtype_detail": "u8 codes, bf16 q/k/v/o, fp16 hi/lo MMA operands, f32 accumulate",
                   "step": "DESIGN.md R16: one decoded token through the attention of all 32 layers (per layer: "
                           "append-encode of the new token + attention, one fused vecinfer_decode_step launch "
                           "when possible); SURVEY c.2's single attention-layer call = roofline.attn_us_avg",
                   "attn_timing_pattern": "back-to-back layer launches in one CUDA graph with programmatic "
                                          "dependent launch (the next layer's static prologue may overlap this "
                                          "layer's tail; its dynamic reads wait for completion)"},
        "us_per_layer_call": step_ms * 1e3 / L,
        "tokens_per_s": B_glob * 1e3 / step_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "kernel": ("attn_stream_kernel<KB,VB> (stream partition, attn_stream.cu)" if kernel_kind == "stream"
                                else "attn_mma_kernel<KB,VB> (split-KV, attn_mma.cu)") +
                               " via vecinfer_attn_decode / vecinfer_decode_step",
                     "attn_us_avg": attn_avg_ms * 1e3, "attn_us_p10": float(np.percentile(attn_ms, 10)) * 1e3,
                     "attn_us_p90": float(np.percentile(attn_ms, 90)) * 1e3,
                     "timing": "CUDA events around K replays of a graph of the 32 layers' vecinfer_attn_decode launches "
                               "(launching stream), per-launch = total/(K*32), inter-kernel gaps included",
                     "algorithmic_bytes_per_launch": code_bytes_rank, "peak_source": peak_src,
                     "lsu_bound": lsu, "gather_bound": gather},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_ms / K, "api": ("32 x vecinfer.decode_step + pinned H2D / D2H copies in 2 chunks per direction (layer 0 | layers 1-31 in, layers 0-30 | layer 31 out; 8 chunks at >= 256 KiB of inputs per layer; packed copies) pipelined on two copy streams, one CUDA graph per step, host waits on the result (event poll); " if g_e2e is not None else "32 eager vecinfer calls, ")
                       + "pinned H2D of q/k/v and D2H of o every step"},
        "gpu_launches": launches_per_step * K,
        "ranks": ranks if world > 1 else None,
        "dist": ({"backend": args.backend, "world": world, "p2p_timeout_flag": p2p_err, "p2p_fallback": p2p_fallback,
                  "nccl_version": (".".join(map(str, torch.cuda.nccl.version())) if args.backend == "nccl" else None),
                  "shard": f"rank r attends tokens [r*N/{world}, (r+1)*N/{world}) (32-aligned)" if seq_sharded else
                  (f"batch slice {B} of {B_glob} sequences per rank" if args.workload == "cfg3" else "replica")}
                 if world > 1 else None),
        "clocks": clk.summary(),
        "prefill_encode": {"tokens_per_s": prefill_tok_s, "alu_frac": prefill_alu_frac, "bound": prefill_bound,
                           "note": "bulk vecinfer_encode_kv, all 8 KV heads, K+V, 4096-token chunks back to back after a warm-up"},
        "setup_s": gen_s,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: cfg2 (configs[1]) at N=1; cfg4 (configs[3], 196k tokens sequence-sharded with a "
                         "per-layer exchange, strong scaling) at N>1; cfg3 = batch x head sharding (weak)")
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-early-cache", action="store_true",
                    help="launch without VECINFER_ATTN_FLAG_EARLY_CACHE (all cache reads after the PDL wait)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N>1 (gloo: ranks may share one GPU; functional check)")
    ap.add_argument("--unfused", action="store_true", help="separate encode_kv + attn_decode launches per layer")
    ap.add_argument("--residual", type=int, default=0,
                    help="full-precision residual window of R tokens (P:494: 128); the step appends into it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="xr", choices=["xr", "p2p", "nccl"],
                    help="cfg4 at N>1: merge fused into the attention launch (xr), a separate fused peer-memory "
                         "exchange+merge kernel (p2p), or NCCL all-gather + merge_lse")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=2.0)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload is None:
        args.workload = "cfg4" if world > 1 else "cfg2"
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        dev_idx = local_rank if args.backend == "nccl" else local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev_idx)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:   # gloo: functional check of the multi-rank paths on a single-GPU box
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
