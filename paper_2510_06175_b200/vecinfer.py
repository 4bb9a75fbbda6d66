"""Thin PyTorch binding of the libvecinfer C ABI (argument marshalling only).

Every step of the hot path runs in the CUDA kernels behind include/vecinfer.h; this module only
checks dtypes/devices, allocates outputs/workspaces with torch (device memory is PyTorch's job),
and passes raw pointers plus torch's current CUDA stream.  There is no CPU fallback: CPU tensors
are rejected and a missing library raises at import.
Names follow the C ABI: calibrate_smooth, encode_kv, attn_decode, merge_lse.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import VQ, I64x2, I64x3, Paged, Residual, check

_lib.load()   # fail loudly at import if the native library is missing

BF16, F32 = 0, 1
ALGOS = {"auto": 0, "mma": 1, "dequant_mma": 1, "lut": 2, "stream": 3, "dequant_mma_stream": 3, "tc": 4, "dequant_tc": 4}
EARLY_CACHE = 0x100   # VECINFER_ATTN_FLAG_EARLY_CACHE (ABI v7), OR-ed into the algo argument


@dataclass(frozen=True)
class VQConfig:
    """Product-VQ config; b2d4 = VQConfig(128, 4, 8) (BASELINE notation bXdY = paper d{Y}b{X*Y})."""
    head_dim: int = 128
    sub_dim: int = 4
    code_bits: int = 8

    @property
    def n_sub(self) -> int:
        return self.head_dim // self.sub_dim

    @property
    def row_bytes(self) -> int:
        return self.n_sub * self.code_bits // 8

    @property
    def n_entries(self) -> int:
        return 1 << self.code_bits

    def c(self) -> VQ:
        return VQ(self.head_dim, self.sub_dim, self.code_bits)


B1D4, B2D4, B4D4 = VQConfig(128, 4, 4), VQConfig(128, 4, 8), VQConfig(128, 4, 16)
# the paper's other configurations, D = 128,
# split kernel: each with itself, plus K-d4b10 / V-d8b12 (2-bit) and K-d8b12 / V-d8b8 (1.25-bit)
D8B8, D8B12, D4B10, D2B8 = VQConfig(128, 8, 8), VQConfig(128, 8, 12), VQConfig(128, 4, 10), VQConfig(128, 2, 8)
D8B16 = VQConfig(128, 8, 16)   # Table 5's 2-bit row: 65 536 eight-dim centroids


def _stream(dev: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _need(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.stride(-1) != 1:
        raise ValueError(f"{name}: innermost dimension must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _cb_stride(cb: torch.Tensor) -> int:
    """[H_kv, 2^b, d] -> elements between heads; [2^b, d] (shared) -> 0."""
    return 0 if cb.dim() == 2 else cb.stride(0)


def _paged(block_table, codes):
    """vecinfer_paged_t for a paged code pool codes [n_pages, H_kv, page_size, row] and an int32
    block table [B, pages_per_seq]; returns (pointer, n_cap)."""
    if block_table.dim() != 2 or block_table.stride(1) != 1:
        raise ValueError("block_table must be [B, pages_per_seq] with contiguous rows")
    n_pages, _, page_size, _ = codes.shape
    pg = Paged(_need(block_table, "block_table", torch.int32).value, block_table.stride(0), page_size, n_pages)
    return ctypes.pointer(pg), block_table.shape[1] * page_size


def _residual(k_res, v_res, res_lens, append_new=False):
    """vecinfer_residual_t for bf16 [B, H_kv, r_cap, D] residual windows (None -> NULL)."""
    if k_res is None:
        return None
    if k_res.shape != v_res.shape or k_res.stride() != v_res.stride() or k_res.stride(2) != k_res.shape[3]:
        raise ValueError("k_res/v_res must be [B, H_kv, r_cap, D] with identical strides and contiguous rows")
    r = Residual(_need(k_res, "k_res", torch.bfloat16).value, _need(v_res, "v_res", torch.bfloat16).value,
                 k_res.stride(0), k_res.stride(1), k_res.shape[2], _need(res_lens, "res_lens", torch.int32).value,
                 1 if append_new else 0)
    return ctypes.pointer(r)


def calibrate_smooth(k_cal: torch.Tensor, eps: float = 1e-6):
    """lambda = sqrt(max |K|) per (KV head, channel) (Eq. 4).  k_cal bf16 [N, H_kv, D]."""
    N, H, D = k_cal.shape
    lam = torch.empty(H, D, dtype=torch.float32, device=k_cal.device)
    inv = torch.empty_like(lam)
    lib = _lib.load()
    nws = lib.vecinfer_calibrate_workspace_bytes(H, D)
    ws = torch.empty(max(nws, 4), dtype=torch.uint8, device=k_cal.device)
    check("vecinfer_calibrate_smooth", lib.vecinfer_calibrate_smooth(
        _need(k_cal, "k_cal", torch.bfloat16), N, H, D, k_cal.stride(0), k_cal.stride(1), eps,
        _need(lam, "lambda"), _need(inv, "inv_lambda"), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
        _stream(k_cal.device)))
    return lam, inv


def encode_workspace(B: int, T: int, H_kv: int, kcfg: VQConfig = B2D4, vcfg: VQConfig = B2D4, device="cuda"):
    n = _lib.load().vecinfer_encode_workspace_bytes(B, T, H_kv, kcfg.c(), vcfg.c())
    return torch.empty(max(n, 8), dtype=torch.uint8, device=device)


def encode_kv(k: torch.Tensor, v: torch.Tensor, inv_lambda: torch.Tensor, ck: torch.Tensor, cv: torch.Tensor,
              k_codes: torch.Tensor, v_codes: torch.Tensor, write_pos: torch.Tensor, kcfg: VQConfig = B2D4,
              vcfg: VQConfig = B2D4, err_flags: torch.Tensor | None = None,
              workspace: torch.Tensor | None = None, block_table: torch.Tensor | None = None) -> None:
    """Encode k, v [B, T, H_kv, D] (bf16) into the packed code caches [B, H_kv, n_cap, row] (uint8)
    at rows write_pos[b] + t (Eq. 8 prefill / Eq. 9 append).  With block_table [B, pages_per_seq]
    (int32) the caches are page pools [n_pages, H_kv, page_size, row] (vecinfer_encode_kv_paged)."""
    B, T, H, D = k.shape
    if v.shape != k.shape:
        raise ValueError("k and v shapes differ")
    pg = None
    if block_table is not None:
        pg, n_cap = _paged(block_table, k_codes)
        if k_codes.shape[1] != H or k_codes.shape[3] != kcfg.row_bytes or v_codes.shape != (
                k_codes.shape[0], H, k_codes.shape[2], vcfg.row_bytes):
            raise ValueError("paged code pool shape mismatch")
    else:
        n_cap = k_codes.shape[2]
        if tuple(k_codes.shape) != (B, H, n_cap, kcfg.row_bytes) or tuple(v_codes.shape) != (B, H, n_cap, vcfg.row_bytes):
            raise ValueError("code cache shape mismatch")
    if not (k_codes.is_contiguous() and v_codes.is_contiguous()):
        raise ValueError("code caches must be contiguous")
    lib = _lib.load()
    nws = lib.vecinfer_encode_workspace_bytes(B, T, H, kcfg.c(), vcfg.c())
    if nws and (workspace is None or workspace.numel() < nws):
        workspace = torch.empty(nws, dtype=torch.uint8, device=k.device)
    wsp = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else ctypes.c_void_p(0)
    wsn = workspace.numel() if workspace is not None else 0
    args = (_need(k, "k", torch.bfloat16), _need(v, "v", torch.bfloat16), B, T, H,
            I64x3(*k.stride()[:3]), I64x3(*v.stride()[:3]), _need(inv_lambda, "inv_lambda", torch.float32),
            _need(ck, "ck", torch.bfloat16), _need(cv, "cv", torch.bfloat16), _cb_stride(ck), _cb_stride(cv),
            kcfg.c(), vcfg.c(), _need(k_codes, "k_codes", torch.uint8), _need(v_codes, "v_codes", torch.uint8), n_cap,
            _need(write_pos, "write_pos", torch.int32),
            ctypes.c_void_p(err_flags.data_ptr()) if err_flags is not None else ctypes.c_void_p(0),
            wsp, wsn, _stream(k.device))
    if pg is not None:
        check("vecinfer_encode_kv_paged", lib.vecinfer_encode_kv_paged(*args, pg))
    else:
        check("vecinfer_encode_kv", lib.vecinfer_encode_kv(*args))


def attn_num_splits(B: int, H_kv: int, n_tokens_max: int, num_splits: int = 0) -> int:
    return _lib.load().vecinfer_attn_num_splits(B, H_kv, n_tokens_max, num_splits)


def attn_num_ctas(B: int, H_kv: int, n_tokens_max: int, num_splits: int = 0) -> int:
    """Virtual CTAs V of the stream partition (the grid is min(V, #SMs) persistent CTAs)."""
    return _lib.load().vecinfer_attn_num_ctas(B, H_kv, n_tokens_max, num_splits)


def attn_kernel_kind(B: int, H_kv: int, n_tokens_max: int, num_splits: int = 0, algo: str = "auto") -> str:
    """Which attention kernel a call runs: "split" (attn_mma.cu), "stream" (attn_stream.cu) or "lut"."""
    k = _lib.load().vecinfer_attn_kernel_kind(B, H_kv, n_tokens_max, num_splits, ALGOS[algo])
    return ("split", "stream", "lut")[k]


def decode_step_launches(B: int, H_kv: int, n_cap: int, kcfg: VQConfig = None, vcfg: VQConfig = None,
                         num_splits: int = 0, algo: str = "auto", residual_append: bool = False) -> int:
    """Kernel launches of one decode_step call (1: the append-encode is fused into attention)."""
    kcfg = kcfg or B2D4
    vcfg = vcfg or B2D4
    return _lib.load().vecinfer_decode_step_launches(B, H_kv, n_cap, kcfg.c(), vcfg.c(), num_splits, ALGOS[algo],
                                                     int(residual_append))


def attn_workspace(B: int, H_q: int, H_kv: int, n_tokens_max: int, num_splits: int = 0, device="cuda"):
    """Zero-filled workspace for attn_decode (counters must start at zero; the kernel resets them)."""
    n = _lib.load().vecinfer_attn_workspace_bytes(B, H_q, H_kv, 128, n_tokens_max, num_splits)
    return torch.zeros(max(n, 256), dtype=torch.uint8, device=device)


def attn_decode(q: torch.Tensor, lam: torch.Tensor, ck: torch.Tensor, cv: torch.Tensor, k_codes: torch.Tensor,
                v_codes: torch.Tensor, seq_lens: torch.Tensor, tok_begin: int = 0, tok_end: int = -1,
                softmax_scale: float | None = None, num_splits: int = 0, algo: str = "auto",
                kcfg: VQConfig = B2D4, vcfg: VQConfig = B2D4, o_dtype: torch.dtype = torch.float32,
                out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                workspace: torch.Tensor | None = None, k_res: torch.Tensor | None = None,
                v_res: torch.Tensor | None = None, res_lens: torch.Tensor | None = None,
                block_table: torch.Tensor | None = None, xr=None, early_cache: bool = False):
    """Decode attention of q [B, H_q, D] (bf16) over the VQ cache (Eq. 10 / Alg. 1), plus an optional
    full-precision residual window k_res/v_res [B, H_kv, r_cap, D] with res_lens [B].
    With block_table [B, pages_per_seq] the code caches are page pools [n_pages, H_kv, page_size, row].
    xr (sharding.XRankWindows): this rank's cache is one sequence shard; the launch merges the
    ranks' partials over peer memory itself (vecinfer_attn_decode_xr) and returns the final o, lse.
    early_cache: VECINFER_ATTN_FLAG_EARLY_CACHE (seq_lens and the codes were not written by the kernel
    just before this launch on the stream: the first code tile is read before the PDL wait).
    Returns (o [B, H_q, D] o_dtype, lse [B, H_q] fp32, natural log)."""
    B, Hq, D = q.shape
    Hkv, n_cap = k_codes.shape[1], k_codes.shape[2]
    pg = None
    if block_table is not None:
        pg, n_cap = _paged(block_table, k_codes)
    if softmax_scale is None:
        softmax_scale = D ** -0.5
    rng = n_cap if tok_end < 0 else max(0, min(tok_end - tok_begin, n_cap))
    if out is None:
        out = torch.empty(B, Hq, D, dtype=o_dtype, device=q.device)
    if lse is None:
        lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    lib = _lib.load()
    need = lib.vecinfer_attn_workspace_bytes(B, Hq, Hkv, D, rng, num_splits)
    if workspace is None or workspace.numel() < need:
        workspace = torch.zeros(max(need, 256), dtype=torch.uint8, device=q.device)
    odt = F32 if out.dtype == torch.float32 else BF16
    if out.dtype not in (torch.float32, torch.bfloat16) or not out.is_contiguous():
        raise TypeError("out must be a contiguous float32 or bfloat16 tensor")
    args = (_need(q, "q", torch.bfloat16), B, Hq, Hkv, q.stride(0), q.stride(1), _need(lam, "lambda", torch.float32),
            _need(ck, "ck", torch.bfloat16), _need(cv, "cv", torch.bfloat16), _cb_stride(ck), _cb_stride(cv),
            kcfg.c(), vcfg.c(), _need(k_codes, "k_codes", torch.uint8), _need(v_codes, "v_codes", torch.uint8), n_cap,
            _need(seq_lens, "seq_lens", torch.int32), tok_begin, tok_end, softmax_scale, num_splits,
            ALGOS[algo] | (EARLY_CACHE if early_cache else 0),
            _need(out, "out"), odt, _need(lse, "lse", torch.float32), ctypes.c_void_p(workspace.data_ptr()),
            workspace.numel(), _stream(q.device), _residual(k_res, v_res, res_lens))
    if xr is not None:
        if pg is not None:
            raise ValueError("the fused cross-rank merge runs on contiguous caches")
        check("vecinfer_attn_decode_xr", lib.vecinfer_attn_decode_xr(*args, xr.desc))
    elif pg is not None:
        check("vecinfer_attn_decode_paged", lib.vecinfer_attn_decode_paged(*args, pg))
    else:
        check("vecinfer_attn_decode", lib.vecinfer_attn_decode(*args))
    return out, lse


def decode_step(q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, lam: torch.Tensor,
                inv_lambda: torch.Tensor, ck: torch.Tensor, cv: torch.Tensor, k_codes: torch.Tensor,
                v_codes: torch.Tensor, write_pos: torch.Tensor, seq_lens: torch.Tensor,
                softmax_scale: float | None = None, num_splits: int = 0, algo: str = "auto",
                kcfg: VQConfig = B2D4, vcfg: VQConfig = B2D4, o_dtype: torch.dtype = torch.float32,
                out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                err_flags: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                k_res: torch.Tensor | None = None, v_res: torch.Tensor | None = None,
                res_lens: torch.Tensor | None = None, append_to_residual: bool = False,
                block_table: torch.Tensor | None = None, xr=None, early_cache: bool = False):
    """Fused layer decode step = encode_kv(T=1) of k_new/v_new [B, H_kv, D] at row write_pos[b]
    followed by attn_decode over [0, seq_lens[b]) -- one launch (vecinfer_decode_step).  With a
    residual window and append_to_residual, the new token is copied to residual row res_lens[b]-1
    instead (no encode) and attended from there.  early_cache: as in attn_decode (write_pos too)."""
    B, Hq, D = q.shape
    Hkv, n_cap = k_codes.shape[1], k_codes.shape[2]
    pg = None
    if block_table is not None:   # page pools [n_pages, H_kv, page_size, row]
        pg, n_cap = _paged(block_table, k_codes)
    if softmax_scale is None:
        softmax_scale = D ** -0.5
    if tuple(k_new.shape) != (B, Hkv, D) or tuple(v_new.shape) != (B, Hkv, D):
        raise ValueError("k_new/v_new must be [B, H_kv, D]")
    if out is None:
        out = torch.empty(B, Hq, D, dtype=o_dtype, device=q.device)
    if lse is None:
        lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    lib = _lib.load()
    need = lib.vecinfer_decode_step_workspace_bytes(B, Hq, Hkv, n_cap, kcfg.c(), vcfg.c(), num_splits)
    if workspace is None or workspace.numel() < need:
        workspace = torch.zeros(max(need, 256), dtype=torch.uint8, device=q.device)
    fn = lib.vecinfer_decode_step_paged if pg is not None else lib.vecinfer_decode_step
    extra = (pg,) if pg is not None else ()
    if xr is not None:   # sequence shard + fused cross-rank merge (vecinfer_decode_step_xr)
        if pg is not None:
            raise ValueError("the fused cross-rank merge runs on contiguous caches")
        fn, extra = lib.vecinfer_decode_step_xr, (xr.desc,)
    check("vecinfer_decode_step", fn(
        _need(q, "q", torch.bfloat16), _need(k_new, "k_new", torch.bfloat16), _need(v_new, "v_new", torch.bfloat16),
        B, Hq, Hkv, I64x2(q.stride(0), q.stride(1)), I64x2(k_new.stride(0), k_new.stride(1)),
        I64x2(v_new.stride(0), v_new.stride(1)), _need(lam, "lambda", torch.float32),
        _need(inv_lambda, "inv_lambda", torch.float32), _need(ck, "ck", torch.bfloat16),
        _need(cv, "cv", torch.bfloat16), _cb_stride(ck), _cb_stride(cv), kcfg.c(), vcfg.c(),
        _need(k_codes, "k_codes", torch.uint8), _need(v_codes, "v_codes", torch.uint8), n_cap,
        _need(write_pos, "write_pos", torch.int32), _need(seq_lens, "seq_lens", torch.int32), softmax_scale,
        num_splits, ALGOS[algo] | (EARLY_CACHE if early_cache else 0), _need(out, "out"),
        F32 if out.dtype == torch.float32 else BF16, _need(lse, "lse", torch.float32),
        ctypes.c_void_p(err_flags.data_ptr()) if err_flags is not None else ctypes.c_void_p(0),
        ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _stream(q.device),
        _residual(k_res, v_res, res_lens, append_to_residual), *extra))
    return out, lse


def decode_step_workspace(B: int, H_q: int, H_kv: int, n_cap: int, kcfg: VQConfig = B2D4, vcfg: VQConfig = B2D4,
                          num_splits: int = 0, device="cuda"):
    n = _lib.load().vecinfer_decode_step_workspace_bytes(B, H_q, H_kv, n_cap, kcfg.c(), vcfg.c(), num_splits)
    return torch.zeros(max(n, 256), dtype=torch.uint8, device=device)


def merge_lse(o_parts: torch.Tensor, lse_parts: torch.Tensor, o_dtype: torch.dtype = torch.float32,
              out: torch.Tensor | None = None, lse: torch.Tensor | None = None):
    """Merge P partials o_parts [P, B, H_q, D] fp32 / lse_parts [P, B, H_q] by log-sum-exp."""
    P, B, Hq, D = o_parts.shape
    if not (o_parts.is_contiguous() and lse_parts.is_contiguous()):
        raise ValueError("partials must be contiguous")
    if out is None:
        out = torch.empty(B, Hq, D, dtype=o_dtype, device=o_parts.device)
    if lse is None:
        lse = torch.empty(B, Hq, dtype=torch.float32, device=o_parts.device)
    check("vecinfer_merge_lse", _lib.load().vecinfer_merge_lse(
        _need(o_parts, "o_parts", torch.float32), _need(lse_parts, "lse_parts", torch.float32), P, B, Hq, D,
        _need(out, "out"), F32 if out.dtype == torch.float32 else BF16, _need(lse, "lse", torch.float32),
        _stream(o_parts.device)))
    return out, lse


def kmeans_step(X: torch.Tensor, C: torch.Tensor, C_new: torch.Tensor | None = None, workspace: torch.Tensor | None = None):
    """One Lloyd iteration of the codebook k-means on the GPU.

    X fp32 [n, d], C fp32 [k, d] (d in {2, 4, 8}).  Returns (C_new fp32 [k, d], assign int32 [n],
    best fp32 [n], objective fp64 [1]) -- all device tensors, nothing synchronised."""
    n, d = X.shape
    k = C.shape[0]
    if C_new is None:
        C_new = torch.empty_like(C)
    assign = torch.empty(n, dtype=torch.int32, device=X.device)
    best = torch.empty(n, dtype=torch.float32, device=X.device)
    obj = torch.empty(1, dtype=torch.float64, device=X.device)
    lib = _lib.load()
    if workspace is None:
        workspace = torch.empty(max(lib.vecinfer_kmeans_workspace_bytes(k, d), 256), dtype=torch.uint8, device=X.device)
    check("vecinfer_kmeans_step", lib.vecinfer_kmeans_step(
        _need(X, "X", torch.float32), n, d, _need(C, "C", torch.float32), k, _need(C_new, "C_new", torch.float32),
        _need(assign, "assign", torch.int32), _need(best, "best", torch.float32), _need(obj, "objective", torch.float64),
        ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _stream(X.device)))
    return C_new, assign, best, obj


def kmeans_fit(X: torch.Tensor, C0: torch.Tensor, max_iters: int = 30):
    """Lloyd iterations from the initial centroids C0 (k-means, <= 30 iterations) until the
    centroids stop changing.  Each iteration is one vecinfer_kmeans_step; the convergence test reads
    one flag back to the host.  Returns (C fp32 [k, d], objective history)."""
    C = C0.contiguous().clone()
    lib = _lib.load()
    ws = torch.empty(max(lib.vecinfer_kmeans_workspace_bytes(C.shape[0], C.shape[1]), 256), dtype=torch.uint8,
                     device=X.device)
    Cn = torch.empty_like(C)
    hist = []
    for _ in range(max_iters):
        _, _, _, obj = kmeans_step(X, C, Cn, ws)
        hist.append(obj)
        if torch.equal(Cn, C):
            break
        C, Cn = Cn, C
    return C, [float(h.item()) for h in hist]
