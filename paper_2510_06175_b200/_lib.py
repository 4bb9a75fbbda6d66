"""ctypes loader for libvecinfer.so and its C-ABI prototypes (include/vecinfer.h).

There is no fallback: if the in-tree library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VECINFER_LIB") or os.path.join(_HERE, "libvecinfer.so")

c_i32, c_i64, c_u32, c_f32, c_sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_float, ctypes.c_size_t
c_void_p, c_char_p = ctypes.c_void_p, ctypes.c_char_p
I64x3 = ctypes.c_int64 * 3
I64x2 = ctypes.c_int64 * 2


class Residual(ctypes.Structure):
    """vecinfer_residual_t: full-precision residual window (NEXT-1)."""
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p), ("stride_b", ctypes.c_int64),
                ("stride_h", ctypes.c_int64), ("r_cap", ctypes.c_int64), ("lens", ctypes.c_void_p),
                ("append_new", ctypes.c_int32)]


class Paged(ctypes.Structure):
    """vecinfer_paged_t: paged code cache [n_pages, H_kv, page_size, row] + block table."""
    _fields_ = [("block_table", ctypes.c_void_p), ("bt_stride", ctypes.c_int64), ("page_size", ctypes.c_int32),
                ("n_pages", ctypes.c_int32)]


class XRank(ctypes.Structure):
    """vecinfer_xrank_t: cross-GPU merge fused into the attention launch."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("windows", ctypes.c_void_p),
                ("rows_max", ctypes.c_int64), ("err_flags", ctypes.c_void_p)]


class VQ(ctypes.Structure):
    """vecinfer_vq_t {head_dim, sub_dim, code_bits}."""
    _fields_ = [("head_dim", c_i32), ("sub_dim", c_i32), ("code_bits", c_i32)]


STATUS = {0: "VECINFER_OK", 1: "VECINFER_ERR_INVALID_ARG", 2: "VECINFER_ERR_SHAPE", 3: "VECINFER_ERR_UNSUPPORTED",
          4: "VECINFER_ERR_EMPTY", 5: "VECINFER_ERR_RANGE", 6: "VECINFER_ERR_WORKSPACE", 7: "VECINFER_ERR_CUDA"}

# name -> (restype, argtypes); mirrors include/vecinfer.h exactly
PROTOTYPES = {
    "vecinfer_abi_version": (c_i32, []),
    "vecinfer_last_error": (c_char_p, []),
    "vecinfer_status_string": (c_char_p, [c_i32]),
    "vecinfer_calibrate_workspace_bytes": (c_sz, [c_i32, c_i32]),
    "vecinfer_kmeans_workspace_bytes": (c_sz, [c_i32, c_i32]),
    "vecinfer_p2p_window_bytes": (c_sz, [c_i32, c_i64, c_i32]),
    "vecinfer_p2p_window_create": (c_i32, [c_sz, c_void_p, c_void_p]),
    "vecinfer_p2p_window_open": (c_i32, [c_void_p, c_void_p]),
    "vecinfer_p2p_window_close": (c_i32, [c_void_p]),
    "vecinfer_p2p_window_destroy": (c_i32, [c_void_p]),
    "vecinfer_merge_lse_p2p": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_u32,
                                       c_void_p, c_i32, c_void_p, c_void_p, c_void_p]),
    "vecinfer_kmeans_step": (c_i32, [c_void_p, c_i64, c_i32, c_void_p, c_i32, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_void_p, c_sz, c_void_p]),
    "vecinfer_calibrate_smooth": (c_i32, [c_void_p, c_i64, c_i32, c_i32, c_i64, c_i64, c_f32, c_void_p, c_void_p,
                                          c_void_p, c_sz, c_void_p]),
    "vecinfer_encode_workspace_bytes": (c_sz, [c_i32, c_i32, c_i32, VQ, VQ]),
    "vecinfer_encode_kv": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_i32, I64x3, I64x3, c_void_p, c_void_p,
                                   c_void_p, c_i64, c_i64, VQ, VQ, c_void_p, c_void_p, c_i64, c_void_p, c_void_p,
                                   c_void_p, c_sz, c_void_p]),
    "vecinfer_encode_kv_paged": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_i32, I64x3, I64x3, c_void_p, c_void_p,
                                         c_void_p, c_i64, c_i64, VQ, VQ, c_void_p, c_void_p, c_i64, c_void_p,
                                         c_void_p, c_void_p, c_sz, c_void_p, ctypes.POINTER(Paged)]),
    "vecinfer_attn_num_splits": (c_i32, [c_i32, c_i32, c_i64, c_i32]),
    "vecinfer_attn_num_ctas": (c_i32, [c_i32, c_i32, c_i64, c_i32]),
    "vecinfer_attn_kernel_kind": (c_i32, [c_i32, c_i32, c_i64, c_i32, c_i32]),
    "vecinfer_decode_step_launches": (c_i32, [c_i32, c_i32, c_i64, VQ, VQ, c_i32, c_i32, c_i32]),
    "vecinfer_attn_workspace_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i32, c_i64, c_i32]),
    "vecinfer_attn_decode": (c_i32, [c_void_p, c_i32, c_i32, c_i32, c_i64, c_i64, c_void_p, c_void_p, c_void_p,
                                     c_i64, c_i64, VQ, VQ, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_i64, c_f32,
                                     c_i32, c_i32, c_void_p, c_i32, c_void_p, c_void_p, c_sz, c_void_p,
                                     ctypes.POINTER(Residual)]),
    "vecinfer_attn_decode_paged": (c_i32, [c_void_p, c_i32, c_i32, c_i32, c_i64, c_i64, c_void_p, c_void_p,
                                           c_void_p, c_i64, c_i64, VQ, VQ, c_void_p, c_void_p, c_i64, c_void_p,
                                           c_i64, c_i64, c_f32, c_i32, c_i32, c_void_p, c_i32, c_void_p, c_void_p,
                                           c_sz, c_void_p, ctypes.POINTER(Residual), ctypes.POINTER(Paged)]),
    "vecinfer_decode_step": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, I64x2, I64x2, I64x2,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, VQ, VQ, c_void_p,
                                     c_void_p, c_i64, c_void_p, c_void_p, c_f32, c_i32, c_i32, c_void_p, c_i32,
                                     c_void_p, c_void_p, c_void_p, c_sz, c_void_p, ctypes.POINTER(Residual)]),
    "vecinfer_decode_step_paged": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, I64x2, I64x2, I64x2,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, VQ, VQ, c_void_p,
                                           c_void_p, c_i64, c_void_p, c_void_p, c_f32, c_i32, c_i32, c_void_p,
                                           c_i32, c_void_p, c_void_p, c_void_p, c_sz, c_void_p,
                                           ctypes.POINTER(Residual), ctypes.POINTER(Paged)]),
    "vecinfer_xr_window_bytes": (c_sz, [c_i32, c_i64, c_i32]),
    "vecinfer_attn_decode_xr": (c_i32, [c_void_p, c_i32, c_i32, c_i32, c_i64, c_i64, c_void_p, c_void_p, c_void_p,
                                        c_i64, c_i64, VQ, VQ, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_i64, c_f32,
                                        c_i32, c_i32, c_void_p, c_i32, c_void_p, c_void_p, c_sz, c_void_p,
                                        ctypes.POINTER(Residual), ctypes.POINTER(XRank)]),
    "vecinfer_decode_step_xr": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, I64x2, I64x2, I64x2,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, VQ, VQ, c_void_p,
                                        c_void_p, c_i64, c_void_p, c_void_p, c_f32, c_i32, c_i32, c_void_p, c_i32,
                                        c_void_p, c_void_p, c_void_p, c_sz, c_void_p, ctypes.POINTER(Residual),
                                        ctypes.POINTER(XRank)]),
    "vecinfer_debug_attn_max_clusters": (c_i32, [c_i32]),
    "vecinfer_decode_step_workspace_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i64, VQ, VQ, c_i32]),
    "vecinfer_merge_lse": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_i32, c_i32, c_void_p, c_i32, c_void_p,
                                   c_void_p]),
}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libvecinfer.so not built at {LIB_PATH}; run `python -m paper_2510_06175_b200.build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            if os.environ.get("VECINFER_LIB") and not hasattr(lib, name):
                continue   # experiment builds (VECINFER_LIB override) may predate a symbol
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class VecInferError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = load().vecinfer_last_error().decode(errors="replace")
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


def check(fn: str, status: int) -> None:
    if status != 0:
        raise VecInferError(fn, status)
