"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/vecinfer.h declares,
contains sm_100a code, and validates arguments before touching CUDA.  No compute calls."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vecinfer.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2510_06175_b200 import build
    if not os.path.exists(build.LIB):
        build.build()
    from paper_2510_06175_b200 import _lib
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vecinfer_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_four_entry_points():
    names = declared_functions()
    for n in ("vecinfer_calibrate_smooth", "vecinfer_encode_kv", "vecinfer_attn_decode", "vecinfer_merge_lse"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2510_06175_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), f"{name} not exported"
        assert name in _lib.PROTOTYPES, f"{name} missing from the Python prototypes"
    assert lib.vecinfer_abi_version() == 7


def test_library_contains_sm100a_code(lib):
    from paper_2510_06175_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation_without_cuda(lib):
    """NULL pointers / bad shapes return a status synchronously (no launch, no CUDA call)."""
    from paper_2510_06175_b200._lib import VQ, I64x3
    cfg = VQ(128, 4, 8)
    st = lib.vecinfer_attn_decode(None, 1, 32, 8, 0, 0, None, None, None, 0, 0, cfg, cfg, None, None, 16, None, 0, -1,
                                  0.088, 0, 0, None, 1, None, None, 0, None, None)
    assert st == 1 and b"NULL" in lib.vecinfer_last_error()
    st = lib.vecinfer_merge_lse(None, None, 1, 1, 1, 128, None, 1, None, None)
    assert st == 1
    st = lib.vecinfer_calibrate_smooth(ctypes.c_void_p(16), 0, 8, 128, 1024, 128, 1e-6, ctypes.c_void_p(16),
                                       ctypes.c_void_p(16), ctypes.c_void_p(256), 1 << 20, None)
    assert st == 4     # EMPTY: Eq. 4 undefined on an empty calibration set
    st = lib.vecinfer_calibrate_smooth(ctypes.c_void_p(16), 5, 8, 128, 1024, 128, 0.0, ctypes.c_void_p(16),
                                       ctypes.c_void_p(16), ctypes.c_void_p(256), 1 << 20, None)
    assert st == 1     # eps <= 0
    bad = VQ(128, 16, 8)   # d = 16: no kernel (d8b8 / d8b12 / d4b10 / d2b8 are NEXT-2 formats)
    st = lib.vecinfer_encode_kv(ctypes.c_void_p(256), ctypes.c_void_p(256), 1, 1, 8, I64x3(0, 1024, 128),
                                I64x3(0, 1024, 128), ctypes.c_void_p(256), ctypes.c_void_p(256), ctypes.c_void_p(256),
                                0, 0, bad, cfg, ctypes.c_void_p(256), ctypes.c_void_p(256), 16, ctypes.c_void_p(256),
                                None, None, 0, None)
    assert st == 3     # UNSUPPORTED (d = 16)
    assert lib.vecinfer_status_string(3) == b"VECINFER_ERR_UNSUPPORTED"
    # k-means step (NEXT-3): d outside {2, 4, 8}, n < k, n == 0, short workspace
    p = ctypes.c_void_p(256)
    assert lib.vecinfer_kmeans_step(p, 100, 3, p, 16, p, p, p, p, p, 1 << 20, None) == 3
    assert lib.vecinfer_kmeans_step(p, 8, 4, p, 16, p, p, p, p, p, 1 << 20, None) == 2
    assert lib.vecinfer_kmeans_step(p, 0, 4, p, 16, p, p, p, p, p, 1 << 20, None) == 4
    assert lib.vecinfer_kmeans_step(p, 100, 4, p, 16, p, p, p, p, p, 16, None) == 6
    assert lib.vecinfer_kmeans_step(None, 100, 4, p, 16, p, p, p, p, p, 1 << 20, None) == 1
    assert lib.vecinfer_kmeans_workspace_bytes(256, 4) >= 256 * 4 * 8 + 256 * 4
    # fused P2P exchange (§8(e)): window size = header + 2 parities x P x rows x ((D + 1) fp32 + flag)
    assert lib.vecinfer_p2p_window_bytes(8, 1024, 128) == 256 + 2 * 8 * 1024 * (129 * 4 + 4)
    assert lib.vecinfer_p2p_window_bytes(0, 1024, 128) == 0
    assert lib.vecinfer_merge_lse_p2p(p, p, p, 2, 2, 1, 32, 128, 0, p, 1, p, None, None) == 2   # rank >= P
    assert lib.vecinfer_merge_lse_p2p(p, p, p, 2, 0, 1, 32, 2048, 0, p, 1, p, None, None) == 2  # D > 1024
    assert lib.vecinfer_merge_lse_p2p(None, p, p, 2, 0, 1, 32, 128, 0, p, 1, p, None, None) == 1
    assert lib.vecinfer_p2p_window_create(0, p, p) == 1


def test_workspace_and_split_queries(lib):
    assert lib.vecinfer_attn_num_splits(1, 8, 32768, 0) >= 1
    assert lib.vecinfer_attn_num_splits(1, 8, 32768, 5) == 5
    assert lib.vecinfer_attn_workspace_bytes(1, 32, 8, 128, 32768, 4) >= 8 * 4 * 4 * 129 * 4
    assert lib.vecinfer_calibrate_workspace_bytes(8, 128) >= 8 * 128 * 4
    from paper_2510_06175_b200._lib import VQ
    assert lib.vecinfer_encode_workspace_bytes(1, 1, 8, VQ(128, 4, 8), VQ(128, 4, 8)) == 0
    # 16-bit books: (lo, hi) fp32 pairs per (token-head, stream, sub-vector, 512-centroid chunk) of one
    # pass of <= 512 token-heads
    assert lib.vecinfer_encode_workspace_bytes(1, 1, 8, VQ(128, 4, 16), VQ(128, 4, 8)) == 8 * 2 * 32 * 128 * 8
    assert lib.vecinfer_encode_workspace_bytes(4, 4096, 8, VQ(128, 4, 16), VQ(128, 4, 16)) == 512 * 2 * 32 * 128 * 8


def test_product_path_never_imports_the_oracle():
    """The CUDA product path shares no code with oracle/ and never routes through it."""
    pkg = os.path.join(ROOT, "paper_2510_06175_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, flags=re.M), f
                assert "import_module(\"oracle" not in txt and "__import__(\"oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(from|import)\s+paper_2510_06175_b200", txt, flags=re.M), f


def test_binding_rejects_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2510_06175_b200 import vecinfer as vi
    with pytest.raises(ValueError, match="CUDA"):
        vi.calibrate_smooth(torch.zeros(4, 1, 128, dtype=torch.bfloat16))
