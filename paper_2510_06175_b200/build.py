"""Build libvecinfer.so in-tree for sm_100a (nvcc, no torch involvement).

    python -m paper_2510_06175_b200.build [--force] [-v]

Compiles every csrc/*.cu with -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 into
objects (in parallel) and links paper_2510_06175_b200/libvecinfer.so (static cudart), so the
library loads on a GPU-less host for the symbol checks and the same file ships to the B200 box.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "vecinfer")
LIB = os.path.join(PKG, "libvecinfer.so")
# profiling variant (phase timestamps), built only on request: python -m paper_2510_06175_b200.build --phase-timing
LIB_PHASE = os.path.join(PKG, "libvecinfer_phase.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "vecinfer.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, phase_timing: bool = False, defines=(), out=None) -> str:
    global BUILD, LIB
    if phase_timing:
        BUILD, LIB = BUILD + "_phase", LIB_PHASE
        FLAGS.append("-DVECINFER_PHASE_TIMING")
    if out:   # experiment variant (-D macros) into its own object dir and library; VECINFER_LIB loads it
        LIB = os.path.abspath(out)
        BUILD = os.path.join(ROOT, "build", os.path.splitext(os.path.basename(out))[0])
    FLAGS.extend("-D" + d for d in defines)
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    headers = [d for d in _deps() if not d.endswith(".cu")]
    objs = []
    jobs = []
    for src in srcs:
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, p

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for cmd, p in ex.map(run, jobs):
            if verbose or p.returncode:
                sys.stderr.write(p.stdout + p.stderr)
            if p.returncode:
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode:
            sys.stderr.write(p.stdout + p.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--phase-timing", action="store_true")
    ap.add_argument("-D", "--define", action="append", default=[], help="experiment macro NAME=VALUE")
    ap.add_argument("--out", help="experiment library path (with --define)")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose, phase_timing=args.phase_timing, defines=args.define,
                out=args.out))
