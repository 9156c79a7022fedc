"""Builds libnpcg.so (all CUDA sources, sm_100a) in-tree.

    python -m paper_2511_23227_b200.build        # incremental
    python -m paper_2511_23227_b200.build --force

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnpcg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
                "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "npcg.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, src[:-3] + ".o")
    s = os.path.join(CSRC, src)
    if (not force and os.path.exists(obj) and os.path.getmtime(obj) > os.path.getmtime(s)
            and os.path.getmtime(obj) > _headers_mtime()):
        return obj
    cmd = [NVCC] + FLAGS + ["-c", s, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if "spill" in r.stderr and "0 bytes spill" not in r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if (force or not os.path.exists(LIB)
            or max(os.path.getmtime(o) for o in objs) > os.path.getmtime(LIB)):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_cpp_tests(verbose: bool = True) -> str:
    """Builds tests/cpp/test_dropin (the C++ drop-in header against libnpcg.so
    and the C oracle).  Requires oracle/liboracle.so."""
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    deps = [src, LIB, os.path.join(ROOT, "include", "npcg", "npconv.hpp"),
            os.path.join(ROOT, "oracle", "liboracle.so")]
    if os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(d) for d in deps):
        return out
    cmd = [NVCC, "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", out,
           "-L" + HERE, "-lnpcg", "-L" + os.path.join(ROOT, "oracle"), "-loracle",
           "-Xlinker", "-rpath", "-Xlinker", "$ORIGIN/../../paper_2511_23227_b200",
           "-Xlinker", "-rpath", "-Xlinker", "$ORIGIN/../../oracle"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ drop-in test build failed:\n{r.stderr}")
    if verbose:
        print(f"built {out}")
    return out


def build_cpp_bench(verbose: bool = True) -> str:
    """Builds tools/cpp/bench_dropin (end-to-end timing through the C++ drop-in
    header, linked against libnpcg.so only: no torch, no oracle)."""
    src = os.path.join(ROOT, "tools", "cpp", "bench_dropin.cpp")
    out = os.path.join(ROOT, "tools", "cpp", "bench_dropin")
    deps = [src, LIB, os.path.join(ROOT, "include", "npcg", "npconv.hpp")]
    if os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(d) for d in deps):
        return out
    cmd = [NVCC, "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", out,
           "-L" + HERE, "-lnpcg", "-Xlinker", "-rpath", "-Xlinker", "$ORIGIN/../../paper_2511_23227_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ drop-in bench build failed:\n{r.stderr}")
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv)
