"""In-tree build of libtnb200.so for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2012_02430_b200.build        # or __graft_entry__.build()

The translation units (runtime, planner and one per kernel family) compile in parallel, then
link into one shared library next to this file.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtnb200.so")
OBJ = os.path.join(CSRC, "build")
SOURCES = ["runtime.cu", "planner.cpp", "launch_gemm.cu", "launch_gemm_hm.cu", "launch_gemm_hm64.cu", "launch_gemm_tc.cu", "launch_gemm_fc.cu", "launch_fc_tc.cu", "launch_pair.cu", "launch_bucket.cu",
           "launch_group_c64.cu", "launch_group_c128.cu"]
HEADERS = ["kernels.cuh", "kernels_tc.cuh", "kernels_hm.cuh", "kernels_fc.cuh", "kernels_fctc.cuh", "launch.cuh", "launch_group.inl", "plan_format.h", "planner.h",
           os.path.join("..", "..", "include", "tn_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def _compile(nvcc: str, src: str, verbose: bool):
    obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, r


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(nvcc, s, verbose), SOURCES))
    for src, _, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    link = [nvcc, *ARCH, "-shared", "-o", LIB + ".tmp"] + [o for _, o, _ in results]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libtnb200.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
