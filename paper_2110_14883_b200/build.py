"""Build the C-ABI library libtp_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2110_14883_b200.build [--force] [-j N]

Every .cu / .cpp under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked against the NCCL shipped with the image (nvidia-nccl wheel, rpath'd).
Objects go to build/ (git-ignored); the .so lands next to this file so gpurun
snapshots carry it to the GPU box.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libtp_b200.so")
BUILD = os.path.join(ROOT, "build", "tp_b200")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel missing)")


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def common_flags():
    inc, _ = nccl_paths()
    extra = os.environ.get("TP_NVCC_FLAGS", "").split()  # diagnostics builds, e.g. -DTP_LOOP_CLOCKS=1
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                   "-I", os.path.join(ROOT, "include"), "-I", inc,
                   "--expt-relaxed-constexpr", "-Xptxas", "-v" if os.environ.get("TP_PTXAS_V") else "-O3"] + extra


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0)


def compile_one(src, force, hm):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hm):
        return obj, None
    cmd = [nvcc()] + common_flags() + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [nvcc(), "-x", "cu"] + common_flags() + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"FAILED: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    return obj, (r.stderr if os.environ.get("TP_PTXAS_V") else None)


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hm = headers_mtime()
    srcs = sources()
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(lambda s: compile_one(s, force, hm), srcs))
    errors = [m for _, m in results if m and m.startswith("FAILED")]
    if errors:
        raise RuntimeError("\n".join(errors))
    if verbose:
        for _, m in results:
            if m:
                print(m)
    objs = [o for o, _ in results]
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < newest:
        _, lib = nccl_paths()
        cmd = [nvcc()] + ARCH + ["-shared", "-o", OUT] + objs + [
            "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-lcudart_static",
            "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return OUT


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v))


if __name__ == "__main__":
    sys.exit(main())
