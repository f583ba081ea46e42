"""Build tests/ncclshim/libncclshim.so (test infrastructure: the one-GPU multi-process NCCL
stand-in, see ncclshim.cpp). Returns the library path; rebuilds when the source is newer."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ncclshim.cpp")
LIB = os.path.join(HERE, "libncclshim.so")


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    from paper_2110_14883_b200.build import nccl_paths
    inc, _ = nccl_paths()
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    tmp = LIB + f".{os.getpid()}.tmp"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall", f"-I{inc}",
                    f"-I{cuda}/include", SRC, "-o", tmp, f"-L{cuda}/lib64", "-lcudart_static",
                    "-ldl", "-lpthread", "-lrt"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
