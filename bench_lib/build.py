"""Build the benchmark-only helpers (not product code): the cuBLASLt
best-of-top-k dense GEMM baseline used by bench.py.

    python bench_lib/build.py
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libsbw_cublaslt_bench.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "cublaslt_best.cpp")
    if force or not os.path.exists(LIB) or os.path.getmtime(src) > os.path.getmtime(LIB):
        cmd = ["g++", "-O2", "-fPIC", "-shared", "-std=c++17", "-I/usr/local/cuda/include", src, "-o", LIB,
               "-L/usr/local/cuda/lib64", "-lcublasLt", "-lcudart"]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
