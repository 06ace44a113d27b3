"""Build libpbng.so (sm_100a) in-tree with nvcc.  No JIT cache, no torch extension:
the shared library sits next to this file so it travels with the repository."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libpbng.so")
SOURCES = [os.path.join(HERE, "csrc", "pbng.cu")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def _deps():
    return SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "pbng.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [NVCC] + FLAGS + ["-o", LIB] + SOURCES
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return LIB


def build_variant(name: str, defines: dict) -> str:
    """Tuning experiments: build lib<name>.so with -D overrides (not used by the product path)."""
    out = os.path.join(HERE, f"libpbng_{name}.so")
    cmd = [NVCC] + FLAGS + [f"-D{k}={v}" for k, v in defines.items()] + ["-o", out] + SOURCES
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
