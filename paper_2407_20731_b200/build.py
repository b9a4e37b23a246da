"""Build recipe of the in-tree CUDA library (sm_100a only)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "isf_lossy.cu"), os.path.join(HERE, "csrc", "gll_host.cpp")]
OUT = os.path.join(HERE, "libisf_lossy.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++20",
    "-ccbin", "/usr/bin/g++", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d))] + [os.path.join(REPO, "include", "isf_lossy.h")]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, log: str | None = None, out: str = OUT, defines=()) -> str:
    if not force and out == OUT and not needs_build():
        return OUT
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SRC, "-ldl", "-lquadmath"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stderr[-4000:]}")
    return OUT


if __name__ == "__main__":
    print(build(force=True, log=os.path.join(REPO, "build", "nvcc.log")))
