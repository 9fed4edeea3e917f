"""Build the CUDA extension in-tree: _lib/libtrihalo_b200.so (sm_100a).

    python -m paper_2504_15814_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libtrihalo_b200.so")
SOURCES = ["builder.cpp", "trihalo.cu"]
HEADERS = ["builder.hpp", os.path.join("..", "..", "include", "trihalo_b200.h")]
NVCC_FLAGS = [
    "-shared", "-Xcompiler", "-fPIC", "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h", ".cu", ".cpp"))]
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    out = out or OUT
    if out == OUT and not force and not _stale():
        return OUT
    os.makedirs(os.path.dirname(out), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("TH_EXTRA_NVCC_FLAGS", "").split()  # A/B builds only (e.g. -DTH_AB_DMMA)
    cmd = [nvcc, *NVCC_FLAGS, *extra, *[os.path.join(CSRC, f) for f in SOURCES], "-o", out + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    with open(os.path.join(os.path.dirname(out), "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python -m paper_2504_15814_b200.build [--force] [--out PATH]   (TH_EXTRA_NVCC_FLAGS for A/B builds)
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose=True, out=o))
