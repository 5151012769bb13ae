"""Build the in-tree native libraries for sm_100a.

    libneo.so      paper_2411_01142_b200/csrc/*.cu  (the product: C ABI of include/neo.h)
    libneo_gen.so  neo_inputs/csrc/neo_gen.cu       (seeded input generator, test/bench infra)

Run ``python -m paper_2411_01142_b200.build`` (``__graft_entry__.build()`` calls it).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]

LIBNEO = os.path.join(PKG, "libneo.so")
LIBGEN = os.path.join(ROOT, "neo_inputs", "libneo_gen.so")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _nvcc(out: str, srcs: list[str], extra: list[str], verbose: bool) -> None:
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-o", tmp, *srcs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed for {out}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> list[str]:
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cpp")))
    deps = srcs + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "neo.h")]
    built = []
    if force or _stale(LIBNEO, deps):
        _nvcc(LIBNEO, srcs, ["-I", os.path.join(ROOT, "include")], verbose)
        built.append(LIBNEO)
    gsrc = [os.path.join(ROOT, "neo_inputs", "csrc", "neo_gen.cu")]
    if force or _stale(LIBGEN, gsrc):
        _nvcc(LIBGEN, gsrc, [], verbose)
        built.append(LIBGEN)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
