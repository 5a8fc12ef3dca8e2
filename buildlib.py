"""Native build for the repo: the seeded generators (synth/), the oracle (oracle/) and the
sm_100a CUDA library behind the C ABI (paper_1412_1741_b200/csrc -> libparem.so).

All artefacts are built in-tree so they travel to the GPU box with the gpurun snapshot.
`python buildlib.py` rebuilds whatever is stale; `__graft_entry__.build()` calls build_all().
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SYNTH_SO = os.path.join(ROOT, "synth", "libsynth.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
PAREM_SO = os.path.join(ROOT, "paper_1412_1741_b200", "libparem.so")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))


def build_synth(force: bool = False) -> str:
    src = os.path.join(ROOT, "synth", "synth.c")
    if force or _stale(SYNTH_SO, [src]):
        _run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", SYNTH_SO, src, "-lm"])
    return SYNTH_SO


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "oracle.c")
    # single-threaded, -O2, no vectorisation tricks: the oracle "as it stands"
    if force or _stale(ORACLE_SO, [src]):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", ORACLE_SO, src])
    return ORACLE_SO


def parem_sources() -> list[str]:
    d = os.path.join(ROOT, "paper_1412_1741_b200", "csrc")
    return sorted(glob.glob(os.path.join(d, "*.cu")) + glob.glob(os.path.join(d, "*.cpp")))


def parem_deps() -> list[str]:
    d = os.path.join(ROOT, "paper_1412_1741_b200", "csrc")
    return parem_sources() + sorted(glob.glob(os.path.join(d, "*.cuh")) + glob.glob(os.path.join(d, "*.h"))) + [
        os.path.join(ROOT, "include", "parem.h")
    ]


def build_parem(force: bool = False, verbose_ptxas: bool = False) -> str:
    if not (force or _stale(PAREM_SO, parem_deps())):
        return PAREM_SO
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    d = os.path.join(ROOT, "paper_1412_1741_b200", "csrc")
    headers = sorted(glob.glob(os.path.join(d, "*.cuh")) + glob.glob(os.path.join(d, "*.h"))) + [
        os.path.join(ROOT, "include", "parem.h")
    ]
    jobs = []
    objs = []
    for src in parem_sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not (force or _stale(obj, [src] + headers)):
            continue
        flags = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-lineinfo"]
        if src.endswith(".cu"):
            flags += ARCH + ["-Xptxas", "-v"] if verbose_ptxas else ARCH
        jobs.append([NVCC, "-c", src, "-o", obj] + flags)
    # the tiny-kernel instantiation TUs dominate: compile every object in parallel
    workers = max(1, min(len(jobs), os.cpu_count() or 1))
    if jobs:
        with concurrent.futures.ThreadPoolExecutor(workers) as ex:
            for f in [ex.submit(_run, j) for j in jobs]:
                f.result()
    _run([NVCC, "-shared", "-o", PAREM_SO] + objs + ARCH)
    return PAREM_SO


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_oracle(force)
    build_parem(force)


if __name__ == "__main__":
    force = "--force" in sys.argv
    if "--host-only" in sys.argv:
        build_synth(force)
        build_oracle(force)
    else:
        build_all(force)
    print("built:", SYNTH_SO, ORACLE_SO, PAREM_SO if os.path.exists(PAREM_SO) else "(no parem)")
