"""Builds ``libsp.so`` in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_1608_01966_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(HERE, "..", "include", "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles every csrc/*.cu to an object in parallel, then links libsp.so."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        jobs.append((src, [NVCC, *compile_flags, "-c", "-o", obj, src], obj))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[1], capture_output=True, text=True), jobs))
    log_lines = []
    failed = False
    for (src, cmd, _), res in zip(jobs, results):
        log_lines.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        failed |= res.returncode != 0
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *[j[2] for j in jobs]]
    if not failed:
        res = subprocess.run(link, capture_output=True, text=True)
        log_lines.append(" ".join(link) + "\n" + res.stdout + res.stderr)
        failed = res.returncode != 0
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write("\n".join(log_lines))
    if failed:
        sys.stderr.write("\n".join(log_lines)[-20000:])
        raise RuntimeError(f"nvcc failed; see {log}")
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("\n".join(log_lines))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
