"""Build libidm.so (the C-ABI CUDA library) in-tree for sm_100a with nvcc.

    python -m paper_2412_16750_b200.build          # incremental
    python -m paper_2412_16750_b200.build --force
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libidm.so")
HEADER = os.path.join(ROOT, "include", "idm.h")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(CSRC, "*.h")) + [HEADER, __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build libidm.so (or a variant at `out` with extra -D defines, for tuning sweeps): each
    .cu compiled to an object in parallel, then one link."""
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    objdir = tempfile.mkdtemp(prefix="idm_build_")
    inc = ["-I", os.path.join(ROOT, "include")]
    dflags = [f"-D{d}" for d in defines]
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *NVCC_FLAGS, *dflags, *inc, "-c", src, "-o", obj]
        jobs.append((cmd, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.PIPE, text=True)))
    logtxt, failed = [], False
    for cmd, _, proc in jobs:
        so, se = proc.communicate()
        logtxt.append(" ".join(cmd) + "\n" + so + se)
        failed |= proc.returncode != 0
    if not failed:
        link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker",
                "--exclude-libs,ALL", *[o for _, o, _ in jobs], "-o", tmp, "-lcudart_static"]
        res = subprocess.run(link, capture_output=True, text=True)
        logtxt.append(" ".join(link) + "\n" + res.stdout + res.stderr)
        failed = res.returncode != 0
    shutil.rmtree(objdir, ignore_errors=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write("\n".join(logtxt))
    if failed:
        sys.stderr.write("\n".join(logtxt)[-20000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write("\n".join(logtxt))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
