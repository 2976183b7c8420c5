"""Build tests/sim/libedit_sim.so (test infrastructure): the simulated single-GPU mesh shim,
linked against the product library libedit_sync.so (same code, driven per member)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SRC = os.path.join(HERE, "edit_sim.cpp")
LIB = os.path.join(HERE, "libedit_sim.so")


def build(force: bool = False) -> str:
    sys.path.insert(0, ROOT)
    from paper_2412_07210_b200 import build as pkg_build
    prod = pkg_build.build()
    deps = [SRC, prod, os.path.join(pkg_build.CSRC, "handle.h"), os.path.join(pkg_build.CSRC, "internal.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(d) <= os.path.getmtime(LIB) for d in deps):
        return LIB
    inc, _ = pkg_build.nccl_paths()
    tmp = f"{LIB}.tmp{os.getpid()}"
    cmd = [pkg_build.NVCC, "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", pkg_build.INCLUDE,
           "-I", pkg_build.CSRC, "-I", inc, SRC, "-L", pkg_build.PKG, "-l:libedit_sync.so",
           "-Xlinker", f"-rpath,{pkg_build.PKG}", "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build of tests/sim/libedit_sim.so failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
