"""Build libheff.so (sm_100a) in-tree with nvcc.  Called by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc"
LIB = PKG / "libheff.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_include() -> str:
    for cand in [Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / "site-packages"
                 / "nvidia" / "nccl" / "include", Path("/usr/include")]:
        if (cand / "nccl.h").exists():
            return str(cand)
    raise FileNotFoundError("nccl.h not found")


def sources():
    return sorted(SRC.glob("*.cu"))


def deps():
    return sorted(list(SRC.glob("*.cu")) + list(SRC.glob("*.cuh")) + list(SRC.glob("*.h")) + [ROOT / "include" / "heff.h"])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and LIB.exists() and all(LIB.stat().st_mtime >= d.stat().st_mtime for d in deps()):
        return LIB
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
           "-I", str(ROOT / "include"), "-I", nccl_include(),
           *map(str, sources()), "-o", str(LIB) + ".tmp", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stdout + r.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
