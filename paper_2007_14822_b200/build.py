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


STAMP = PKG / "libheff.so.srchash"


def source_hash(cmd: list[str]) -> str:
    """sha256 over every source/header the library is built from and the nvcc command."""
    import hashlib
    h = hashlib.sha256()
    for d in deps():
        h.update(d.name.encode())
        h.update(d.read_bytes())
    h.update(" ".join(c for c in cmd if not c.startswith("/")).encode())
    return h.hexdigest()[:16]


def build_hash() -> str | None:
    """The source hash libheff.so was built from (None if unknown)."""
    return STAMP.read_text().strip() if STAMP.exists() else None


def build(force: bool = False, verbose: bool = False) -> Path:
    cmd = _cmd(verbose)
    want = source_hash(cmd)
    # rebuild whenever the sources differ from the ones the shipped .so was built from
    # (content hash, not mtimes: a stale .so pushed with newer sources is never reused)
    if not force and LIB.exists() and build_hash() == want:
        return LIB
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stdout + r.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    STAMP.write_text(want + "\n")
    return LIB


def _cmd(verbose: bool = False) -> list[str]:
    return [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
           "-I", str(ROOT / "include"), "-I", nccl_include(),
           *map(str, sources()), "-o", str(LIB) + ".tmp", "-ldl"]


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
