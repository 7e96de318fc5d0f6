"""Time the two-site split (heff_svd_split) at the config sizes on one GPU.

Psi is the two-site matrix (mL d) x (d mR) of configs C1..C4: the seeded N(0,1) psi of the
config (reading R8) and a graded stand-in with a DMRG-like decaying spectrum
(heffgen.configs.graded_matrix).  Reports ms per split (CUDA events on the launching
stream, after one warm-up), Jacobi sweeps, and the per-sweep streaming figures.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import heff  # noqa: E402

SIZES = {"c1": 16, "c2": 256, "c3": 1024, "c4": 4096}


_DMRG_CACHE = {}


def dmrg_psi(m: int, dev):
    """Centre two-site wavefunction of a DMRG run (Heisenberg chain, maxdim m, cutoff 0) whose
    bond reaches m: the realistic input of the split (tools/dmrg_gpu.py)."""
    if m not in _DMRG_CACHE:
        from heffgen import mpo
        from tools.dmrg_gpu import dmrg
        N = 2 * (max(1, (m - 1).bit_length()) + 2)
        cap = {}
        sched = [min(m, 16 * 2 ** s) for s in range(max(2, (m // 16).bit_length() + 1))] + [m]
        dmrg([mpo.heisenberg_chain_W()] * N, sched, cutoff=0.0, lanczos_iter=8, log=lambda *_: None, capture=cap)
        _DMRG_CACHE[m] = cap["psi"]
    return _DMRG_CACHE[m]


def run(m: int, kind: str, reps: int, maxdim: int, direction: int):
    dev = torch.device("cuda:0")
    if kind == "random":
        psi = C.random_psi(1000 + m, (m, 2, 2, m), dev)
    elif kind == "dmrg":
        psi = dmrg_psi(m, dev)
    else:
        psi = torch.from_numpy(C.graded_matrix(2 * m, 2 * m, 7, 12.0)).to(dev).view(m, 2, 2, m)
    heff.svd_split(psi, maxdim=maxdim, direction=direction)      # warm-up (arena, module load)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ts, sweeps = [], []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        r = heff.svd_split(psi, maxdim=maxdim, direction=direction)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        sweeps.append(r.sweeps)
    ts.sort()
    M = psi.shape[0] * psi.shape[1]
    nblk = ((M + 15) // 16 + 1) // 2 * 2
    # per sweep: every round streams X once for the Gram (read) and once for the rotation
    # (read + write): 24 B per element, (nblk - 1) rounds
    bytes_per_sweep = 24.0 * M * (nblk * 16) * (nblk - 1)
    return dict(m=m, M=M, shape=list(psi.shape), kind=kind, dir=direction, maxdim=maxdim, ms=ts[len(ts) // 2], ms_min=ts[0],
                sweeps=sweeps[-1], n=r.n, trunc_err=r.trunc_err,
                ms_per_sweep=ts[len(ts) // 2] / sweeps[-1],
                stream_GBps=bytes_per_sweep * sweeps[-1] / (ts[len(ts) // 2] * 1e-3) / 1e9)


def oracle_time(m: int, kind: str, maxdim: int, direction: int):
    """The CPU oracle (oracle/split.py: LAPACK SVD + the truncation rule) on the same Psi,
    all host cores -- the reported baseline beside the GPU number."""
    import os
    from oracle import split as osplit
    dev = torch.device("cuda:0")
    if kind == "random":
        Psi = C.random_psi(1000 + m, (m, 2, 2, m)).numpy().reshape(2 * m, 2 * m)
    elif kind == "dmrg":
        Psi = dmrg_psi(m, dev).cpu().numpy()
        Psi = Psi.reshape(Psi.shape[0] * Psi.shape[1], -1)
    else:
        Psi = C.graded_matrix(2 * m, 2 * m, 7, 12.0)
    t0 = time.perf_counter()
    osplit.svd_split(Psi, maxdim=maxdim, direction=direction)
    return time.perf_counter() - t0, os.cpu_count()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", action="store_true", help="also time the CPU oracle (C4 takes minutes)")
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--kinds", default="random,graded")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for c in a.configs.split(","):
        m = SIZES[c]
        for kind in a.kinds.split(","):
            for d in (0, 1):
                row = dict(config=c, **run(m, kind, a.reps if m < 4096 else max(1, a.reps - 1), m, d))
                if a.oracle and d == 0:
                    t, cores = oracle_time(m, kind, m, d)
                    row.update(oracle_s=t, oracle_cores=cores, gpu_speedup=t / (row["ms"] * 1e-3))
                print(json.dumps(row), flush=True)
                rows.append(row)
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
