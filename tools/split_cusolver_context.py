"""Context only (not a product path): time the vendor dense eigen/SVD solvers torch exposes
(cuSOLVER via torch.linalg) on the same Psi matrices as tools/bench_split.py, next to
heff_svd_split.  Prints one JSON object per (size, solver).  Nothing here is called by the
library; it answers "is the hand-written Jacobi split competitive with the library route"."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import heff  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best


def main():
    dev = torch.device("cuda:0")
    for m in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024,4096").split(",")]:
        psi = C.random_psi(1000 + m, (m, 2, 2, m), dev)
        P = psi.reshape(2 * m, 2 * m)
        ref = torch.linalg.svdvals(P)
        rows = {"heff_svd_split": lambda: heff.svd_split(psi, direction=0),
                "torch.linalg.svd gesvd": lambda: torch.linalg.svd(P, full_matrices=False, driver="gesvd"),
                "torch.linalg.svd gesvdj": lambda: torch.linalg.svd(P, full_matrices=False, driver="gesvdj"),
                "torch.linalg.eigh(Psi Psi^T) syevd": lambda: torch.linalg.eigh(P @ P.T)}
        for name, fn in rows.items():
            try:
                t = timed(fn)
                out = fn()
                if name == "heff_svd_split":
                    s = out.S
                elif "eigh" in name:
                    s = out[0].clamp_min(0).sqrt().flip(0)
                else:
                    s = out[1]
                err = float((s[: ref.numel()] - ref).abs().max() / ref[0])
                print(json.dumps(dict(m=m, rows=2 * m, solver=name, ms=t, max_rel_sv_diff_vs_svdvals=err)), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps(dict(m=m, solver=name, error=str(e)[:200])), flush=True)


if __name__ == "__main__":
    main()
