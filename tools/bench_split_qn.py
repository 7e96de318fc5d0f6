"""U(1) two-site split (heff_svd_split_qn) vs the dense split of the same sector-structured
Psi on one GPU: chain C3-QN (m = 1024) and the C4-QN cylinder (6x6, m = 4096, Sz = 0).

    python tools/bench_split_qn.py [--out profiles/r01_split_qn.json]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from heffgen import qn  # noqa: E402
from paper_2007_14822_b200 import heff  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        r = fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c3qn,c4qn")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for case in a.cases.split(","):
        t0 = time.perf_counter()
        if case == "c3qn":
            z = qn.heisenberg_chain_qn(24, 11, 1024, 1104, device=dev)
        else:
            z = qn.cylinder_qn(6, 17, 4096, 1105, device=dev)
        gen = time.perf_counter() - t0
        psi = z.x.psi
        m = psi.shape[0]
        qr, qc = heff.psi_row_col_charges(z.qa, z.qs1, z.qs2, z.qb)
        tq, rq = timed(lambda: heff.svd_split_qn(psi, qr, qc, maxdim=m))
        td, rd = timed(lambda: heff.svd_split(psi, maxdim=m), reps=1)
        sectors = sorted(set(qr) & set(qc))
        blocks = [(sum(1 for v in qr if v == c), sum(1 for v in qc if v == c)) for c in sectors]
        row = dict(case=case, shape=list(psi.shape), gen_s=gen, qn_ms=tq, dense_ms=td, speedup=td / tq,
                   n_qn=rq.n, n_dense=rd.n, err_qn=rq.trunc_err, err_dense=rd.trunc_err,
                   max_abs_dS=float((rq.S - rd.S).abs().max()), qn_sweeps_max=rq.sweeps, dense_sweeps=rd.sweeps,
                   nblocks=len(blocks), largest_block=max(blocks, key=lambda x: x[0] * x[1]))
        print(json.dumps(row), flush=True)
        rows.append(row)
        del z, psi
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
