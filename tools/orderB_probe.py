"""One order-B shard matvec at the P-way shard shape of a config, plus the all-gather
re-layout kernel: the launch list an ncu capture of the order-B kernels profiles.

    python tools/orderB_probe.py [--config c4] [--P 8] [--reps 3]
Prints per-kernel CUDA-event times of the shard matvec's steps (HEFF_OPT_PROFILE) and of
heff_relayout_blocked, with the order-B MPO kernel's algorithmic bytes per launch.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402
from paper_2007_14822_b200.heff import OPT_PROFILE, relayout_blocked  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--full", action="store_true",
                    help="GEMM_A from the full psi (heff_apply: the NCCL all-gather path's kernels) instead of "
                         "the blocked shards (heff_apply_blocked: the gather-fused path's)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    x = C.make(a.config, device=dev)
    d = x.dims
    P, mR = a.P, d["mR"]
    nb = mR // P
    rows = d["mL"] * d["d1"] * d["d2"]
    blocked = x.psi.reshape(rows, P, nb).permute(1, 0, 2).contiguous()
    Rg = x.R[:nb].contiguous()
    res = dict(config=a.config, P=P, nb=nb)
    with Heff(x.L, x.W1, x.W2, Rg, dist=dict(nranks=P, rank=0, b_lo=0, b_hi=nb)) as h:
        out = torch.empty(h.out_shape, dtype=torch.float64, device=dev)
        run = (lambda: h.apply(x.psi, out)) if a.full else (lambda: h.apply_blocked(blocked, out))
        run()
        torch.cuda.synchronize()
        h.set_option(OPT_PROFILE, 1)
        for _ in range(a.reps):
            run()
        g1, mpo, g4, n = h.last_timings()
        h.set_option(OPT_PROFILE, 0)
    # the order-B MPO kernel reads V1 and writes V3: (kR + kL) d1 d2 doubles per (a, b')
    mpo_bytes = 8.0 * d["mL"] * nb * d["d1"] * d["d2"] * (d["kR"] + d["kL"])
    res.update(gemmA_ms=g1 / n, mpo_ms=mpo / n, gemmD_ms=g4 / n, mpo_bytes=mpo_bytes,
               mpo_gbs=mpo_bytes / (mpo / n * 1e-3) / 1e9)
    s = torch.cuda.current_stream()
    relayout_blocked(blocked, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        relayout_blocked(blocked, P)
    e1.record(s)
    e1.synchronize()
    t = e0.elapsed_time(e1) / a.reps
    res.update(relayout_ms=t, relayout_bytes=16.0 * rows * mR, relayout_gbs=16.0 * rows * mR / (t * 1e-3) / 1e9)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
