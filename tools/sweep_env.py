"""Timing of the environment update (NEXT-1) at the C2..C4 sizes on one GPU.

    python tools/sweep_env.py [--out profiles/env.json]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from heffgen import mpo  # noqa: E402
from paper_2007_14822_b200 import env_update_left, env_update_right  # noqa: E402

PEAK = 148 * 128 * 1.965e9 / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for name, m, d, W in (("c2", 256, 2, mpo.heisenberg_chain_W()), ("c3", 1024, 2, mpo.heisenberg_chain_W()),
                          ("c4", 4096, 2, mpo.cylinder_W(17)), ("c5", 8192, 4, mpo.hubbard_W())):
        k = W.shape[0]
        g = torch.Generator(device=dev).manual_seed(0)
        L = torch.randn((m, k, m), dtype=torch.float64, device=dev, generator=g)
        A = torch.randn((m, d, m), dtype=torch.float64, device=dev, generator=g)
        Wt = torch.from_numpy(W).to(dev)
        res = {"config": name, "m": m, "d": d, "k": k}
        for side, fn in (("left", env_update_left), ("right", env_update_right)):
            fn(L, A, Wt)
            torch.cuda.synchronize()
            reps = 2 if m >= 4096 else 10
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn(L, A, Wt)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            flop = 2.0 * (m * k * m * d * m) * 2 + 2.0 * m * k * d * d * k * m  # two GEMMs + dense MPO step
            res[f"{side}_ms"] = ms
            res[f"{side}_tflops"] = flop / ms / 1e9
            res[f"{side}_frac_peak"] = flop / ms / 1e9 / PEAK
        print(json.dumps(res), flush=True)
        rows.append(res)
        del L, A
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
