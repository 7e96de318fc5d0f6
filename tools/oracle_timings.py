"""CPU-oracle timings on the GPU box's host (BASELINE.md section 4 / SURVEY.md 8(d) timing
protocol): the oracle is the reported CPU baseline, never the target.

  * host: `lscpu` model name, nproc, the OpenMP threads used;
  * C1-C3: one order-A matvec, median of 3 (C3 at 1 thread: one run), at 1 thread and at
    all cores;
  * C4: ONE WHOLE matvec at all cores (~10 min), next to the row-sample extrapolation that
    bench.py's cpu_baseline and --impl reference use (96 rows), to validate it.

    python tools/oracle_timings.py [--skip-c4] [--out profiles/r02_oracle_timings.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from heffgen import configs as C  # noqa: E402
from oracle import oracle  # noqa: E402


def lscpu_model() -> str | None:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def time_apply(args, reps, rows=None):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.heff_apply(*args, rows=rows)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), ts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    oracle.build()
    cores = os.cpu_count() or 1
    res = {"host": {"lscpu_model": lscpu_model(), "nproc": cores}, "configs": {}}
    for cfg in ("c1", "c2", "c3"):
        x = C.make(cfg)
        args = x.numpy()[:5]
        flops = C.flops_per_matvec(x.dims)
        row = {"dims": x.dims, "flops": flops}
        for th in (1, cores):
            oracle.set_threads(th)
            reps = 1 if (cfg == "c3" and th == 1) else 3
            med, ts = time_apply(args, reps)
            row[f"threads_{th}"] = {"median_s": med, "runs_s": ts, "gflops": flops / med / 1e9,
                                    "matvec_per_s": 1.0 / med}
        res["configs"][cfg] = row
        print(json.dumps({cfg: row}), flush=True)
    if not a.skip_c4:
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        x = C.make("c4", device=dev).to("cpu")
        args = x.numpy()[:5]
        flops = C.flops_per_matvec(x.dims)
        oracle.set_threads(cores)
        mL = x.dims["mL"]
        t0 = time.perf_counter()
        oracle.heff_apply(*args, rows=(0, 96))
        t_rows = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.heff_apply(*args)
        t_full = time.perf_counter() - t0
        row = {"dims": x.dims, "flops": flops, "threads": cores, "whole_matvec_s": t_full,
               "whole_matvec_per_s": 1.0 / t_full, "gflops": flops / t_full / 1e9,
               "rows96_s": t_rows, "rows96_extrapolated_matvec_s": t_rows * mL / 96,
               "extrapolation_ratio": (t_rows * mL / 96) / t_full}
        res["configs"]["c4"] = row
        print(json.dumps({"c4": row}), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
