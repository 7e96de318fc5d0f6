"""Per-config timing of libheff on one GPU: H_eff.psi matvec (single launch, and back to back
as lanczos_ground enqueues them) and Lanczos-step latency for C1..C4 (and C5 when it fits).  Writes one JSON object per config (stdout, and --out).

    python tools/sweep.py [--configs c1,c2,c3,c4] [--reps 20] [--out profiles/sweep.json]
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

from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402
from paper_2007_14822_b200.heff import OPT_PROFILE  # noqa: E402

PEAK = 148 * 128 * 1.965e9 / 1e12


def time_matvec(h, psi, out, reps):
    s = torch.cuda.current_stream()
    for _ in range(3):
        h.apply(psi, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        h.apply(psi, out)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def time_matvec_b2b(h, psi, out, n):
    """Back-to-back matvecs (the way lanczos_ground enqueues them: no host wait between
    launches): device time of n consecutive applies / n."""
    s = torch.cuda.current_stream()
    for _ in range(3):
        h.apply(psi, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        h.apply(psi, out)
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    res = []
    for spec in args.configs.split(","):
        name, _, mm = spec.partition(":")   # "c4:128" = preset c4 at bond cap m = 128
        t0 = time.perf_counter()
        x = C.make(name, device=dev, m=int(mm) if mm else None)
        gen_s = time.perf_counter() - t0
        d = x.dims
        flops = C.flops_per_matvec(d)
        big = flops > 1e12
        reps = 3 if big else args.reps
        with Heff(x.L, x.W1, x.W2, x.R) as h:
            out = torch.empty_like(x.psi)
            ms = time_matvec(h, x.psi, out, reps)
            ms_b2b = time_matvec_b2b(h, x.psi, out, 3 if big else 200)
            h_launches = h.get_option(2)
            h.set_option(OPT_PROFILE, 1)
            h.apply(x.psi, out)
            g1, mpo, g4, n = h.last_timings()
            h.set_option(OPT_PROFILE, 0)
            steps = 2 if flops > 1e14 else (3 if big else 20)
            v = x.psi.clone()
            h.lanczos_ground(v, max_iter=steps)
            torch.cuda.synchronize()
            v = x.psi.clone()
            t0 = time.perf_counter()
            r = h.lanczos_ground(v, max_iter=steps)
            lz = (time.perf_counter() - t0) / steps * 1e3
        g1f = 2.0 * d["mL"] * d["kL"] * d["mL"] * d["d1"] * d["d2"] * d["mR"]
        g4f = C.gemm_flops_per_matvec(d) - g1f
        row = {"config": spec, **d, "gen_s": round(gen_s, 2), "matvec_ms": ms, "matvec_b2b_ms": ms_b2b,
               "tflops_b2b": flops / ms_b2b / 1e9, "frac_peak_b2b": flops / ms_b2b / 1e9 / PEAK,
               "launches_per_matvec": h_launches, "matvecs_per_s": 1e3 / ms,
               "tflops": flops / ms / 1e9, "frac_peak": flops / ms / 1e9 / PEAK,
               "gemm_first_ms": g1, "mpo_ms": mpo, "gemm_last_ms": g4,
               "gemm_first_tflops": g1f / g1 / 1e9 if g1 else None, "gemm_last_tflops": g4f / g4 / 1e9 if g4 else None,
               "lanczos_step_ms": lz, "lanczos_steps": steps, "energy": r.energy}
        print(json.dumps(row), flush=True)
        res.append(row)
        del x
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
