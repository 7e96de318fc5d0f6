"""Complex H_eff (NEXT-4) timing on one GPU: DM chain at m = 1024 and a complex C4-size
cylinder-shaped problem (random complex environments of the C4 dims).

    python tools/sweep_complex.py [--out profiles/complex.json]
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
from heffgen import mpo  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402
from paper_2007_14822_b200.heff import OPT_PROFILE  # noqa: E402

PEAK = 148 * 128 * 1.965e9 / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    cyl = [mpo.cylinder_W(j).astype(complex) for j in range(36)]
    for name, mk in (("dm_m1024", lambda: C.dm_chain(24, 11, 1024, seed=5, device=dev)),
                     ("cyl_m4096_complex", lambda: C.model_inputs_complex(cyl, 17, 4096, seed=6, device=dev))):
        x = mk()
        d = x.dims
        real_flops = 4 * C.flops_per_matvec(d)        # a complex MAC = 4 real MACs
        reps = 2 if d["mL"] >= 4096 else 10
        with Heff(x.L, x.W1, x.W2, x.R) as h:
            out = torch.empty_like(x.psi)
            for _ in range(2):
                h.apply(x.psi, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                h.apply(x.psi, out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            h.set_option(OPT_PROFILE, 1)
            h.apply(x.psi, out)
            g1, mpo_ms, g4, _ = h.last_timings()
        row = {"config": name, **d, "matvec_ms": ms, "real_tflops": real_flops / ms / 1e9,
               "frac_peak": real_flops / ms / 1e9 / PEAK, "gemm_first_ms": g1, "mpo_ms": mpo_ms, "gemm_last_ms": g4}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del x
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
