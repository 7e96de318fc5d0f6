"""U(1) block-sparse H_eff (NEXT-3) vs dense on the same sector-structured inputs, one GPU.

    python tools/sweep_qn.py [--out profiles/qn.json]
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
from heffgen import qn  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402
from paper_2007_14822_b200.heff import OPT_PROFILE, OPT_SPARSE_KBLOCKS  # noqa: E402

PEAK = 148 * 128 * 1.965e9 / 1e12


def t_apply(h, psi, out, reps):
    for _ in range(2):
        h.apply(psi, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        h.apply(psi, out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", default="c3qn,c4qn")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    makers = {"c2qn": lambda: qn.heisenberg_chain_qn(20, 9, 256, seed=2002, device=dev),
              "c3qn": lambda: qn.heisenberg_chain_qn(24, 11, 1024, seed=2003, device=dev),
              "c4qn": lambda: qn.cylinder_qn(6, 17, 4096, seed=2004, device=dev)}
    for name in args.configs.split(","):
        t0 = time.perf_counter()
        z = makers[name]()
        gen = time.perf_counter() - t0
        x = z.x
        d = x.dims
        flops = C.flops_per_matvec(d)
        reps = 2 if d["mL"] >= 4096 else 10
        with Heff(x.L, x.W1, x.W2, x.R) as h:
            out = torch.empty_like(x.psi)
            ms_dense = t_apply(h, x.psi, out, reps)
            ref = out.clone()
            h.set_qn(z.qn_dict())
            nkb = h.get_option(OPT_SPARSE_KBLOCKS)
            ms_sparse = t_apply(h, x.psi, out, reps)
            err = (torch.linalg.norm(out - ref) / torch.linalg.norm(ref)).item()
            h.set_option(OPT_PROFILE, 1)
            h.apply(x.psi, out)
            g1, mpo_ms, g4, _ = h.last_timings()
            h.set_option(OPT_PROFILE, 0)
            steps = 3 if d["mL"] >= 4096 else 20
            h.lanczos_ground(x.psi.clone(), max_iter=steps)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            h.lanczos_ground(x.psi.clone(), max_iter=steps)
            lz_sparse = (time.perf_counter() - t1) / steps * 1e3
        sched_flops = nkb * 2.0 * 128 * 128 * 16        # tile-padded work actually scheduled
        row = {"config": name, **d, "gen_s": round(gen, 1), "sector_dim": int(z.mask().sum()),
               "dense_elems": int(z.mask().size), "dense_ms": ms_dense, "sparse_ms": ms_sparse,
               "speedup": ms_dense / ms_sparse, "rel_diff_vs_dense": err, "sched_kblock_tiles": nkb,
               "sched_gemm_tflops": sched_flops / ((g1 + g4) / 1e3) / 1e12 if (g1 + g4) else None,
               "sparse_gemm_first_ms": g1, "sparse_mpo_ms": mpo_ms, "sparse_gemm_last_ms": g4,
               "dense_equiv_tflops": flops / ms_sparse / 1e9, "sparse_lanczos_step_ms": lz_sparse}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del x, z
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
