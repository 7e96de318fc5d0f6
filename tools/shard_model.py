"""Per-rank compute of the P-way b'-sharded matvec, measured on one GPU.

Only one GPU is available to this build, so the P > 1 path cannot run end to end.  What one
GPU can measure is the work every rank does: the order-B matvec of one b'-shard (GEMM_A
from the P shards through per-shard TMA descriptors, the order-B MPO kernel, GEMM_D) at the
shard shapes of P = 1, 2, 4, 8 -- `heff_apply_blocked` on virtual shards.  The predicted
strong-scaling efficiency t(1) / (P t_rank(P)) ignores the exchange, which the
gather-fused path spreads over GEMM_A (0.47 GB per rank per matvec at C4, P = 8: ~0.6 ms at
NVLink rates against ~77 ms of compute) and the Lanczos scalar all-reduces.

    python tools/shard_model.py [--config c4] [--ranks 1,2,4,8] [--out profiles/...json]
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

PEAK = 148 * 128 * 1.965e9 / 1e12


def timed(fn, reps):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    x = C.make(a.config, device=dev)
    d = x.dims
    flops = C.flops_per_matvec(d)
    rows = d["mL"] * d["d1"] * d["d2"]
    mR = d["mR"]
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        out = torch.empty_like(x.psi)
        t_a = timed(lambda: h.apply(x.psi, out), a.reps)
    res = []
    t1 = None
    for P in [int(p) for p in a.ranks.split(",")]:
        nb = mR // P
        blocked = x.psi.reshape(rows, P, nb).permute(1, 0, 2).contiguous()
        row = dict(config=a.config, P=P, nb=nb)
        for g in sorted({0, P - 1}):
            Rg = x.R[g * nb:(g + 1) * nb].contiguous()
            torch.cuda.synchronize()
            free0, _ = torch.cuda.mem_get_info()
            with Heff(x.L, x.W1, x.W2, Rg, dist=dict(nranks=P, rank=g, b_lo=g * nb, b_hi=(g + 1) * nb)) as h:
                torch.cuda.synchronize()
                row["plan_workspace_gb_measured"] = (free0 - torch.cuda.mem_get_info()[0]) / 2**30
                o = torch.empty(h.out_shape, dtype=torch.float64, device=dev)
                t = timed(lambda: h.apply_blocked(blocked, o), a.reps)
            row[f"rank{g}_ms"] = t
            del Rg
        # per-rank device memory of a communicating rank (analytic, bytes): full L, W1/W2, its R
        # rows, V1 + V3 (order-B intermediates), the gathered full psi + the blocked all-gather
        # buffer, a 20-vector Krylov basis of shards and the work vector
        shard = rows * nb
        mem = {"L": d["mL"] * d["kL"] * d["mL"], "R_shard": nb * d["kR"] * mR,
               "V1": rows * nb * d["kR"], "V3": d["kL"] * rows * nb, "psi_full": rows * mR,
               "allgather_buffer": rows * mR if P > 1 else 0, "krylov_basis_20": 20 * shard, "work": shard}
        row["per_rank_memory_gb"] = {k: v * 8 / 2**30 for k, v in mem.items()}
        row["per_rank_memory_gb"]["total"] = sum(mem.values()) * 8 / 2**30
        t_rank = max(row[f"rank{g}_ms"] for g in sorted({0, P - 1}))
        if P == 1:
            t1 = t_rank
        row.update(t_rank_ms=t_rank, rank_tflops=flops / P / (t_rank * 1e-3) / 1e12,
                   rank_frac_peak=flops / P / (t_rank * 1e-3) / 1e12 / PEAK,
                   predicted_matvec_per_s=1e3 / t_rank, orderA_1gpu_ms=t_a,
                   predicted_efficiency_vs_orderB_P1=(t1 / (P * t_rank)) if t1 else None,
                   predicted_efficiency_vs_orderA=t_a / (P * t_rank))
        print(json.dumps(row), flush=True)
        res.append(row)
        del blocked
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
