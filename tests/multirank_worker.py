"""One rank of the multi-GPU parity test (tests/test_gpu_multirank.py), started by
torch.multiprocessing.spawn with one process per GPU (never several ranks on one GPU).

Rank r owns b' in [r nb, (r+1) nb) of the C2-shaped workload, builds the communicating
b'-sharded libheff plan (order B, NCCL), and runs
  * heff_apply on the full psi -> its out shard,
  * lanczos_ground (fixed steps) through the NCCL all-gather + re-layout exchange,
  * lanczos_ground through the gather-fused path (NCCL symmetric window, NVLink peer reads),
then all-gathers the shards to rank 0, which writes them to `outdir` for the parent test to
compare with the oracle.  Inputs are generated identically on every rank (seeded, CPU).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def run(rank: int, world: int, port: int, outdir: str, config: str, steps: int):
    import numpy as np
    import torch
    import torch.distributed as dist

    from heffgen import configs as C
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200 import dist as hdist
    from paper_2007_14822_b200.heff import OPT_COMM_STATE, OPT_FUSED_GATHER, nccl_unique_id

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    try:
        x = C.make(config)                       # CPU, seeded: identical on every rank
        mR = x.dims["mR"]
        lo, hi = hdist.shard_range(mR, world, rank)
        xd = x.to(dev)
        uid = hdist.broadcast_uid(nccl_unique_id() if rank == 0 else None, device=dev)
        Rg = xd.R[lo:hi].contiguous()
        res = {}

        def gather_shards(t):
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t.contiguous())
            return torch.cat(parts, dim=-1)       # [mL, d1, d2, mR] in natural layout

        with Heff(xd.L, xd.W1, xd.W2, Rg, dist=dict(nranks=world, rank=rank, b_lo=lo, b_hi=hi, uid=uid)) as h:
            assert h.get_option(OPT_COMM_STATE) == 1
            out = h.apply(xd.psi)
            full_out = gather_shards(out)
            psi0 = xd.psi[..., lo:hi].contiguous()
            for mode in ("allgather", "fused"):
                h.set_option(OPT_FUSED_GATHER, 1 if mode == "fused" else 0)
                v = psi0.clone()
                r = h.lanczos_ground(v, max_iter=steps)
                fused_used = (h.get_option(OPT_FUSED_GATHER) & 2) != 0
                vf = gather_shards(v)
                res[mode] = dict(energy=r.energy, iters=r.iters, alpha=r.alpha, beta=r.beta, fused_used=fused_used)
                if rank == 0:
                    np.save(Path(outdir) / f"ritz_{mode}.npy", vf.cpu().numpy())
        if rank == 0:
            np.save(Path(outdir) / "matvec.npy", full_out.cpu().numpy())
            (Path(outdir) / "result.json").write_text(json.dumps(res))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def main(rank: int, world: int, port: int, outdir: str, config: str, steps: int):  # mp.spawn entry
    run(rank, world, port, outdir, config, steps)
