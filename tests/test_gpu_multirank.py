"""Multi-GPU parity of the b'-sharded path (north_star (4)): P ranks, one per
GPU, each running order B on its b'-shard with NCCL, against the CPU oracle.

The matvec gathered from the P out-shards must match the oracle to 1e-12 (relative
Frobenius); the fixed-step Lanczos energy through BOTH exchanges (ncclAllGather + re-layout,
and the gather-fused NVLink path) must match the oracle's fixed-step Lanczos to 1e-10, and
the Ritz vectors gathered from the shards must agree with the oracle's.  Skipped when fewer
than P GPUs are visible -- ranks are never emulated as processes sharing one GPU.
"""
import json
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-12
ENERGY_TOL = 1e-10
STEPS = 6


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_lanczos_multirank(P, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs, {torch.cuda.device_count() if torch.cuda.is_available() else 0} visible")
    import torch.multiprocessing as mp

    import __graft_entry__ as g
    g.build()
    from heffgen import configs as C
    from oracle import oracle
    from tests import multirank_worker

    cfg = "c2"                                    # m = 256: nb = 128 / 64 / 32 (fused path needs nb % 16 == 0)
    mp.spawn(multirank_worker.main, args=(P, _free_port(), str(tmp_path), cfg, STEPS), nprocs=P, join=True)

    oracle.build()
    x = C.make(cfg)
    L, W1, W2, R, psi = x.numpy()
    ref = oracle.heff_apply(L, W1, W2, R, psi)
    out = np.load(tmp_path / "matvec.npy")
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= MATVEC_TOL
    o = oracle.lanczos_heff(L, W1, W2, R, psi, max_iter=STEPS)
    res = json.loads((tmp_path / "result.json").read_text())
    assert res["fused"]["fused_used"] and not res["allgather"]["fused_used"]
    for mode in ("allgather", "fused"):
        r = res[mode]
        assert r["iters"] == o.iters
        assert abs(r["energy"] - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy)), (mode, r["energy"], o.energy)
        v = np.load(tmp_path / f"ritz_{mode}.npy").reshape(-1)
        assert abs(abs(float(np.dot(v, o.x.reshape(-1)))) - 1.0) <= 1e-10, mode
