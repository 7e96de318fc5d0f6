"""Multi-process (world_size 2, gloo, CPU) tests of the b'-sharded path's host logic
(DESIGN.md §8): the partition, the uid broadcast, max-over-ranks timing, the
all-gather layout map, and the distributed Lanczos decomposition (local order-B shard
matvecs + all-gather of psi + all-reduced dot products) against the single-process
oracle.  The shard matvec here is the oracle's order B; libheff runs the same
decomposition with its kernels and NCCL (tests/test_gpu_parity.py covers those on one GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_lanczos(rank, world, x, steps):
    """CGS2 Lanczos on b'-shards, organised like libheff's lanczos_ground."""
    from oracle import oracle
    from paper_2007_14822_b200 import dist as hdist

    L, W1, W2, R, psi = x
    mL, d1, d2, mR = psi.shape
    lo, hi = hdist.shard_range(mR, world, rank)
    rows = mL * d1 * d2

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    def matvec(v_shard):
        parts = [torch.empty(rows * (hi - lo), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(v_shard).ravel()))
        blocked = torch.stack(parts).reshape(world, rows, hi - lo)
        full = hdist.blocked_to_natural(blocked, world).numpy().reshape(mL, d1, d2, mR)
        return oracle.heff_apply_B(L, W1, W2, R, full, cols=(lo, hi))

    v = psi[..., lo:hi].copy()
    v /= np.sqrt(allreduce([np.vdot(v, v)])[0])
    V = [v]
    alpha, beta = [], []
    for j in range(steps):
        w = matvec(V[-1])
        c1 = allreduce([np.vdot(q, w) for q in V])
        w = w - sum(c * q for c, q in zip(c1, V))
        c2 = allreduce([np.vdot(q, w) for q in V])
        w = w - sum(c * q for c, q in zip(c2, V))
        alpha.append(c1[-1] + c2[-1])
        b = np.sqrt(allreduce([np.vdot(w, w)])[0])
        beta.append(b)
        V.append(w / b)
    T = np.diag(alpha) + np.diag(beta[:-1], 1) + np.diag(beta[:-1], -1)
    return float(np.linalg.eigvalsh(T)[0])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from heffgen import configs as C
        from paper_2007_14822_b200 import dist as hdist

        out = {}
        # partition
        out["ranges"] = [hdist.shard_range(64, world, r) for r in range(world)]
        # uid broadcast (rank 0's bytes reach everyone)
        uid = bytes(range(128)) if rank == 0 else None
        out["uid_ok"] = hdist.broadcast_uid(uid) == bytes(range(128))
        # max over ranks
        out["max"] = hdist.max_over_ranks(float(rank + 1))
        # distributed Lanczos vs the single-process oracle
        x = C.make("c2", m=32)
        xs = x.numpy()
        out["energy"] = _dist_lanczos(rank, world, xs, steps=12)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_host_logic_world2(oracle_lib):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from heffgen import configs as C
    x = C.make("c2", m=32)
    L, W1, W2, R, psi = x.numpy()
    ref = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=12)
    for r in range(world):
        assert res[r]["ranges"] == [(0, 32), (32, 64)]
        assert res[r]["uid_ok"]
        assert res[r]["max"] == 2.0
        assert abs(res[r]["energy"] - ref.energy) <= 1e-10 * max(1.0, abs(ref.energy))


def test_shard_range_errors():
    from paper_2007_14822_b200 import dist as hdist
    with pytest.raises(ValueError):
        hdist.shard_range(10, 3, 0)
    with pytest.raises(ValueError):
        hdist.shard_range(8, 2, 2)
    assert [hdist.shard_range(8192, 8, r) for r in (0, 7)] == [(0, 1024), (7168, 8192)]


def test_blocked_to_natural_layout():
    from paper_2007_14822_b200 import dist as hdist
    P, rows, nb = 3, 4, 5
    full = torch.arange(rows * P * nb, dtype=torch.float64).reshape(rows, P * nb)
    blocked = torch.stack([full[:, g * nb:(g + 1) * nb] for g in range(P)])
    assert torch.equal(hdist.blocked_to_natural(blocked, P), full)
