"""Full-size sharded parity (BASELINE.json configs[3-4]): every P = 8 b'-shard
plan of C4 (m = 4096, nb = 512) and C5 (m = 8192, d = 4, nb = 1024) built on one GPU, in the
launch configuration the multi-GPU bench runs (order B; GEMM_A from the full psi and, through
heff_apply_blocked, from the blocked all-gather layout's P shard descriptors).

The oracle (order B, oracle.heff_apply_B_cols) computes sampled output columns b' one by
one: both edges of every shard plus interior columns; each must match to 1e-12 relative.
heff_apply and heff_apply_blocked must agree with each other on the whole shard.
"""
import numpy as np
import pytest
import torch

from heffgen import configs as C

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-12
P = 8


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    return torch.device("cuda:0")


def _shard_parity(dev, cfg, interior):
    from oracle import oracle
    from paper_2007_14822_b200 import Heff
    oracle.build()
    x = C.make(cfg, device=dev)
    d = x.dims
    mR = d["mR"]
    nb = mR // P
    rows = d["mL"] * d["d1"] * d["d2"]
    cols, got = [], []
    blocked = x.psi.reshape(rows, P, nb).permute(1, 0, 2).contiguous()   # what the all-gather delivers
    for g in range(P):
        Rg = x.R[g * nb:(g + 1) * nb].contiguous()
        with Heff(x.L, x.W1, x.W2, Rg, dist=dict(nranks=P, rank=g, b_lo=g * nb, b_hi=(g + 1) * nb)) as h:
            out = h.apply(x.psi)
            outb = h.apply_blocked(blocked)
            torch.cuda.synchronize()
            diff = float(torch.linalg.norm(out - outb) / torch.linalg.norm(out))
            assert diff <= 1e-14, (g, diff)
            loc = sorted({0, nb - 1, *[(i * 131 + 17 * g) % nb for i in range(interior)]})
            cols += [g * nb + j for j in loc]
            got.append(outb[..., loc].cpu().numpy())
        del Rg
    del blocked
    torch.cuda.empty_cache()
    got = np.concatenate(got, axis=3)
    L, W1, W2, R, psi = (t.cpu().numpy() for t in (x.L, x.W1, x.W2, x.R, x.psi))
    ref = oracle.heff_apply_B_cols(L, W1, W2, R, psi, cols)
    for i, b in enumerate(cols):
        e = np.linalg.norm(got[..., i] - ref[..., i]) / np.linalg.norm(ref[..., i])
        assert e <= MATVEC_TOL, (cfg, b, e)


def test_c4_p8_shards_fullsize(dev):
    _shard_parity(dev, "c4", interior=2)


def test_c5_p8_shards_fullsize(dev):
    free, _ = torch.cuda.mem_get_info()
    if free < 60 * 2**30:
        pytest.skip("C5 shard parity needs ~45 GB of free device memory")
    _shard_parity(dev, "c5", interior=0)
