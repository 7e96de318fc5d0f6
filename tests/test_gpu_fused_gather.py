"""NEXT-5 gather-fused order-B path: GEMM_A reads psi's b-shards through
one TMA descriptor per shard -- local blocked buffers here (virtual shards on one GPU), NCCL
symmetric-window peer pointers in the communicating Lanczos -- against the oracle."""
import numpy as np
import pytest
import torch

from heffgen import configs as C

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-12
ENERGY_TOL = 1e-10


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name,m,P", [("c2", None, 1), ("c2", None, 2), ("c2", None, 4), ("c2", None, 8),
                                      ("c4", 64, 4), ("c3", None, 8)])
def test_apply_blocked_virtual_shards(dev, orc, name, m, P):
    from paper_2007_14822_b200 import Heff
    x = C.make(name, m=m)
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = x.to(dev)
    mL, d1, d2, mR = psi.shape
    nb = mR // P
    rows = mL * d1 * d2
    blocked = xd.psi.reshape(rows, P, nb).permute(1, 0, 2).contiguous()   # the all-gather layout
    parts = []
    for g in range(P):
        Rg = xd.R[g * nb:(g + 1) * nb].contiguous()
        with Heff(xd.L, xd.W1, xd.W2, Rg, dist=dict(nranks=P, rank=g, b_lo=g * nb, b_hi=(g + 1) * nb)) as h:
            out = h.apply_blocked(blocked)
            full = h.apply(xd.psi)
            torch.cuda.synchronize()
            assert torch.equal(out, full) or rel(out.cpu().numpy(), full.cpu().numpy()) <= 1e-14
            parts.append(out.cpu().numpy())
    got = np.concatenate(parts, axis=3)
    assert rel(got, ref) <= MATVEC_TOL


def test_apply_blocked_rejects_bad_shapes(dev):
    from paper_2007_14822_b200 import Heff, HeffError
    x = C.random_dense(dict(mL=12, d1=2, d2=2, mR=24, kL=3, kM=3, kR=3), seed=5).to(dev)
    with Heff(x.L, x.W1, x.W2, x.R[:12].contiguous(), dist=dict(nranks=2, rank=0, b_lo=0, b_hi=12)) as h:
        with pytest.raises(HeffError):                       # nb = 12 is not a multiple of 16
            h.apply_blocked(x.psi.reshape(48, 2, 12).permute(1, 0, 2).contiguous())
    with Heff(x.L, x.W1, x.W2, x.R) as h:                    # not sharded
        with pytest.raises(HeffError):
            h.apply_blocked(x.psi)


@pytest.mark.parametrize("mode", ["fixed", "converge"])
def test_lanczos_fused_gather_single_rank(dev, orc, mode):
    """The communicating Lanczos with the basis in an NCCL symmetric window and GEMM_A on the
    window's peer pointers (P = 1: the rank's own window through its LSA pointer)."""
    from paper_2007_14822_b200 import Heff, nccl_unique_id
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    conv = mode == "converge"
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=60 if conv else 20, tol=1e-10 if conv else 0.0, converge=conv)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R, dist=dict(nranks=1, rank=0, b_lo=0, b_hi=R.shape[0],
                                                   uid=nccl_unique_id())) as h:
        h.set_option(7, 1)
        for _ in range(2):                                    # second call reuses the window (epoch)
            v = xd.psi.clone()
            r = h.lanczos_ground(v, max_iter=60 if conv else 20, tol=1e-10 if conv else 0.0, converge=conv)
            assert h.get_option(7) == 3                      # requested and used
            assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy)), (r.energy, o.energy)
            assert r.iters == o.iters
        ov = abs(float(np.vdot(v.cpu().numpy().ravel(), o.x.ravel())))
        assert ov >= 1 - 1e-8
