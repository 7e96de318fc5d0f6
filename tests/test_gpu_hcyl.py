"""The d = 4, k = 26 Hubbard cylinder (width 6; k d1 d2 = 416 staged MPO rows, above the
128-wide column tile's 200-row budget): the MPO kernels run 32-wide column tiles, the
two-site MPO CSR is built on the device.  Parity against the oracle in both orders, Lanczos,
and the CSR's nonzero count against a plain numpy contraction of W1 W2."""
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


@pytest.mark.parametrize("path", [0, 1, 2])
def test_hcyl6_matvec_order_A(dev, orc, path):
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200.heff import OPT_MPO_NNZ
    x = C.make("hcyl6", m=64)
    L, W1, W2, R, psi = x.numpy()
    assert W1.shape == (26, 4, 4, 26)
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_option(1, path)
        out = h.apply(xd.psi).cpu().numpy()
        Wc = np.einsum("asbx,xtcy->stybac", W1, W2)      # rows (s1',s2',w2), cols (w,s1,s2)
        assert h.get_option(OPT_MPO_NNZ) == int(np.count_nonzero(Wc))
    assert rel(out, ref) <= MATVEC_TOL


def test_hcyl6_lanczos(dev, orc):
    from paper_2007_14822_b200 import Heff
    x = C.make("hcyl6", m=48)
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=16)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        r = h.lanczos_ground(xd.psi.clone(), max_iter=16)
    assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))


@pytest.mark.parametrize("P", [2, 4])
def test_hcyl6_order_B_shards(dev, orc, P):
    """Order B (GEMM_A on the (w2, b')-reordered R shard, the order-B MPO CSR on the device,
    416 staged rows -> 32-wide tiles) on virtual shards, full psi and blocked layout."""
    from paper_2007_14822_b200 import Heff
    x = C.make("hcyl6", m=64)
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply_B(L, W1, W2, R, psi)
    xd = x.to(dev)
    mL, d1, d2, mR = psi.shape
    nb = mR // P
    rows = mL * d1 * d2
    blocked = xd.psi.reshape(rows, P, nb).permute(1, 0, 2).contiguous()
    parts = []
    for g in range(P):
        Rg = xd.R[g * nb:(g + 1) * nb].contiguous()
        with Heff(xd.L, xd.W1, xd.W2, Rg, dist=dict(nranks=P, rank=g, b_lo=g * nb, b_hi=(g + 1) * nb)) as h:
            out = h.apply(xd.psi)
            outb = h.apply_blocked(blocked)
            torch.cuda.synchronize()
            assert rel(outb.cpu().numpy(), out.cpu().numpy()) <= 1e-14
            parts.append(out.cpu().numpy())
    assert rel(np.concatenate(parts, axis=3), ref) <= MATVEC_TOL


def test_hcyl6_large_bond_sampled_rows(dev, orc):
    """m = 1024 (k d^2 m^2 ... the T1/T3 intermediates 3.5 GB each): sampled output rows a'."""
    from paper_2007_14822_b200 import Heff
    x = C.make("hcyl6", m=1024, device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        out = h.apply(x.psi)
        torch.cuda.synchronize()
    L, W1, W2, R, psi = (t.cpu().numpy() for t in (x.L, x.W1, x.W2, x.R, x.psi))
    for a in (0, 517, 1023):
        ref = orc.heff_apply(L, W1, W2, R, psi, rows=(a, a + 1))[0]
        assert rel(out[a].cpu().numpy(), ref) <= MATVEC_TOL, a


def test_env_update_d4_k26(dev, orc):
    """Environment updates with the k = 26, d = 4 site MPO (one-site CSR built on the device)."""
    from heffgen import mpo
    from paper_2007_14822_b200 import heff
    rng = np.random.default_rng(3)
    W = mpo.hubbard_cylinder_W(14)
    mi, mo, d, k = 40, 56, 4, W.shape[0]
    L = rng.standard_normal((mi, k, mi))
    A = rng.standard_normal((mi, d, mo))
    ref = orc.env_left(L, A, W)
    got = heff.env_update_left(*(torch.from_numpy(np.ascontiguousarray(t)).to(dev) for t in (L, A, W))).cpu().numpy()
    assert rel(got, ref) <= MATVEC_TOL
    Rt = rng.standard_normal((mi, k, mi))
    B = rng.standard_normal((mo, d, mi))
    ref = orc.env_right(Rt, B, W)
    got = heff.env_update_right(*(torch.from_numpy(np.ascontiguousarray(t)).to(dev) for t in (Rt, B, W))).cpu().numpy()
    assert rel(got, ref) <= MATVEC_TOL
