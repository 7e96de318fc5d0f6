"""GPU parity for the NEXT-4 matvec variants: MPO sums (heff_create_sum) and the
excited-state energy penalty (heff_set_penalty), through the C ABI."""
import numpy as np
import pytest
import torch

from heffgen import configs as C
from tests import ed_ref

pytestmark = pytest.mark.gpu


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


def test_mpo_sum_matvec_parity(dev, orc):
    from paper_2007_14822_b200 import Heff, HeffSum
    terms = C.heisenberg_chain_split(20, 9, 256, seed=1002)
    ref = orc.heff_apply_sum([t.numpy()[:4] for t in terms], terms[0].psi.numpy())
    td = [t.to(dev) for t in terms]
    plans = [Heff(t.L, t.W1, t.W2, t.R) for t in td]
    hs = HeffSum(plans)
    out = hs.apply(td[0].psi).cpu().numpy()
    assert rel(out, ref) <= 1e-12
    # plain-load GEMM path (accumulating epilogue of the non-TMA kernel)
    for p in plans:
        p.set_option(1, 1)
    out1 = hs.apply(td[0].psi).cpu().numpy()
    assert rel(out1, ref) <= 1e-12
    hs.close()
    for p in plans:
        p.close()


def test_mpo_sum_lanczos_ed(dev):
    from paper_2007_14822_b200 import Heff, HeffSum
    terms = [t.to(dev) for t in C.heisenberg_chain_split(10, 4, 16, seed=8)]
    plans = [Heff(t.L, t.W1, t.W2, t.R) for t in terms]
    with HeffSum(plans) as hs:
        r = hs.lanczos_ground(terms[0].psi.clone(), max_iter=300, tol=1e-10, converge=True)
    e0 = np.linalg.eigvalsh(ed_ref.heisenberg(10, ed_ref.chain_bonds(10)).toarray())[0]
    assert abs(r.energy - e0) <= 1e-10


def test_penalty_matvec_parity(dev, orc):
    from paper_2007_14822_b200 import Heff
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    rng = np.random.default_rng(3)
    phis = rng.standard_normal((3,) + psi.shape)
    phis /= np.linalg.norm(phis.reshape(3, -1), axis=1)[:, None, None, None, None]
    ref = orc.heff_apply_penalty(L, W1, W2, R, psi, phis, 2.5)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_penalty(torch.from_numpy(phis).to(dev), 2.5)
        out = h.apply(xd.psi).cpu().numpy()
        assert rel(out, ref) <= 1e-12
        h.set_penalty(None)
        out0 = h.apply(xd.psi).cpu().numpy()
    assert rel(out0, orc.heff_apply(L, W1, W2, R, psi)) <= 1e-12


def test_penalty_lanczos_first_excited_level(dev, orc):
    """with the ground state penalised the solver lands on the first excited level."""
    from paper_2007_14822_b200 import Heff
    x = C.make("c1_n8")
    L, W1, W2, R, psi = x.numpy()
    H = orc.heff_dense(L, W1, W2, R)
    ev, vec = np.linalg.eigh(0.5 * (H + H.T))
    phi0 = vec[:, 0].reshape((1,) + psi.shape)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_penalty(torch.from_numpy(phi0).to(dev), 10.0)
        r = h.lanczos_ground(xd.psi.clone(), max_iter=300, tol=1e-10, converge=True)
    ed = np.linalg.eigvalsh(ed_ref.heisenberg(8, ed_ref.chain_bonds(8)).toarray())
    assert abs(r.energy - ed[1]) <= 1e-10


def test_penalty_unaligned_psi(dev, orc):
    """psi / out only 8-byte aligned: the penalty kernels take their scalar path."""
    from paper_2007_14822_b200 import Heff
    x = C.random_dense(dict(mL=7, d1=2, d2=3, mR=5, kL=3, kM=2, kR=4), seed=5)
    L, W1, W2, R, psi = x.numpy()
    phis = np.random.default_rng(1).standard_normal((2,) + psi.shape)
    ref = orc.heff_apply_penalty(L, W1, W2, R, psi, phis, -1.5)
    xd = x.to(dev)
    n = psi.size
    buf_in = torch.zeros(n + 1, dtype=torch.float64, device=dev)
    buf_out = torch.zeros(n + 1, dtype=torch.float64, device=dev)
    pin, pout = buf_in[1:], buf_out[1:]
    pin.copy_(xd.psi.ravel())
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_penalty(torch.from_numpy(phis).to(dev), -1.5)
        h.apply(pin.view(psi.shape), pout.view(psi.shape))
    assert rel(pout.cpu().numpy().reshape(psi.shape), ref) <= 1e-12
