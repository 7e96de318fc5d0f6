"""Full-output checks of the CUDA path at full size against a closed form
(heffgen.closed.permuted_diagonal, tests/closed_form.py): every one of the 67 M outputs of
a C4-sized (m = 4096, d = 2) matvec in order A, every b'-shard of an 8-way order-B split of
it, and a d = 4 ragged case (m = 1024, mR = 768) -- where the sampled-row oracle parity of
test_gpu_parity.py sees only a few rows.  The expected values come from torch indexing and
a site-leg einsum, never from libheff."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    return torch.device("cuda:0")


def _maxrel(a, b):
    return float((a - b).abs().max() / b.abs().max())


@pytest.mark.parametrize("m,d,mR", [(4096, 2, 4096), (1024, 4, 768)])
def test_closed_form_full_output_order_A(dev, m, d, mR):
    from heffgen import closed
    from paper_2007_14822_b200 import Heff
    from tests import closed_form

    x = closed.permuted_diagonal(m, d, seed=12 + m, mR=mR).to(dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        out = h.apply(x.psi)
    ref = closed_form.expected_full_torch(closed.permuted_diagonal(m, d, seed=12 + m, mR=mR).meta, x.psi)
    assert _maxrel(out, ref) <= TOL


@pytest.mark.parametrize("m,d,mR,P", [(4096, 2, 4096, 8), (1024, 4, 768, 3)])
def test_closed_form_full_output_order_B_shards(dev, m, d, mR, P):
    from heffgen import closed
    from paper_2007_14822_b200 import Heff
    from tests import closed_form

    xc = closed.permuted_diagonal(m, d, seed=12 + m, mR=mR)
    x = xc.to(dev)
    ref = closed_form.expected_full_torch(xc.meta, x.psi)
    nb = mR // P
    for g in range(P):
        lo, hi = g * nb, (g + 1) * nb
        with Heff(x.L, x.W1, x.W2, x.R[lo:hi].contiguous(), dist=dict(nranks=P, rank=g, b_lo=lo, b_hi=hi)) as h:
            out = h.apply(x.psi)
        assert _maxrel(out, ref[..., lo:hi].contiguous()) <= TOL, g


@pytest.mark.parametrize("m,d,mR", [(4096, 2, 4096), (1024, 4, 768)])
def test_closed_form_lanczos_full_size(dev, m, d, mR):
    """lanczos_ground at full size against the closed-form ground state of the separable
    member (heffgen.closed.separable): E0 = min eL + min eig O1 + min eig O2 + min eR and the
    product ground state."""
    from heffgen import closed
    from paper_2007_14822_b200 import Heff

    xc = closed.separable(m, d, seed=33 + m, mR=mR)
    x = xc.to(dev)
    mt = xc.meta
    l1, u1 = np.linalg.eigh(mt["O1"])
    l2, u2 = np.linalg.eigh(mt["O2"])
    a0, b0 = int(np.argmin(mt["eL"])), int(np.argmin(mt["eR"]))
    E0 = mt["eL"][a0] + l1[0] + l2[0] + mt["eR"][b0]
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        v = x.psi.clone()
        r = h.lanczos_ground(v, max_iter=300, tol=1e-12, converge=True)
    assert abs(r.energy - E0) <= 1e-10 * max(1.0, abs(E0)), (r.energy, E0, r.iters)
    x0 = np.einsum("i,j->ij", u1[:, 0], u2[:, 0])
    ov = float(np.sum(v[a0, :, :, b0].cpu().numpy() * x0))
    assert abs(abs(ov) - 1.0) <= 1e-9, ov
