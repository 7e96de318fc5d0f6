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
