"""GPU parity of complex plans (heff_create_z; NEXT-4 complex) against the complex oracle:
matvec at several sizes and both GEMM load paths, Hermitian Lanczos vs oracle and ED."""
import numpy as np
import pytest
import torch

from heffgen import configs as C
from tests.test_oracle_complex import dm_dense

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


def random_complex(dims, seed):
    rng = np.random.default_rng(seed)
    c = lambda *s: torch.from_numpy(rng.standard_normal(s) + 1j * rng.standard_normal(s))
    mL, d1, d2, mR, kL, kM, kR = (dims[k] for k in ("mL", "d1", "d2", "mR", "kL", "kM", "kR"))
    psi = c(mL, d1, d2, mR)
    return C.HeffInputs(c(mL, kL, mL), c(kL, d1, d1, kM), c(kM, d2, d2, kR), c(mR, kR, mR), psi / psi.norm())


CASES = {
    "dm_n8": lambda: C.dm_chain(8, 2, 16, seed=3),
    "dm_m256": lambda: C.dm_chain(20, 9, 256, seed=4),
    "dm_m1024": lambda: C.dm_chain(24, 11, 1024, seed=5),
    "ragged": lambda: random_complex(dict(mL=37, d1=3, d2=2, mR=29, kL=4, kM=3, kR=5), seed=6),
    "tails": lambda: random_complex(dict(mL=130, d1=2, d2=2, mR=258, kL=3, kM=2, kR=5), seed=7),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("path", [0, 1])
def test_complex_matvec_parity(dev, orc, case, path):
    from paper_2007_14822_b200 import Heff
    x = CASES[case]()
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply_z(L, W1, W2, R, psi)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_option(1, path)
        out = h.apply(xd.psi).cpu().numpy()
    assert out.dtype == np.complex128
    assert rel(out, ref) <= 1e-12, rel(out, ref)


def test_complex_lanczos_parity_and_ed(dev, orc):
    from paper_2007_14822_b200 import Heff
    x = C.dm_chain(20, 9, 256, seed=8)
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff_z(L, W1, W2, R, psi, max_iter=15)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        v = xd.psi.clone()
        r = h.lanczos_ground(v, max_iter=15)
    assert abs(r.energy - o.energy) <= 1e-10 * max(1.0, abs(o.energy))
    np.testing.assert_allclose(r.alpha, o.alpha, atol=1e-10)
    np.testing.assert_allclose(r.beta, o.beta, atol=1e-10)
    vc = v.cpu().numpy()
    assert abs(abs(np.vdot(vc, o.x)) - 1.0) < 1e-8
    # full rank N = 8: converged energy = ED of the complex Hermitian Hamiltonian
    x = C.dm_chain(8, 2, 16, seed=9).to(dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        r = h.lanczos_ground(x.psi.clone(), max_iter=300, tol=1e-10, converge=True)
    assert abs(r.energy - np.linalg.eigvalsh(dm_dense(8))[0]) <= 1e-10


def test_complex_apply_host_and_guards(dev, orc):
    from paper_2007_14822_b200 import Heff, HeffError
    x = C.dm_chain(20, 9, 64, seed=10)
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply_z(L, W1, W2, R, psi)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        out = torch.empty(x.psi.shape, dtype=torch.complex128).pin_memory()
        h.apply_host(x.psi.contiguous(), out)
        assert rel(out.numpy(), ref) <= 1e-12
        with pytest.raises((HeffError, TypeError)):
            h.set_penalty(torch.zeros((1,) + tuple(x.psi.shape), dtype=torch.complex128, device=dev), 1.0)
        with pytest.raises(TypeError):
            h.apply(xd.psi.real.contiguous())


def test_complex_c4_size_sampled_rows(dev, orc):
    """A complex problem of the C4 size (6x6 cylinder MPO, m = 4096, random complex
    environments) in the launch configuration of tools/sweep_complex.py; the complex oracle
    computes sampled output rows a' one by one."""
    from heffgen import mpo
    from paper_2007_14822_b200 import Heff
    cyl = [mpo.cylinder_W(j).astype(complex) for j in range(36)]
    x = C.model_inputs_complex(cyl, 17, 4096, seed=6, device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        out = h.apply(x.psi)
        torch.cuda.synchronize()
    rows = [0, 2047, 4095]
    outc = out[rows].cpu().numpy()
    del out
    L, W1, W2, R, psi = x.numpy()
    del x
    torch.cuda.empty_cache()
    for i, a in enumerate(rows):
        ref = orc.heff_apply_z(L, W1, W2, R, psi, rows=(a, a + 1))[0]
        assert rel(outc[i], ref) <= 1e-12, (a, rel(outc[i], ref))
