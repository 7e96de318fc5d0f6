"""GPU parity of the environment update (NEXT-1) against the oracle, through the C ABI."""
import numpy as np
import pytest
import torch

from heffgen import env, mpo
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


CASES = [  # (mi, d, mo, kl, kr, W-maker)
    (128, 2, 256, 5, 5, lambda: mpo.heisenberg_chain_W()),
    (64, 2, 128, 20, 20, lambda: mpo.cylinder_W(17)),
    (64, 4, 256, 6, 6, lambda: mpo.hubbard_W()),
    (1024, 2, 1024, 5, 5, lambda: mpo.heisenberg_chain_W()),
    (37, 3, 29, 4, 3, None),                       # ragged, odd pitches -> plain-load GEMM path
    (1, 2, 2, 5, 5, lambda: mpo.heisenberg_chain_W()),   # the boundary step
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_env_update_parity(dev, orc, case):
    from paper_2007_14822_b200 import env_update_left, env_update_right
    mi, d, mo, kl, kr, wm = CASES[case]
    rng = np.random.default_rng(100 + case)
    W = wm() if wm else rng.standard_normal((kl, d, d, kr))
    L, A = rng.standard_normal((mi, kl, mi)), rng.standard_normal((mi, d, mo))
    R, B = rng.standard_normal((mi, kr, mi)), rng.standard_normal((mo, d, mi))
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    gl = env_update_left(t(L), t(A), t(W)).cpu().numpy()
    gr = env_update_right(t(R), t(B), t(W)).cpu().numpy()
    assert rel(gl, orc.env_left(L, A, W)) <= 1e-12
    assert rel(gr, orc.env_right(R, B, W)) <= 1e-12


def test_gpu_grown_environment_block_ED(dev):
    """Grow L on the GPU from the trivial boundary over a full-rank 6-site block: the done
    channel carries the block Hamiltonian's exact spectrum."""
    from paper_2007_14822_b200 import env_update_left
    n = 6
    As = env.draw_left_block(np.random.default_rng(1), n, 2, 64, dev)
    W = torch.from_numpy(mpo.heisenberg_chain_W()).to(dev)
    L = torch.zeros((1, 5, 1), dtype=torch.float64, device=dev)
    L[0, 4, 0] = 1.0
    for A in As:
        L = env_update_left(L, A.contiguous(), W)
    Lc = L.cpu().numpy()
    np.testing.assert_allclose(Lc[:, 4, :], np.eye(64), atol=1e-13)
    ev = np.linalg.eigvalsh(0.5 * (Lc[:, 0, :] + Lc[:, 0, :].T))
    np.testing.assert_allclose(ev, np.linalg.eigvalsh(ed_ref.heisenberg(n, ed_ref.chain_bonds(n)).toarray()),
                               atol=1e-12)


def test_env_update_c4_size_sampled_rows(dev, orc):
    """Environment updates at the C4 size (bond 4096 -> 4096, d = 2, the cylinder's k = 20
    MPO; L and the result 2.7 GB each) in the DMRG sweep's launch configuration; the oracle
    computes sampled output rows one by one."""
    from paper_2007_14822_b200 import env_update_left, env_update_right
    m, d = 4096, 2
    W = mpo.cylinder_W(17)
    k = W.shape[0]
    g = torch.Generator(device=dev).manual_seed(44)
    L = torch.randn((m, k, m), dtype=torch.float64, device=dev, generator=g)
    A = torch.randn((m, d, m), dtype=torch.float64, device=dev, generator=g)
    Wt = torch.from_numpy(W).to(dev)
    rows = [0, 1, 2047, m - 1]
    gl = env_update_left(L, A, Wt)[rows].cpu().numpy()
    Lh, Ah = L.cpu().numpy(), A.cpu().numpy()
    del L
    torch.cuda.empty_cache()
    ref = orc.env_left_rows(Lh, Ah, W, rows)
    for i in range(len(rows)):
        assert rel(gl[i], ref[i]) <= 1e-12, (rows[i], rel(gl[i], ref[i]))
    del Lh
    R = torch.randn((m, k, m), dtype=torch.float64, device=dev, generator=g)
    B = A.reshape(m, d, m)                       # any [b, s, y] tensor
    gr = env_update_right(R, B, Wt)[rows].cpu().numpy()
    ref = orc.env_right_rows(R.cpu().numpy(), Ah, W, rows)
    for i in range(len(rows)):
        assert rel(gr[i], ref[i]) <= 1e-12, (rows[i], rel(gr[i], ref[i]))
