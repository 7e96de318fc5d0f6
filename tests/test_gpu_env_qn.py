"""U(1) environment updates (heff_env_update_left_qn / _right_qn, NEXT-1 x NEXT-3) against
the dense oracle environment update on the same charge-conserving inputs."""
import numpy as np
import pytest
import torch

from heffgen import mpo
from heffgen import qn as hqn

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


def _new_bond(values, mo):
    v = np.sort(np.asarray(values))
    idx = np.linspace(0, v.size - 1, mo).round().astype(int)
    return v[idx]


def _site_tensor(rng, q_left, qs, q_right):
    """A[x, s, a] ~ N(0,1) where q(a) = q(x) + q(s), else 0 (left-counted charges, R18)."""
    mask = q_right[None, None, :] == q_left[:, None, None] + qs[None, :, None]
    return rng.standard_normal(mask.shape) * mask


@pytest.mark.parametrize("force", [False, True])
@pytest.mark.parametrize("case", [("chain", 14, 6, 64, 48), ("chain", 16, 7, 128, 100), ("cyl", 12, 5, 64, 64)])
def test_env_update_qn_matches_dense_oracle(orc, case, force, monkeypatch):
    if force:   # the block-sparse schedule even where the dense one would be faster
        monkeypatch.setenv("HEFF_QN_FORCE_SPARSE", "1")
    from paper_2007_14822_b200 import heff
    model, N, window, m, mo = case
    z = (hqn.heisenberg_chain_qn(N, window, m, 3) if model == "chain" else hqn.cylinder_qn(N // 6, window, m, 3))
    W = mpo.heisenberg_chain_W() if model == "chain" else mpo.cylinder_W(window)
    c = hqn.heisenberg_channel_charges() if model == "chain" else hqn.cylinder_channel_charges()
    qs = np.array([1, -1])
    rng = np.random.default_rng(7)
    L, R = z.x.L.numpy(), z.x.R.numpy()
    # left: L's bond x (charges qa) grows by a site into bond a
    qa_new = _new_bond((z.qa[:, None] + qs[None, :]).ravel(), mo)
    A = _site_tensor(rng, z.qa, qs, qa_new)
    ref = orc.env_left(L, A, W)
    Wd = torch.from_numpy(W).to(DEV)
    got = heff.env_update_left(torch.from_numpy(L).to(DEV), torch.from_numpy(A).to(DEV), Wd,
                               qn=dict(q_in=z.qa, q_out=qa_new, qs=qs, cl=c, cr=c)).cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    # right: R's bond y (charges qb, left-counted) grows by a site into bond b, q(y) = q(b) + q(s)
    qb_new = _new_bond((z.qb[None, :] - qs[:, None]).ravel(), mo)
    B = np.transpose(_site_tensor(rng, qb_new, qs, z.qb), (0, 1, 2))
    ref = orc.env_right(R, B, W)
    got = heff.env_update_right(torch.from_numpy(R).to(DEV), torch.from_numpy(B).to(DEV), Wd,
                                qn=dict(q_in=z.qb, q_out=qb_new, qs=qs, cl=c, cr=c)).cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
