"""GPU parity of the U(1) two-site split (heff_svd_split_qn, NEXT-2 x NEXT-3, reading R24)
against the oracle's block split (oracle/split.py svd_split_qn) on the same inputs."""
import numpy as np
import pytest
import torch

from heffgen import qn as hqn
from oracle import split as osplit

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _heff():
    from paper_2007_14822_b200 import heff
    return heff


def _cases():
    out = []
    for name, z in (("chain_m64", hqn.heisenberg_chain_qn(16, 7, 64, 5)),
                    ("chain_m128_Q2", hqn.heisenberg_chain_qn(18, 8, 128, 6, Q=2)),
                    ("cyl_m64", hqn.cylinder_qn(2, 5, 64, 7))):
        psi = z.x.psi.numpy()
        mL, d1, d2, mR = psi.shape
        qr, qc = osplit.qn_row_col_charges(z.qa, z.qs1, z.qs2, z.qb)
        out.append((name, psi.reshape(mL * d1, d2 * mR), qr, qc, z))
    return out


CASES = _cases()


@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("trunc", [dict(), dict(maxdim=40), dict(cutoff=1e-4), dict(cutoff=1e-8, maxdim=100)])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_qn_split_parity(case, trunc, direction):
    heff = _heff()
    name, Psi, qr, qc, z = CASES[case]
    qr_b, qc_b = heff.psi_row_col_charges(z.qa, z.qs1, z.qs2, z.qb)       # the binding's own bookkeeping
    assert list(qr_b) == list(qr) and list(qc_b) == list(qc)
    ref = osplit.svd_split_qn(Psi, qr, qc, direction=direction, **trunc)
    got = heff.svd_split_qn(torch.from_numpy(Psi).to(DEV), qr, qc, direction=direction, **trunc)
    fro = float(np.linalg.norm(Psi))
    np.testing.assert_allclose(got.S.cpu().numpy(), ref.S, rtol=0, atol=1e-12 * fro)
    assert got.n == ref.n and got.qk == list(ref.qk)
    assert got.trunc_err == pytest.approx(ref.trunc_err, rel=1e-9, abs=1e-14)
    np.testing.assert_allclose(got.Sk.cpu().numpy(), ref.Sk, rtol=0, atol=1e-12 * fro)
    Q, C = got.Q.cpu().numpy(), got.C.cpu().numpy()
    for k in range(got.n):                                               # charge conservation
        u = Q[:, k] if direction == 0 else C[:, k]
        v = C[k, :] if direction == 0 else Q[k, :]
        assert np.all(u[np.asarray(qr) != got.qk[k]] == 0.0) and np.all(v[np.asarray(qc) != got.qk[k]] == 0.0)
    G = Q.T @ Q if direction == 0 else Q @ Q.T
    np.testing.assert_allclose(G, np.eye(got.n), atol=1e-12)
    s = ref.S
    if got.n == s.size or s[got.n - 1] - s[got.n] > 1e-6 * s[0]:
        a = Q @ C if direction == 0 else C @ Q
        b = ref.Q @ ref.C if direction == 0 else ref.C @ ref.Q
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-11 * fro)


def test_qn_split_rejects_out_of_sector_entries():
    heff = _heff()
    name, Psi, qr, qc, z = CASES[0]
    bad = Psi.copy()
    i, j = np.nonzero(np.asarray(qr)[:, None] != np.asarray(qc)[None, :])
    bad[i[0], j[0]] = 1e-3
    with pytest.raises(heff.HeffError):
        heff.svd_split_qn(torch.from_numpy(bad).to(DEV), qr, qc)


def test_release_caches_frees_workspaces_and_splits_still_work():
    heff = _heff()
    name, Psi, qr, qc, z = CASES[1]
    P = torch.from_numpy(Psi).to(DEV)
    a = heff.svd_split_qn(P, qr, qc, maxdim=40)
    big = torch.from_numpy(np.random.default_rng(1).standard_normal((1024, 1024))).to(DEV)
    heff.svd_split(big, maxdim=100)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    heff.release_caches()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 > free0                                   # arenas returned to the device
    b = heff.svd_split_qn(P, qr, qc, maxdim=40)            # and re-grown on demand
    assert torch.equal(a.S, b.S) and a.qk == b.qk
