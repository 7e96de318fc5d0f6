"""Pins for the U(1) inputs of the block-sparse H_eff (NEXT-3): the declared structure
holds, H_eff maps the sector to itself, and the sector's lowest eigenvalue is the ED
ground energy of the conserved-Sz block.  CPU only."""
import numpy as np

from heffgen import mpo, qn
from tests import ed_ref


def test_mpo_channel_charges_conserve_sz():
    assert qn.check_mpo_charges(mpo.heisenberg_chain_W(), qn.heisenberg_channel_charges(), qn.SPIN_Q)
    assert all(qn.check_mpo_charges(mpo.cylinder_W(j), qn.cylinder_channel_charges(), qn.SPIN_Q) for j in range(36))
    bad = qn.heisenberg_channel_charges().copy()
    bad[1] = 2
    assert not qn.check_mpo_charges(mpo.heisenberg_chain_W(), bad, qn.SPIN_Q)


def _violations(z):
    L, W1, W2, R, psi = z.x.numpy()
    qa, qb = z.qa, z.qb
    mL = (qa[:, None, None] - qa[None, None, :] != z.cL[None, :, None]) & (np.abs(L) > 0)
    mR = (qb[:, None, None] - qb[None, None, :] != z.cR[None, :, None]) & (np.abs(R) > 0)
    mP = (~z.mask()) & (np.abs(psi) > 0)
    return int(mL.sum()), int(mR.sum()), int(mP.sum())


def test_declared_structure_holds():
    for z in (qn.heisenberg_chain_qn(20, 9, 64, seed=1), qn.cylinder_qn(2, 5, 32, seed=2),
              qn.heisenberg_chain_qn(12, 5, 24, seed=3, Q=2)):
        assert _violations(z) == (0, 0, 0)
        assert np.all(np.diff(z.qa) >= 0) and np.all(np.diff(z.qb) >= 0)


def test_heff_preserves_sector(oracle_lib):
    z = qn.heisenberg_chain_qn(20, 9, 64, seed=4)
    L, W1, W2, R, psi = z.x.numpy()
    out = oracle_lib.heff_apply(L, W1, W2, R, psi)
    assert np.abs(out[~z.mask()]).max() == 0.0
    assert np.abs(out[z.mask()]).max() > 1e-3


def test_sector_ground_energy_is_ED(oracle_lib):
    """N = 10 full rank, Sz = 0 sector (dim C(10,5) = 252) and Sz = 1 (2Sz = 2, dim 210)."""
    H = ed_ref.heisenberg(10, ed_ref.chain_bonds(10)).toarray()
    sz2 = np.array([sum(1 if (i >> (9 - k)) & 1 == 0 else -1 for k in range(10)) for i in range(1024)])
    for Q in (0, 2):
        z = qn.heisenberg_chain_qn(10, 4, 16, seed=5, Q=Q)
        L, W1, W2, R, psi = z.x.numpy()
        m = z.mask().ravel()
        Hs = oracle_lib.heff_dense(L, W1, W2, R)[np.ix_(m, m)]
        sect = sz2 == Q
        assert m.sum() == sect.sum()
        np.testing.assert_allclose(np.linalg.eigvalsh(0.5 * (Hs + Hs.T)), np.linalg.eigvalsh(H[np.ix_(sect, sect)]),
                                   atol=1e-12)
        r = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=300, tol=1e-10, converge=True)
        assert abs(r.energy - np.linalg.eigvalsh(H[np.ix_(sect, sect)])[0]) <= 1e-10
