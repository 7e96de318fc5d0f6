"""Pins for the environment-update oracle (NEXT-1; SPEC ProjMPO S:L737-755, Sec. 6.2
P:L705-737).  Independent sides: ED of the block Hamiltonian (Kronecker), the identity
channel, and the full-rank H_eff spectrum."""
import numpy as np
import torch

from heffgen import env, mpo
from tests import ed_ref


def grow_left_oracle(orc, Ws, As):
    k = Ws[0].shape[0]
    L = np.zeros((1, k, 1))
    L[0, k - 1, 0] = 1.0
    for A, W in zip(As, Ws):
        L = orc.env_left(L, A, W)
    return L


def grow_right_oracle(orc, Ws, Bs):
    k = Ws[-1].shape[3]
    R = np.zeros((1, k, 1))
    R[0, 0, 0] = 1.0
    for B, W in zip(reversed(Bs), reversed(Ws)):
        R = orc.env_right(R, B, W)
    return R


def full_rank_blocks(n, d, seed):
    rng = np.random.default_rng(seed)
    As = [t.numpy() for t in env.draw_left_block(rng, n, d, d ** n, "cpu")]
    Bs = [t.numpy() for t in env.draw_right_block(rng, n, d, d ** n, "cpu")]
    return As, Bs


def test_left_env_done_channel_spectrum_is_block_ED(oracle_lib):
    n = 5
    As, Bs = full_rank_blocks(n, 2, seed=3)
    W = mpo.heisenberg_chain_W()
    L = grow_left_oracle(oracle_lib, [W] * n, As)
    assert L.shape == (32, 5, 32)
    np.testing.assert_allclose(L[:, 4, :], np.eye(32), atol=1e-13)          # identity channel
    ev = np.linalg.eigvalsh(0.5 * (L[:, 0, :] + L[:, 0, :].T))             # projected block H
    ev_ed = np.linalg.eigvalsh(ed_ref.heisenberg(n, ed_ref.chain_bonds(n)).toarray())
    np.testing.assert_allclose(ev, ev_ed, atol=1e-12)


def test_right_env_done_channel_spectrum_is_block_ED(oracle_lib):
    n = 5
    As, Bs = full_rank_blocks(n, 2, seed=4)
    W = mpo.heisenberg_chain_W()
    R = grow_right_oracle(oracle_lib, [W] * n, Bs)
    np.testing.assert_allclose(R[:, 0, :], np.eye(32), atol=1e-13)
    ev = np.linalg.eigvalsh(0.5 * (R[:, 4, :] + R[:, 4, :].T))             # start channel = block H
    ev_ed = np.linalg.eigvalsh(ed_ref.heisenberg(n, ed_ref.chain_bonds(n)).toarray())
    np.testing.assert_allclose(ev, ev_ed, atol=1e-12)


def test_cylinder_column_block_ED(oracle_lib):
    n = 6                                     # one full column of the width-6 cylinder
    As, _ = full_rank_blocks(n, 2, seed=5)
    Ws = [mpo.cylinder_W(j) for j in range(n)]
    L = grow_left_oracle(oracle_lib, Ws, As)
    ev = np.linalg.eigvalsh(0.5 * (L[:, 0, :] + L[:, 0, :].T))
    bonds = [(i, j, J) for (i, j, J) in ed_ref.cylinder_bonds(2) if j < n]
    ev_ed = np.linalg.eigvalsh(ed_ref.heisenberg(n, bonds).toarray())
    np.testing.assert_allclose(ev, ev_ed, atol=1e-12)


def test_oracle_environments_give_ED_spectrum(oracle_lib):
    """H_eff built from oracle-grown L, R (N = 10 chain, window (4,5), full rank) has the ED spectrum."""
    As, Bs = full_rank_blocks(4, 2, seed=6)
    W = mpo.heisenberg_chain_W()
    L = grow_left_oracle(oracle_lib, [W] * 4, As)
    R = grow_right_oracle(oracle_lib, [W] * 4, Bs)
    H = oracle_lib.heff_dense(L, W, W, R)
    ev = np.linalg.eigvalsh(0.5 * (H + H.T))
    ev_ed = np.linalg.eigvalsh(ed_ref.heisenberg(10, ed_ref.chain_bonds(10)).toarray())
    np.testing.assert_allclose(ev, ev_ed, atol=1e-11)


def test_env_ragged_brute_force(oracle_lib):
    rng = np.random.default_rng(9)
    mi, d, mo, kl, kr = 3, 2, 5, 4, 3
    L, A, W = rng.standard_normal((mi, kl, mi)), rng.standard_normal((mi, d, mo)), rng.standard_normal((kl, d, d, kr))
    ref = np.einsum("xpa,xwy,wpsv,ysb->avb", A, L, W, A, optimize=False)
    np.testing.assert_allclose(oracle_lib.env_left(L, A, W), ref, rtol=1e-13, atol=1e-13)
    R, B = rng.standard_normal((mi, kr, mi)), rng.standard_normal((mo, d, mi))
    ref = np.einsum("apx,xvy,wpsv,bsy->awb", B, R, W, B, optimize=False)
    np.testing.assert_allclose(oracle_lib.env_right(R, B, W), ref, rtol=1e-13, atol=1e-13)


def test_env_row_oracle_matches_full_update():
    """The row-at-a-time environment oracle (used for sampled checks at full size) against
    the full C update on random and ragged shapes, every row."""
    from oracle import oracle as orc
    orc.build()
    rng = np.random.default_rng(5)
    for (mi, d, mo, kl, kr) in ((7, 2, 9, 5, 5), (16, 3, 11, 4, 6), (1, 2, 2, 5, 5)):
        L, A = rng.standard_normal((mi, kl, mi)), rng.standard_normal((mi, d, mo))
        R, B = rng.standard_normal((mi, kr, mi)), rng.standard_normal((mo, d, mi))
        W = rng.standard_normal((kl, d, d, kr))
        full_l, full_r = orc.env_left(L, A, W), orc.env_right(R, B, W)
        rows = list(range(mo))
        np.testing.assert_allclose(orc.env_left_rows(L, A, W, rows), full_l, rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(orc.env_right_rows(R, B, W, rows), full_r, rtol=1e-13, atol=1e-13)
