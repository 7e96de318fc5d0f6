"""Pins for the NEXT-4 matvec variants: MPO sums and the
excited-state energy penalty.  CPU only."""
import numpy as np
import pytest

from heffgen import configs as C
from heffgen import mpo
from tests import ed_ref


def test_split_mpo_terms_sum_to_eq1():
    l3, r3 = mpo.boundary_vectors(3)
    l4, r4 = mpo.boundary_vectors(4)
    for N in (2, 3, 4):
        Hzz = ed_ref.mpo_dense([mpo.heisenberg_zz_W()] * N, l3, r3)
        Hfl = ed_ref.mpo_dense([mpo.heisenberg_flip_W()] * N, l4, r4)
        Hk = ed_ref.heisenberg(N, ed_ref.chain_bonds(N)).toarray()
        assert np.array_equal(Hzz + Hfl, Hk)
        # the Sz Sz part alone is diagonal in the Sz basis
        assert np.array_equal(Hzz, np.diag(np.diag(Hzz)))


def test_mpo_sum_matvec_equals_single_mpo(oracle_lib):
    terms = C.heisenberg_chain_split(20, 9, 32, seed=7)
    full = C.model_inputs([mpo.heisenberg_chain_W()] * 20, 9, 32, seed=7)
    psi = full.psi.numpy()
    assert np.array_equal(psi, terms[0].psi.numpy())
    a = oracle_lib.heff_apply_sum([t.numpy()[:4] for t in terms], psi)
    b = oracle_lib.heff_apply(*full.numpy()[:4], psi)
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)


def test_mpo_sum_lanczos_ed(oracle_lib):
    terms = C.heisenberg_chain_split(10, 4, 16, seed=8)     # full rank, mL = mR = 16
    tt = [t.numpy()[:4] for t in terms]
    psi = terms[0].psi.numpy()
    r = oracle_lib.lanczos(lambda v: oracle_lib.heff_apply_sum(tt, v.reshape(psi.shape)).ravel(), psi, 300,
                           tol=1e-10, converge=True)
    e0 = np.linalg.eigvalsh(ed_ref.heisenberg(10, ed_ref.chain_bonds(10)).toarray())[0]
    assert abs(r.energy - e0) <= 1e-10


def test_penalty_gives_first_excited_level(oracle_lib):
    """SPEC.md:783 example: with the ground state penalised, the local solver finds the first
    excited ED level of the N = 8 chain (full-rank environments)."""
    x = C.make("c1_n8")
    L, W1, W2, R, psi = x.numpy()
    H = oracle_lib.heff_dense(L, W1, W2, R)
    ev, vec = np.linalg.eigh(0.5 * (H + H.T))
    phi0 = vec[:, 0].reshape(psi.shape)
    w = 10.0
    r = oracle_lib.lanczos(lambda v: oracle_lib.heff_apply_penalty(L, W1, W2, R, v.reshape(psi.shape), [phi0], w).ravel(),
                           psi, 300, tol=1e-10, converge=True)
    ed = np.linalg.eigvalsh(ed_ref.heisenberg(8, ed_ref.chain_bonds(8)).toarray())
    assert ed[1] - ed[0] > 1e-3
    assert abs(r.energy - ed[1]) <= 1e-10
    # the penalised operator is the plain one plus a rank-1 term
    rng = np.random.default_rng(0)
    v = rng.standard_normal(psi.shape)
    lhs = oracle_lib.heff_apply_penalty(L, W1, W2, R, v, [phi0], w)
    rhs = (H @ v.ravel() + w * phi0.ravel() * np.dot(phi0.ravel(), v.ravel())).reshape(psi.shape)
    np.testing.assert_allclose(lhs, rhs, atol=1e-12)
