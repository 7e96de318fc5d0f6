"""Pins for the complex H_eff oracle (NEXT-4 complex; ITensor Dense{ComplexF64}):
the Dzyaloshinskii-Moriya chain is a genuinely complex Hermitian model whose full-rank
H_eff must have the ED spectrum; Hermiticity, real energies, the definition by brute force,
and agreement with the real oracle on real data.  CPU only."""
import numpy as np
import scipy.sparse as sp

from heffgen import configs as C
from heffgen import mpo
from tests import ed_ref


def dm_dense(N, D=0.5):
    H = sp.csr_matrix((2 ** N, 2 ** N), dtype=complex)
    for i in range(N - 1):
        j = i + 1
        H = H + 0.5 * (1 + 1j * D) * (ed_ref._site_op(ed_ref.SP, i, N) @ ed_ref._site_op(ed_ref.SM, j, N)) \
              + 0.5 * (1 - 1j * D) * (ed_ref._site_op(ed_ref.SM, i, N) @ ed_ref._site_op(ed_ref.SP, j, N)) \
              + ed_ref._site_op(ed_ref.SZ, i, N) @ ed_ref._site_op(ed_ref.SZ, j, N)
    return H.toarray()


def test_dm_mpo_is_the_kronecker_hamiltonian():
    l, r = mpo.boundary_vectors(5)
    for N in (2, 3, 4):
        Hm = ed_ref.mpo_dense([mpo.dm_chain_W()] * N, l, r)
        np.testing.assert_allclose(Hm, dm_dense(N), atol=1e-15)
        assert np.abs(Hm.imag).max() > 0.1          # genuinely complex


def test_complex_heff_spectrum_is_ed(oracle_lib):
    x = C.dm_chain(8, 2, 16, seed=3)                # full rank: mL = 4, mR = 16
    L, W1, W2, R, psi = x.numpy()
    n = psi.size
    H = np.zeros((n, n), complex)
    for i in range(n):
        e = np.zeros(n, complex)
        e[i] = 1
        H[:, i] = oracle_lib.heff_apply_z(L, W1, W2, R, e.reshape(psi.shape)).ravel()
    assert np.abs(H - H.conj().T).max() < 1e-13
    np.testing.assert_allclose(np.linalg.eigvalsh(H), np.linalg.eigvalsh(dm_dense(8)), atol=1e-12)
    r = oracle_lib.lanczos_heff_z(L, W1, W2, R, psi, 300, tol=1e-10, converge=True)
    assert abs(r.energy - np.linalg.eigvalsh(dm_dense(8))[0]) <= 1e-10
    # Ritz vector: unit norm, residual small, <x|H|x> real (P7)
    xv = r.x.ravel()
    e = np.vdot(xv, H @ xv)
    assert abs(e.imag) <= 1e-14 * abs(e.real)
    assert abs(np.linalg.norm(xv) - 1) < 1e-13


def test_complex_definition_brute_force_and_real_agreement(oracle_lib):
    rng = np.random.default_rng(0)
    c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    L, W1, W2, R, psi = c(3, 2, 3), c(2, 2, 2, 3), c(3, 3, 3, 4), c(5, 4, 5), c(3, 2, 3, 5)
    ref = np.einsum("xwa,wpsu,uqtv,yvb,astb->xpqy", L, W1, W2, R, psi, optimize=False)
    out = oracle_lib.heff_apply_z(L, W1, W2, R, psi)
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)
    x = C.make("c2", m=16)
    Lr, W1r, W2r, Rr, pr = x.numpy()
    np.testing.assert_allclose(oracle_lib.heff_apply_z(Lr, W1r, W2r, Rr, pr).real,
                               oracle_lib.heff_apply(Lr, W1r, W2r, Rr, pr), atol=1e-14)


def test_complex_hermiticity_truncated(oracle_lib):
    x = C.dm_chain(20, 9, 32, seed=5)
    L, W1, W2, R, psi = x.numpy()
    rng = np.random.default_rng(1)
    phi = rng.standard_normal(psi.shape) + 1j * rng.standard_normal(psi.shape)
    a = np.vdot(phi, oracle_lib.heff_apply_z(L, W1, W2, R, psi))
    b = np.vdot(oracle_lib.heff_apply_z(L, W1, W2, R, phi), psi)
    assert abs(a - b) <= 1e-12 * abs(a)
