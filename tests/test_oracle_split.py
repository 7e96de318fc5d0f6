"""Pins of the two-site split oracle (oracle/split.py) against values
the paper and the mathematics fix.  Each pin has an independent side: a closed form (the
singlet, a product state), exact diagonalisation (Schmidt coefficients squared are the
eigenvalues of the partial-trace reduced density matrix of the ED ground state; SU(2)
multiplets), a brute-force scan of every cut point, or an identity of
exact arithmetic (Eckart-Young).  CPU only.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from heffgen import configs as C
from oracle import split as osplit
from tests import ed_ref

GOLD = json.loads((Path(__file__).parent / "golden" / "closed_forms.json").read_text())


def _ed_ground(N, bonds=None):
    H = ed_ref.heisenberg(N, bonds if bonds is not None else ed_ref.chain_bonds(N))
    if N <= 8:
        w, v = np.linalg.eigh(H.toarray())
        return w[0], v[:, 0]
    w, v = spla.eigsh(H, k=1, which="SA", tol=1e-14, v0=np.ones(H.shape[0]))
    return w[0], v[:, 0]


def _reduced_density_spectrum(psi, nleft, N):
    """Eigenvalues (descending) of rho_A = Tr_B |psi><psi| for A = sites 0..nleft-1, by an
    explicit partial trace over B's basis states (site 0 most significant)."""
    dA, dB = 2 ** nleft, 2 ** (N - nleft)
    rho = np.zeros((dA, dA))
    for j in range(dB):                       # Tr_B: sum over B basis states
        col = psi[j::dB]                      # amplitudes <i_A, j_B | psi> for all i_A
        rho += np.outer(col, col)
    return np.sort(np.linalg.eigvalsh(rho))[::-1]


# ---------------------------------------------------------------- closed forms
def test_singlet_schmidt_values_closed_form():
    """N = 2 ground state of Eq. (1) is the singlet (|ud> - |du>)/sqrt 2: two Schmidt values
    1/sqrt 2; keeping one leaves truncation error exactly 1/2."""
    E, psi = _ed_ground(2)
    assert E == pytest.approx(GOLD["two_site_singlet_energy"]["value"], abs=1e-14)
    sp = osplit.svd_split(psi.reshape(2, 2))
    np.testing.assert_allclose(sp.S, [GOLD["singlet_schmidt_value"]["value"]] * 2, atol=1e-15)
    assert sp.n == 2 and sp.trunc_err == pytest.approx(0.0, abs=1e-30)
    t = osplit.svd_split(psi.reshape(2, 2), maxdim=1)
    assert t.n == 1 and t.trunc_err == pytest.approx(0.5, abs=1e-15)


def test_product_state_has_one_singular_value():
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(24), rng.standard_normal(40)
    sp = osplit.svd_split(np.outer(x, y))
    assert sp.S[0] == pytest.approx(np.linalg.norm(x) * np.linalg.norm(y), rel=1e-14)
    assert np.all(sp.S[1:] <= 1e-14 * sp.S[0])
    assert sp.n == 1                                  # numerical zeros are never kept (R21)
    for d in (0, 1):
        s = osplit.svd_split(np.outer(x, y), direction=d)
        np.testing.assert_allclose(s.Q @ s.C if d == 0 else s.C @ s.Q, np.outer(x, y), atol=1e-13)


# ---------------------------------------------------------------- ED: Schmidt spectra
@pytest.mark.parametrize("N,nleft", [(8, 4), (8, 3), (10, 5), (10, 2)])
def test_schmidt_values_equal_reduced_density_matrix_spectrum(N, nleft):
    E, psi = _ed_ground(N)
    lam = _reduced_density_spectrum(psi, nleft, N)
    sp = osplit.svd_split(psi.reshape(2 ** nleft, 2 ** (N - nleft)))
    np.testing.assert_allclose(sp.S ** 2, lam[: sp.S.size], atol=1e-13)
    assert np.sum(sp.S ** 2) == pytest.approx(1.0, abs=1e-13)


@pytest.mark.parametrize("N", [8, 10])
def test_schmidt_spectrum_su2_multiplets(N):
    """The open-chain ground state is an SU(2) singlet, so each half's reduced density
    matrix commutes with the half's total spin: eigenvalues come in multiplets of size
    2S+1 -- odd for a half of N/2 = 4 sites (integer S), even for 5 sites (half-integer S)."""
    E, psi = _ed_ground(N)
    h = N // 2
    s2 = osplit.svd_split(psi.reshape(2 ** h, 2 ** h)).S ** 2
    s2 = s2[s2 > 1e-9]
    groups, i = [], 0
    while i < s2.size:
        j = i
        while j + 1 < s2.size and abs(s2[j + 1] - s2[i]) <= 1e-9 * max(1.0, s2[i]) + 1e-12:
            j += 1
        groups.append(j - i + 1)
        i = j + 1
    assert all(g % 2 == (h % 2 == 0) for g in groups), groups
    assert groups[0] == (1 if h % 2 == 0 else 2)      # singlet / doublet on top


def test_two_site_dmrg_state_schmidt_values_match_ed():
    """C1 (N = 10 chain, window (4,5), full-rank orthonormal blocks): the converged H_eff
    ground state, split at the window's centre bond, has the ED ground state's Schmidt
    values across sites 0..4 | 5..9 (the block maps are orthogonal at full rank)."""
    from oracle import oracle
    x = C.make("c1")
    L, W1, W2, R, psi0 = x.numpy()
    res = oracle.lanczos_heff(L, W1, W2, R, psi0, max_iter=200, tol=1e-12, converge=True)
    E, psi_ed = _ed_ground(10)
    assert res.energy == pytest.approx(E, abs=1e-10)
    sp = osplit.svd_split(osplit.psi_matrix(res.x.reshape(psi0.shape)))
    lam = _reduced_density_spectrum(psi_ed, 5, 10)
    np.testing.assert_allclose(sp.S ** 2, lam, atol=1e-9)


# ---------------------------------------------------------------- truncation rule
def _brute_kept(s, cutoff, maxdim, mindim):
    """Scan every cut point n = 1..len(s); the smallest with relative discarded weight within
    cutoff, then mindim / maxdim / numerical rank (reading R21)."""
    p = s ** 2
    tot = p.sum()
    rank = int(np.sum(s > osplit.RANK_EPS * s[0]))
    ok = [n for n in range(1, s.size + 1) if p[n:].sum() <= cutoff * tot]
    n = min(ok[0], rank)
    n = max(n, min(mindim, rank))
    return min(n, maxdim) if maxdim > 0 else n


def test_truncate_spectrum_examples():
    assert osplit.truncate_spectrum(np.array([1.0, 0, 0, 0])) == (1, 0.0)
    n, e = osplit.truncate_spectrum(np.array([1.0, 1, 1, 1]) / 2, maxdim=2)
    assert n == 2 and e == pytest.approx(0.5)
    n, e = osplit.truncate_spectrum(np.array([1.0, 1e-3, 1e-5]), cutoff=1e-8)
    assert n == 2 and e == pytest.approx(1e-10 / (1 + 1e-6 + 1e-10))
    n, _ = osplit.truncate_spectrum(np.array([1.0, 1e-3, 1e-5]), cutoff=1e-8, mindim=3)
    assert n == 3
    with pytest.raises(ValueError):
        osplit.truncate_spectrum(np.array([1.0]), cutoff=-1.0)
    with pytest.raises(ValueError):
        osplit.truncate_spectrum(np.array([]))


def test_truncate_spectrum_matches_brute_force_scan():
    rng = np.random.default_rng(11)
    for trial in range(300):
        n = int(rng.integers(1, 40))
        s = np.sort(np.exp(rng.uniform(-30, 0, n)))[::-1]
        if rng.random() < 0.2:
            s[rng.integers(0, n):] = 0.0 if s.size > 1 else s[0]
            s[0] = max(s[0], 1e-3)
            s = np.sort(s)[::-1]
        cutoff = float(10 ** rng.uniform(-16, -1)) if rng.random() < 0.9 else 0.0
        maxdim = int(rng.integers(0, n + 3))
        mindim = int(rng.integers(1, n + 2))
        k, err = osplit.truncate_spectrum(s, cutoff, maxdim, mindim)
        assert k == _brute_kept(s, cutoff, maxdim, mindim), (trial, s, cutoff, maxdim, mindim)
        assert err == pytest.approx((s[k:] ** 2).sum() / (s ** 2).sum(), rel=1e-12, abs=0)


# ---------------------------------------------------------------- factor identities
@pytest.mark.parametrize("shape", [(37, 23), (23, 37), (32, 32)])
@pytest.mark.parametrize("direction", [0, 1])
def test_untruncated_split_reconstructs_and_is_isometric(shape, direction):
    rng = np.random.default_rng(sum(shape) + direction)
    Psi = rng.standard_normal(shape)
    sp = osplit.svd_split(Psi, direction=direction)
    n = min(shape)
    assert sp.n == n
    rec = sp.Q @ sp.C if direction == 0 else sp.C @ sp.Q
    np.testing.assert_allclose(rec, Psi, atol=1e-13 * np.abs(Psi).max())
    G = sp.Q.T @ sp.Q if direction == 0 else sp.Q @ sp.Q.T
    np.testing.assert_allclose(G, np.eye(n), atol=1e-14)
    # the centre carries the singular values: rows (dir 0) / columns (dir 1) orthogonal with norms s
    CC = sp.C @ sp.C.T if direction == 0 else sp.C.T @ sp.C
    np.testing.assert_allclose(CC, np.diag(sp.S[:n] ** 2), atol=1e-13 * sp.S[0] ** 2)


@pytest.mark.parametrize("direction", [0, 1])
def test_eckart_young_discarded_weight(direction):
    """||Psi - truncated||_F^2 = sum of discarded s^2 (Eckart-Young-Mirsky)."""
    rng = np.random.default_rng(5)
    Psi = rng.standard_normal((48, 40)) * np.exp(-np.arange(40) / 6.0)[None, :]
    Psi /= np.linalg.norm(Psi)
    sp = osplit.svd_split(Psi, cutoff=1e-6, maxdim=30, direction=direction)
    rec = sp.Q @ sp.C if direction == 0 else sp.C @ sp.Q
    assert np.linalg.norm(Psi - rec) ** 2 == pytest.approx(sp.trunc_err, rel=1e-8, abs=1e-28)
    assert sp.trunc_err <= 1e-6 or sp.n == 30


def test_directions_agree_and_gauge():
    rng = np.random.default_rng(9)
    Psi = rng.standard_normal((30, 26))
    a = osplit.svd_split(Psi, maxdim=12, direction=0)
    b = osplit.svd_split(Psi, maxdim=12, direction=1)
    np.testing.assert_allclose(a.Q @ a.C, b.C @ b.Q, atol=1e-13)
    np.testing.assert_array_equal(a.S, b.S)
    for vecs in (a.Q.T, b.Q):                          # largest-|.| entry positive (R22)
        idx = np.argmax(np.abs(vecs), axis=1)
        assert np.all(vecs[np.arange(vecs.shape[0]), idx] > 0)
    assert math.isclose(a.trunc_err, b.trunc_err)


def test_zero_matrix_is_an_error():
    with pytest.raises(ValueError):
        osplit.svd_split(np.zeros((4, 4)))


# ---------------------------------------------------------------- U(1) block split (NEXT-2 x NEXT-3)
def _qn_psi(N=10, seed=3):
    """Sz = 0 ground state of the N-site chain as a two-site matrix with its charges."""
    E, psi = _ed_ground(N)
    h = N // 2
    sz = lambda n: np.array([sum(1 if (i >> (n - 1 - b)) & 1 == 0 else -1 for b in range(n)) for i in range(2 ** n)])
    qr, qc = sz(h), -sz(N - h)                               # q(left half) + q(right half) = 0
    Psi = psi.reshape(2 ** h, 2 ** h) * (qr[:, None] == qc[None, :])   # drop eigsh's out-of-sector noise
    return Psi / np.linalg.norm(Psi), qr, qc


def test_qn_split_equals_dense_split():
    """The block split of a charge-block-diagonal Psi has the dense split's spectrum, kept
    count, truncation error and truncated approximation (a block-diagonal matrix's SVD is
    the union of its blocks' SVDs)."""
    Psi, qr, qc = _qn_psi()
    for kw in (dict(), dict(maxdim=17), dict(cutoff=1e-6), dict(cutoff=1e-3, maxdim=30)):
        for d in (0, 1):
            a = osplit.svd_split_qn(Psi, qr, qc, direction=d, **kw)
            b = osplit.svd_split(Psi, direction=d, **kw)
            np.testing.assert_allclose(a.S, b.S, atol=1e-14)
            assert a.n == b.n and a.trunc_err == pytest.approx(b.trunc_err, abs=1e-15)
            ra = a.Q @ a.C if d == 0 else a.C @ a.Q
            rb = b.Q @ b.C if d == 0 else b.C @ b.Q
            s = b.S
            if a.n == s.size or s[a.n - 1] - s[a.n] > 1e-8:
                np.testing.assert_allclose(ra, rb, atol=1e-12)


def test_qn_split_charge_conservation_and_order():
    Psi, qr, qc = _qn_psi()
    for d in (0, 1):
        sp = osplit.svd_split_qn(Psi, qr, qc, maxdim=40, direction=d)
        assert np.all(np.diff(sp.qk) >= 0)                       # sector-sorted new bond
        for k in range(sp.n):
            u = sp.Q[:, k] if d == 0 else sp.C[:, k]
            v = sp.C[k, :] if d == 0 else sp.Q[k, :]
            assert np.all(u[qr != sp.qk[k]] == 0.0) and np.all(v[qc != sp.qk[k]] == 0.0)
        for c in set(sp.qk.tolist()):                            # descending inside a sector
            assert np.all(np.diff(sp.Sk[sp.qk == c]) <= 0)
        G = sp.Q.T @ sp.Q if d == 0 else sp.Q @ sp.Q.T
        np.testing.assert_allclose(G, np.eye(sp.n), atol=1e-13)


def test_qn_split_spin_flip_symmetry():
    """The Sz = 0 ground state is spin-flip symmetric: the Schmidt values of the left half's
    sectors Sz and -Sz coincide."""
    Psi, qr, qc = _qn_psi()
    sp = osplit.svd_split_qn(Psi, qr, qc)
    for c in set(sp.qk.tolist()):
        if c > 0:
            np.testing.assert_allclose(np.sort(sp.Sk[sp.qk == c]), np.sort(sp.Sk[sp.qk == -c]), atol=1e-12)


def test_qn_split_rejects_charge_violations():
    Psi, qr, qc = _qn_psi()
    bad = Psi.copy()
    i, j = np.nonzero(qr[:, None] != qc[None, :])
    bad[i[0], j[0]] = 1.0
    with pytest.raises(ValueError):
        osplit.svd_split_qn(bad, qr, qc)
