"""Pins of the CPU oracle against values the paper and the mathematics fix (SURVEY.md 8(c)
P1-P11).  None of these compares the oracle with itself only: each has an independent
side -- a closed form, exact diagonalisation of a Kronecker-built Hamiltonian, a library
eigen-solver, or brute force of the definition.  CPU only.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from heffgen import configs as C
from heffgen import mpo
from tests import ed_ref

GOLD = json.loads((Path(__file__).parent / "golden" / "closed_forms.json").read_text())


def _np(x):
    return x.numpy()


# ---------------------------------------------------------------- P11: MPO generators
def test_p11_heisenberg_mpo_bond_dim_and_dense():
    W = mpo.heisenberg_chain_W()
    assert W.shape[0] == GOLD["heisenberg_mpo_bond_dim"]["value"]
    l, r = mpo.boundary_vectors(5)
    for N in (2, 3, 4):
        Hm = ed_ref.mpo_dense([W] * N, l, r)
        Hk = ed_ref.heisenberg(N, ed_ref.chain_bonds(N)).toarray()
        assert np.array_equal(Hm, Hk), N                                    # exact: entries 0, +-1/4, 1/2


def test_p11_cylinder_mpo_vs_kronecker():
    Lx = 2
    N = Lx * 6
    Ws = [mpo.cylinder_W(j) for j in range(N)]
    assert Ws[0].shape[0] == 20
    l, r = mpo.boundary_vectors(20)
    H = ed_ref.heisenberg(N, ed_ref.cylinder_bonds(Lx))
    rng = np.random.default_rng(0)
    for _ in range(3):
        x = rng.standard_normal(2 ** N)
        np.testing.assert_allclose(ed_ref.mpo_apply(Ws, l, r, x), H @ x, atol=1e-12)


def test_p11_hubbard_mpo_vs_jordan_wigner():
    N = 4
    W = mpo.hubbard_W()
    l, r = mpo.boundary_vectors(6)
    Hm = ed_ref.mpo_dense([W] * N, l, r)
    Hj = ed_ref.hubbard(N).toarray()
    # the JW mode basis orders a site as (n_up n_dn) = (00, 01, 10, 11); the MPO's is (0, up, dn, updn)
    perm1 = np.array([0, 2, 1, 3])
    idx = np.arange(4 ** N).reshape((4,) * N)
    p = idx
    for ax in range(N):
        p = np.take(p, perm1, axis=ax)
    p = p.reshape(-1)
    np.testing.assert_allclose(Hm, Hj[np.ix_(p, p)], atol=1e-13)


def _jw_perm(N):
    """Site basis permutation: the JW mode basis orders a site (n_up n_dn) = (00, 01, 10, 11),
    the MPO's is (0, up, dn, updn)."""
    p = np.arange(4 ** N).reshape((4,) * N)
    for ax in range(N):
        p = np.take(p, np.array([0, 2, 1, 3]), axis=ax)
    return p.reshape(-1)


@pytest.mark.parametrize("width,Lx", [(3, 2), (4, 2), (6, 1)])
def test_p11_hubbard_cylinder_mpo_vs_jordan_wigner(width, Lx):
    """The d = 4, k = 4 width + 2 Hubbard-cylinder MPO (k = 26 at width 6) against the
    Jordan-Wigner Hamiltonian of the same cylinder built from fermionic mode operators
    (column, y-wrap and x hoppings; (6, 1) is the k = 26 generator on one ring)."""
    N = width * Lx
    Ws = [mpo.hubbard_cylinder_W(j, width) for j in range(N)]
    k = Ws[0].shape[0]
    assert k == 4 * width + 2 and Ws[0].shape[1] == 4
    l, r = mpo.boundary_vectors(k)
    H = ed_ref.hubbard(N, bonds=ed_ref.cylinder_bonds(Lx, width))
    p = _jw_perm(N)
    rng = np.random.default_rng(width)
    for _ in range(2):
        x = rng.standard_normal(4 ** N)
        xj = np.zeros_like(x)
        xj[p] = x
        np.testing.assert_allclose(ed_ref.mpo_apply(Ws, l, r, x), (H @ xj)[p], atol=1e-12)


# ---------------------------------------------------------------- P1: N=2, trivial boundary
def test_p1_two_site_trivial_boundary_is_dense_H(oracle_lib):
    x = C.trivial_two_site()
    L, W1, W2, R, psi = x.numpy()
    H = oracle_lib.heff_dense(L, W1, W2, R)
    Hk = ed_ref.heisenberg(2, ed_ref.chain_bonds(2)).toarray()
    assert np.array_equal(H, Hk)
    ev = np.linalg.eigvalsh(H)
    assert ev[0] == GOLD["two_site_singlet_energy"]["value"]
    np.testing.assert_array_equal(ev[1:], [GOLD["two_site_triplet_energy"]["value"]] * 3)


def test_p1_direct_sum_two_site(oracle_lib):
    x = C.trivial_two_site()
    L, W1, W2, R, psi = x.numpy()
    Hk = ed_ref.heisenberg(2, ed_ref.chain_bonds(2)).toarray()
    out = oracle_lib.heff_direct(L, W1, W2, R, psi)
    np.testing.assert_allclose(out.ravel(), Hk @ psi.ravel(), atol=1e-15)


# ---------------------------------------------------------------- P2: ED
def test_p2_closed_form_n4(oracle_lib):
    x = C.heisenberg_chain(4, 1, 4, seed=5)          # full rank: mL = 2, mR = 2
    L, W1, W2, R, psi = x.numpy()
    res = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=200, tol=1e-12, converge=True)
    exact = -(3 + 2 * math.sqrt(3)) / 4
    assert exact == pytest.approx(GOLD["four_site_chain_ground_energy"]["value"], abs=1e-15)
    assert abs(res.energy - exact) <= 1e-10


@pytest.mark.parametrize("name,N", [("c1_n8", 8), ("c1", 10)])
def test_p2_spectrum_equals_ed(oracle_lib, name, N):
    x = C.make(name)
    L, W1, W2, R, psi = x.numpy()
    H = oracle_lib.heff_dense(L, W1, W2, R)
    assert H.shape == (2 ** N, 2 ** N)
    ev = np.linalg.eigvalsh(0.5 * (H + H.T))
    ev_ed = np.linalg.eigvalsh(ed_ref.heisenberg(N, ed_ref.chain_bonds(N)).toarray())
    np.testing.assert_allclose(ev, ev_ed, atol=1e-12)


@pytest.mark.parametrize("name,N", [("c1_n8", 8), ("c1", 10)])
def test_p2_lanczos_converged_equals_ed(oracle_lib, name, N):
    x = C.make(name)
    L, W1, W2, R, psi = x.numpy()
    res = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=300, tol=1e-10, converge=True)
    e0 = spla.eigsh(ed_ref.heisenberg(N, ed_ref.chain_bonds(N)), k=1, which="SA", tol=1e-14)[0][0]
    assert abs(res.energy - e0) <= 1e-10
    # ground vector: residual of the returned Ritz pair
    Hx = oracle_lib.heff_apply(L, W1, W2, R, res.x)
    assert np.linalg.norm(Hx - res.energy * res.x) < 1e-4
    assert abs(np.linalg.norm(res.x) - 1.0) < 1e-13


def test_p2_cylinder_ed(oracle_lib):
    # 2x6 cylinder, full rank around the window (5,6): mL = mR = 32
    Ws = [mpo.cylinder_W(j) for j in range(12)]
    x = C.model_inputs(Ws, 5, 32, seed=11)
    L, W1, W2, R, psi = x.numpy()
    assert L.shape[0] == 32 and R.shape[0] == 32
    res = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=400, tol=1e-10, converge=True)
    e0 = spla.eigsh(ed_ref.heisenberg(12, ed_ref.cylinder_bonds(2)), k=1, which="SA", tol=1e-14)[0][0]
    assert abs(res.energy - e0) <= 1e-10


def test_p2_hubbard_ed(oracle_lib):
    x = C.model_inputs([mpo.hubbard_W()] * 4, 1, 4, seed=12)    # mL = mR = 4, dim 256
    L, W1, W2, R, psi = x.numpy()
    res = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=300, tol=1e-10, converge=True)
    e0 = np.linalg.eigvalsh(ed_ref.hubbard(4).toarray())[0]
    assert abs(res.energy - e0) <= 1e-10


def test_p2_hubbard_cylinder_ed(oracle_lib):
    """Full-rank environments of the 2 x 3 Hubbard cylinder (d = 4, k = 14; window (2,3):
    mL = mR = 16, dim 4096 = 4^6): the oracle's converged Lanczos equals the ground energy of
    the Jordan-Wigner Hamiltonian."""
    width, Lx = 3, 2
    N = width * Lx
    Ws = [mpo.hubbard_cylinder_W(j, width) for j in range(N)]
    x = C.model_inputs(Ws, 2, 16, seed=13)
    L, W1, W2, R, psi = x.numpy()
    assert L.shape[0] * 16 * R.shape[0] == 4 ** N
    res = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=400, tol=1e-10, converge=True)
    e0 = spla.eigsh(ed_ref.hubbard(N, bonds=ed_ref.cylinder_bonds(Lx, width)), k=1, which="SA", tol=1e-14)[0][0]
    assert abs(res.energy - e0) <= 1e-10, (res.energy, e0)


# ---------------------------------------------------------------- P3, P4, P5, P6, P9
def test_p3_identity_channels():
    for x in (C.make("c2", m=64), C.make("c4", m=32), C.make("c5", m=32)):
        L, W1, W2, R, psi = x.numpy()
        k = L.shape[1]
        np.testing.assert_allclose(L[:, k - 1, :], np.eye(L.shape[0]), atol=1e-13)
        np.testing.assert_allclose(R[:, 0, :], np.eye(R.shape[0]), atol=1e-13)


@pytest.mark.parametrize("name,m", [("c2", 64), ("c4", 32), ("c5", 32)])
def test_p4_hermitian(oracle_lib, name, m):
    x = C.make(name, m=m)
    L, W1, W2, R, psi = x.numpy()
    rng = np.random.default_rng(3)
    phi = rng.standard_normal(psi.shape)
    Hpsi = oracle_lib.heff_apply(L, W1, W2, R, psi)
    Hphi = oracle_lib.heff_apply(L, W1, W2, R, phi)
    lhs, rhs = np.vdot(phi, Hpsi), np.vdot(Hphi, psi)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(phi) * np.linalg.norm(Hpsi)


def test_p5_order_invariance(oracle_lib):
    for x in (C.make("c2", m=64), C.make("c5", m=16),
              C.random_dense(dict(mL=5, d1=2, d2=3, mR=7, kL=3, kM=4, kR=2), seed=9)):
        L, W1, W2, R, psi = x.numpy()
        a = oracle_lib.heff_apply(L, W1, W2, R, psi)
        b = oracle_lib.heff_apply_B(L, W1, W2, R, psi)
        assert np.linalg.norm(a - b) <= 1e-14 * np.linalg.norm(a)
        assert abs(np.vdot(psi, a) - np.vdot(psi, b)) <= 1e-14 * np.linalg.norm(a)


def test_p6_direct_sum_equals_four_steps(oracle_lib):
    for dims in (dict(mL=3, d1=2, d2=3, mR=5, kL=2, kM=3, kR=4), dict(mL=4, d1=2, d2=2, mR=3, kL=5, kM=5, kR=5)):
        x = C.random_dense(dims, seed=4)
        L, W1, W2, R, psi = x.numpy()
        a = oracle_lib.heff_direct(L, W1, W2, R, psi)
        b = oracle_lib.heff_apply(L, W1, W2, R, psi)
        c = np.einsum("xwa,wpsu,uqtv,yvb,astb->xpqy", L, W1, W2, R, psi, optimize=False)
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(a)
        assert np.linalg.norm(a - c) <= 1e-13 * np.linalg.norm(a)
    x = C.make("c1")   # m = 16: 1.3e8 terms of the 7-fold sum
    L, W1, W2, R, psi = x.numpy()
    a = oracle_lib.heff_direct(L, W1, W2, R, psi)
    b = oracle_lib.heff_apply(L, W1, W2, R, psi)
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(a)


def test_p9_linearity_and_scaling(oracle_lib):
    x = C.make("c2", m=32)
    L, W1, W2, R, psi = x.numpy()
    rng = np.random.default_rng(8)
    phi = rng.standard_normal(psi.shape)
    H = lambda v: oracle_lib.heff_apply(L, W1, W2, R, v)
    lhs = H(2.5 * psi - 0.75 * phi)
    rhs = 2.5 * H(psi) - 0.75 * H(phi)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)
    np.testing.assert_allclose(oracle_lib.heff_apply(3.0 * L, W1, W2, R, psi), 3.0 * H(psi), rtol=1e-13, atol=1e-15)


def test_row_and_column_ranges(oracle_lib):
    x = C.random_dense(dict(mL=9, d1=2, d2=2, mR=7, kL=3, kM=2, kR=4), seed=2)
    L, W1, W2, R, psi = x.numpy()
    full = oracle_lib.heff_apply(L, W1, W2, R, psi)
    np.testing.assert_array_equal(oracle_lib.heff_apply(L, W1, W2, R, psi, rows=(2, 6)), full[2:6])
    fb = oracle_lib.heff_apply_B(L, W1, W2, R, psi)
    np.testing.assert_array_equal(oracle_lib.heff_apply_B(L, W1, W2, R, psi, cols=(3, 7)), fb[..., 3:7])
    assert oracle_lib.heff_apply(L, W1, W2, R, psi, rows=(4, 4)).shape == (0, 2, 2, 7)


# ---------------------------------------------------------------- P8: variational / interlacing
def test_p8_variational(oracle_lib):
    x = C.heisenberg_chain(10, 4, 4, seed=21)      # truncated: mL = mR = 4 < 16
    L, W1, W2, R, psi = x.numpy()
    res = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=64, tol=1e-12, converge=True)
    e0 = spla.eigsh(ed_ref.heisenberg(10, ed_ref.chain_bonds(10)), k=1, which="SA", tol=1e-14)[0][0]
    assert res.energy >= e0 - 1e-12
    assert np.all(np.diff(res.thetas) <= 1e-12)


# ---------------------------------------------------------------- P10: tridiagonal + SPEC examples
def test_p10_tridiagonal_vs_library(oracle_lib):
    rng = np.random.default_rng(1)
    for j in (1, 2, 3, 7, 40, 200):
        a, b = rng.standard_normal(j), np.abs(rng.standard_normal(j - 1))
        th, y = oracle_lib.tridiag_lowest(a, b)
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        ev, vec = np.linalg.eigh(T)
        assert abs(th - ev[0]) <= 1e-13 * max(1.0, np.abs(ev).max())
        assert abs(abs(np.dot(y, vec[:, 0])) - 1.0) < 1e-10
        assert y[np.argmax(np.abs(y))] > 0
    # a multiple eigenvalue at the bottom (beta = 0 splits T)
    for a, b in (([-1.0, -1.0, 2.0], [0.0, 0.5]), ([-1.0, 3.0, -1.0], [0.0, 0.0])):
        th, y = oracle_lib.tridiag_lowest(a, b)
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        assert abs(th - np.linalg.eigvalsh(T)[0]) < 1e-15
        assert np.linalg.norm(T @ y - th * y) < 1e-12


def test_spec_lanczos_examples(oracle_lib):
    rng = np.random.default_rng(0)
    r = oracle_lib.lanczos(lambda v: v, rng.standard_normal(6), 10)
    assert abs(r.energy - 1.0) < 1e-12 and r.iters == 1
    r = oracle_lib.lanczos(lambda v: np.array([-1.0, 1.0]) * v, rng.standard_normal(2), 10)
    assert abs(r.energy + 1.0) < 1e-12
    A = rng.standard_normal((16, 16)); A = A + A.T
    r = oracle_lib.lanczos(lambda v: A @ v, rng.standard_normal(16), 60, tol=1e-12, converge=True)
    assert abs(r.energy - np.linalg.eigvalsh(A)[0]) < 1e-10
    with pytest.raises(ValueError):
        oracle_lib.lanczos(lambda v: v, np.zeros(4), 5)


def test_lanczos_fixed_steps_count(oracle_lib):
    x = C.make("c2", m=16)
    L, W1, W2, R, psi = x.numpy()
    r = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=20)
    assert r.iters == 20
    assert np.all(np.diff(r.thetas) <= 1e-12)


# ---------------------------------------------------------------- P12: closed form at full size
@pytest.mark.parametrize("m,d,mR", [(4096, 2, 4096), (1024, 4, 768), (37, 3, 53)])
def test_p12_closed_form_full_size(oracle_lib, m, d, mR):
    """heffgen.closed.permuted_diagonal: (D) has a closed form at any size (weighted
    permutations in the environments, one non-symmetric site operator per MPO); the oracle's
    order A (sampled output rows a') and order B (sampled columns b') match it at the C4 size
    (m = 4096, d = 2, psi 537 MB), at d = 4 and at ragged tiny dims -- a size-dependent
    indexing or chunking mistake, a transposed environment (pi vs pi^-1) or a transposed site
    operator would fail."""
    from heffgen import closed
    from tests import closed_form

    x = closed.permuted_diagonal(m, d, seed=12 + m, mR=mR)
    L, W1, W2, R, psi = x.numpy()
    rows = sorted({0, 1, m // 2, m - 2, m - 1})
    for a in rows:
        got = oracle_lib.heff_apply(L, W1, W2, R, psi, rows=(a, a + 1))
        ref = closed_form.expected_rows(x.meta, psi, [a])
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max(), a
    cols = sorted({0, mR // 3, mR - 1})
    for b in cols:
        got = oracle_lib.heff_apply_B(L, W1, W2, R, psi, cols=(b, b + 1))
        ref = closed_form.expected_cols(x.meta, psi, [b])
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max(), b
    if m * d * d * mR <= 10 ** 6:  # tiny: the whole output, and the literal 7-fold sum
        ref = closed_form.expected_rows(x.meta, psi, range(m))
        assert np.abs(oracle_lib.heff_apply(L, W1, W2, R, psi) - ref).max() <= 1e-13 * np.abs(ref).max()
        assert np.abs(oracle_lib.heff_direct(L, W1, W2, R, psi) - ref).max() <= 1e-13 * np.abs(ref).max()


def test_p12_separable_lanczos_closed_form(oracle_lib):
    """The oracle's Lanczos on the Hermitian member of the P12 family reaches the closed-form
    ground energy min eL + min eig O1 + min eig O2 + min eR (no ED involved)."""
    from heffgen import closed

    x = closed.separable(96, 3, seed=7, mR=80)
    L, W1, W2, R, psi = x.numpy()
    mt = x.meta
    E0 = mt["eL"].min() + np.linalg.eigvalsh(mt["O1"])[0] + np.linalg.eigvalsh(mt["O2"])[0] + mt["eR"].min()
    o = oracle_lib.lanczos_heff(L, W1, W2, R, psi, max_iter=120)
    assert abs(o.energy - E0) <= 1e-10 * abs(E0), (o.energy, E0)
