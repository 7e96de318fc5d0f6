"""GPU parity of the two-site split (heff_svd_split) against the
oracle (oracle/split.py) on the same seeded inputs.

Compared element by element: the full singular spectrum (|ds| <= 1e-12 ||Psi||_F, the
backward-error bound of the Jacobi rotations, R23), the kept
count and truncation error, the truncated approximation U.C (unique whenever s_n > s_{n+1}),
and -- where the kept singular values are separated -- Q and C themselves (gauge fixed by
reading R22).  Degenerate spectra (the Heisenberg ground state's SU(2) multiplets) are
compared through the spectrum and U.C only.  At the C4 size the checks are the
properties that define the truncated SVD at any size.
"""
import numpy as np
import pytest
import torch

from heffgen import configs as C
from oracle import split as osplit

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _gpu():
    from paper_2007_14822_b200 import heff
    return heff


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def _graded(M, N, seed, decades=12.0):
    """Psi = U diag(s) V^T with random orthonormal U, V and s spanning `decades` decades."""
    return C.graded_matrix(M, N, seed, decades)


def _compare(Psi, cutoff=0.0, maxdim=0, mindim=1, direction=0, vectors=True):
    heff = _gpu()
    ref = osplit.svd_split(Psi, cutoff, maxdim, mindim, direction)
    got = heff.svd_split(torch.from_numpy(Psi).to(DEV), cutoff, maxdim, mindim, direction)
    torch.cuda.synchronize()
    s1 = ref.S[0]
    fro = float(np.linalg.norm(ref.S))
    S = got.S.cpu().numpy()
    np.testing.assert_allclose(S, ref.S, rtol=0, atol=1e-12 * fro)
    assert got.n == ref.n, (got.n, ref.n)
    assert got.trunc_err == pytest.approx(ref.trunc_err, rel=1e-9, abs=1e-14)
    Q, Cc = got.Q.cpu().numpy(), got.C.cpu().numpy()
    approx = Q @ Cc if direction == 0 else Cc @ Q
    approx_ref = ref.Q @ ref.C if direction == 0 else ref.C @ ref.Q
    n = ref.n
    gap_ok = n == S.size or ref.S[n - 1] - ref.S[n] > 1e-6 * s1
    if gap_ok:
        np.testing.assert_allclose(approx, approx_ref, rtol=0, atol=1e-11 * fro)
    G = Q.T @ Q if direction == 0 else Q @ Q.T
    np.testing.assert_allclose(G, np.eye(n), atol=1e-12)
    if vectors:
        kept = ref.S[: n + 1] if n < ref.S.size else np.append(ref.S[:n], 0.0)
        sep = np.min(np.abs(np.diff(kept))) / s1 if n > 0 else 1.0
        if sep > 1e-5:
            np.testing.assert_allclose(Q, ref.Q, rtol=0, atol=1e-12 * (fro / s1) / sep)
            np.testing.assert_allclose(Cc, ref.C, rtol=0, atol=1e-12 * fro / sep)
    return got, ref


# auto: one-CTA kernel for sides <= 48; block: HEFF_SVD_NO_SMALL forces the block path;
# small: HEFF_SVD_SMALL_N = 128 sends every side <= 128 to the one-CTA kernel (its full capacity)
PATHS = ["auto", "block", "small"]


def _path(monkeypatch, path):
    if path == "block":
        monkeypatch.setenv("HEFF_SVD_NO_SMALL", "1")
    else:
        monkeypatch.delenv("HEFF_SVD_NO_SMALL", raising=False)
    if path == "small":
        monkeypatch.setenv("HEFF_SVD_SMALL_N", "128")
    else:
        monkeypatch.delenv("HEFF_SVD_SMALL_N", raising=False)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("shape", [(32, 32), (37, 23), (23, 37), (1, 5), (5, 1), (3, 3), (96, 96), (100, 300),
                                   (130, 64)])
def test_split_small_shapes(shape, direction, path, monkeypatch):
    _path(monkeypatch, path)
    _compare(_rand(shape, 17 + sum(shape)), direction=direction)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("trunc", [dict(cutoff=1e-8), dict(maxdim=10), dict(cutoff=1e-6, maxdim=40),
                                   dict(cutoff=1e-3, mindim=30), dict(cutoff=0.5)])
def test_split_truncation(trunc, direction, path, monkeypatch):
    _path(monkeypatch, path)
    _compare(_graded(96, 80, 5, decades=10.0), direction=direction, **trunc)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("direction", [0, 1])
def test_split_c1_ground_state_degenerate_spectrum(direction, path, monkeypatch):
    _path(monkeypatch, path)
    """C1's converged two-site ground state: SU(2) multiplets, so compare the spectrum and
    the truncated approximation (cut between multiplets) -- not the vectors."""
    from oracle import oracle
    x = C.make("c1")
    L, W1, W2, R, psi0 = x.numpy()
    res = oracle.lanczos_heff(L, W1, W2, R, psi0, max_iter=200, tol=1e-12, converge=True)
    Psi = osplit.psi_matrix(res.x.reshape(psi0.shape))
    s = osplit.svd_split(Psi).S
    # a cut between two multiplets: the first n with a relative gap > 1e-6
    n = next(i for i in range(8, s.size) if s[i - 1] - s[i] > 1e-6)
    _compare(Psi, maxdim=n, direction=direction, vectors=False)


@pytest.mark.parametrize("name,seed", [("c2", 1003), ("c3", 1004)])
def test_split_config_sizes(name, seed):
    m = {"c2": 256, "c3": 1024}[name]
    Psi = C.random_psi(seed, (m * 2, 2 * m)).numpy()
    _compare(Psi, direction=0, vectors=False)
    _compare(Psi, maxdim=m, direction=1, vectors=False)


def test_split_graded_c2_size_vectors():
    Psi = _graded(512, 512, 21, decades=8.0)
    _compare(Psi, cutoff=1e-12, direction=0)


def test_split_deterministic():
    heff = _gpu()
    Psi = torch.from_numpy(_rand((300, 260), 4)).to(DEV)
    a = heff.svd_split(Psi, maxdim=100)
    b = heff.svd_split(Psi, maxdim=100)
    torch.cuda.synchronize()
    assert torch.equal(a.Q, b.Q) and torch.equal(a.C, b.C) and torch.equal(a.S, b.S)


@pytest.mark.parametrize("path", PATHS)
def test_split_errors(path, monkeypatch):
    _path(monkeypatch, path)
    heff = _gpu()
    bad = torch.ones((8, 8), dtype=torch.float64, device=DEV)
    bad[3, 4] = float("nan")
    with pytest.raises(heff.HeffError):
        heff.svd_split(bad)
    with pytest.raises(heff.HeffZeroVector):
        heff.svd_split(torch.zeros((8, 8), dtype=torch.float64, device=DEV))
    with pytest.raises(heff.HeffError):
        heff.svd_split(torch.ones((8, 8), dtype=torch.float64, device=DEV), cutoff=-1.0)


def test_split_rank_one_product_state():
    x, y = _rand(40, 1), _rand(24, 2)
    got, ref = _compare(np.outer(x, y), direction=0)
    assert got.n == 1


def test_split_c4_size_properties():
    """Full C4 size (Psi 8192 x 8192, the bench workload), maxdim = m = 4096: the outputs
    satisfy the defining properties of the truncated SVD (checked in fp64 on the GPU)."""
    heff = _gpu()
    m = 4096
    psi = C.random_psi(1005, (m, 2, 2, m), DEV)
    got = heff.svd_split(psi, maxdim=m, direction=0)
    Psi = psi.view(2 * m, 2 * m)
    U, Cc, S = got.Q, got.C, got.S
    assert got.n == m
    assert torch.all(S[1:] <= S[:-1])
    I = U.T @ U
    assert (I - torch.eye(m, dtype=torch.float64, device=DEV)).abs().max().item() < 1e-12
    CC = Cc @ Cc.T                                               # = diag(s^2)
    fro = torch.linalg.norm(Psi).item()
    # |d(s^2)| <= 2 s_1 |ds|, |ds| <= 1e-12 ||Psi||_F (R23)
    assert (CC - torch.diag(S[:m] ** 2)).abs().max().item() < 2e-12 * S[0].item() * fro
    resid2 = torch.linalg.norm(Psi - U @ Cc).item() ** 2         # Eckart-Young
    tot = (S ** 2).sum().item()
    assert resid2 == pytest.approx(got.trunc_err * tot, rel=1e-8)
    # sum_i s_i^2 = ||Psi||_F^2: n values each within 1e-12 ||Psi||_F (R23) -> 2 sqrt(n) 1e-12
    assert tot == pytest.approx(torch.linalg.norm(Psi).item() ** 2, rel=2e-12 * (2 * m) ** 0.5)


@pytest.mark.parametrize("direction", [0, 1])
def test_split_identity_and_orthogonal_inputs(direction):
    """Psi = I (all singular values 1, already orthogonal columns) and a random orthogonal
    Psi: every s_i = 1, U.C reconstructs Psi; truncating to 10 keeps error 1 - 10/n."""
    heff = _gpu()
    n = 96
    for Psi in (np.eye(n), np.linalg.qr(_rand((n, n), 8))[0]):
        got = heff.svd_split(torch.from_numpy(Psi).to(DEV), direction=direction)
        np.testing.assert_allclose(got.S.cpu().numpy(), np.ones(n), atol=1e-13)
        Q, Cc = got.Q.cpu().numpy(), got.C.cpu().numpy()
        np.testing.assert_allclose(Q @ Cc if direction == 0 else Cc @ Q, Psi, atol=1e-13)
        t = heff.svd_split(torch.from_numpy(Psi).to(DEV), maxdim=10, direction=direction)
        assert t.n == 10 and t.trunc_err == pytest.approx(1 - 10 / n, rel=1e-12)


@pytest.mark.parametrize("direction", [0, 1])
def test_split_rank_deficient(direction):
    """rank-3 Psi (64 x 80): three singular values, the rest numerical zeros never kept (R21)."""
    rng = np.random.default_rng(12)
    Psi = rng.standard_normal((64, 3)) @ rng.standard_normal((3, 80))
    got, ref = _compare(Psi, direction=direction)
    assert got.n == 3


@pytest.mark.parametrize("scale", [1e-150, 1e150])
def test_split_scale_invariance(scale):
    """The Jacobi tolerances are relative: Psi * 1e-150 and Psi * 1e150 give the scaled spectrum
    and the same singular vectors (no underflow/overflow in the Gram products)."""
    heff = _gpu()
    Psi = _graded(80, 64, 3, decades=6.0)
    a = heff.svd_split(torch.from_numpy(Psi).to(DEV), maxdim=20)
    b = heff.svd_split(torch.from_numpy(Psi * scale).to(DEV), maxdim=20)
    np.testing.assert_allclose(b.S.cpu().numpy() / scale, a.S.cpu().numpy(), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(b.Q.cpu().numpy(), a.Q.cpu().numpy(), atol=1e-10)
    assert a.n == b.n


@pytest.mark.parametrize("shape", [(1, 300), (300, 1), (2, 700), (700, 3)])
@pytest.mark.parametrize("direction", [0, 1])
def test_split_extreme_aspect(shape, direction):
    _compare(_rand(shape, 41 + shape[0]), direction=direction)
