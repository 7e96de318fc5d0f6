"""CPU ORACLE for the two-site split: the truncated SVD that follows
every local eigensolve of a two-site DMRG sweep.

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(paper_2007_14822_b200) never imports it, and this module imports nothing from it.

What it computes (citations: lines of /root/reference/PAPER.md, SPEC.md):

* The SVD ``U,S,V = svd(W,(j,i))`` with the row indices named, ``U*S*V ~ W``
  (Sec. 5).  For the two-site wavefunction psi[a,s1,s2,b] the rows are
  (a, s1) and the columns (s2, b): Psi = U S V^T with Psi of shape (mL d1) x (d2 mR).
* "ITensor decompositions do not truncate, though they do always compute the thin
  version"; with cutoff/maxdim "the truncation will be determined by
  summing the squares of the singular values from smallest to largest until the
  truncation error reaches [cutoff] while also ensuring that the maximum number of
  singular values kept is less than or equal to [maxdim]".  SPEC.md
  makes the error relative (Spectrum: sum of discarded s^2 / sum of all s^2)
  and adds mindim.
* The two factors a sweep keeps (Sec. 6.2): moving right (dir = 0) the
  left-orthonormal A = U[(a s1), k] and the next centre C = S V^T [k, (s2 b)]; moving left
  (dir = 1) the right-orthonormal B = V^T[k, (s2 b)] and the centre C = U S [(a s1), k].

Readings (R20-R22): the kept count is the smallest n with
sum_{i>=n} s_i^2 <= cutoff * sum_i s_i^2, then raised to mindim and capped at maxdim; a
singular value s_i <= RANK_EPS * s_1 is a numerical zero and is never kept (mindim is
clamped to the numerical rank); the sign of each kept singular vector pair is fixed so
that the largest-|.| entry of the orthonormal factor's vector (U's column for dir 0, V^T's
row for dir 1; first such entry on ties) is positive.

The SVD itself is LAPACK's (numpy.linalg.svd) -- a library primitive serving as one step;
the truncation rule, gauge and factor assembly are written out below.  Pinned in
tests/test_oracle_split.py against closed forms (singlet, product state), exact
diagonalisation (Schmidt spectra = eigenvalues of partial-trace reduced density matrices)
and a brute-force scan of every cut point.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

RANK_EPS = 1e-12   # reading R21: s_i <= RANK_EPS * s_1 is a numerical zero


@dataclass
class Split:
    Q: np.ndarray        # dir 0: U [M, n]; dir 1: V^T [n, N]  (the orthonormal factor)
    S: np.ndarray        # all min(M, N) singular values, descending
    C: np.ndarray        # dir 0: S V^T [n, N]; dir 1: U S [M, n]  (the next centre)
    n: int               # kept count
    trunc_err: float     # sum_{i>=n} s_i^2 / sum_i s_i^2


def truncate_spectrum(s: np.ndarray, cutoff: float = 0.0, maxdim: int = 0, mindim: int = 1) -> tuple[int, float]:
    """Kept count and relative truncation error for descending singular values s
    ("truncate_spectrum").  maxdim <= 0: unlimited.

    Written as the paper words it: walk from the smallest value upwards, discarding while
    the accumulated discarded square-sum stays within cutoff * total."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        raise ValueError("empty spectrum")
    if cutoff < 0:
        raise ValueError("cutoff < 0")
    if np.any(np.diff(s) > 0) or s[-1] < 0:
        raise ValueError("spectrum must be descending and non-negative")
    p = s * s
    total = float(np.sum(p))
    if total == 0.0:
        raise ValueError("zero spectrum")
    rank = int(np.count_nonzero(s > RANK_EPS * s[0]))
    n = s.size
    discarded = 0.0
    while n > 1 and discarded + p[n - 1] <= cutoff * total:   # discard smallest while within cutoff
        discarded += p[n - 1]
        n -= 1
    n = min(n, rank)                                           # numerical zeros are never kept
    n = max(n, min(mindim, rank))
    if maxdim > 0:
        n = min(n, maxdim)
    err = float(np.sum(p[n:])) / total
    return n, err


def _fix_sign(vecs: np.ndarray) -> np.ndarray:
    """+/-1 per row of vecs so that each row's largest-|.| entry (first on ties) is positive."""
    idx = np.argmax(np.abs(vecs), axis=1)
    return np.where(vecs[np.arange(vecs.shape[0]), idx] < 0, -1.0, 1.0)


def svd_split(psi_mat: np.ndarray, cutoff: float = 0.0, maxdim: int = 0, mindim: int = 1, direction: int = 0) -> Split:
    """Truncated two-site split of Psi [M, N] (rows (a s1), columns (s2 b))."""
    Psi = np.asarray(psi_mat, dtype=np.float64)
    if Psi.ndim != 2 or Psi.size == 0:
        raise ValueError("Psi must be a non-empty matrix")
    U, s, Vt = np.linalg.svd(Psi, full_matrices=False)        # Psi = U diag(s) Vt
    n, err = truncate_spectrum(s, cutoff, maxdim, mindim)
    U, sk, Vt = U[:, :n], s[:n], Vt[:n, :]
    sign = _fix_sign(U.T) if direction == 0 else _fix_sign(Vt)  # gauge (reading R22)
    U = U * sign[None, :]
    Vt = Vt * sign[:, None]
    if direction == 0:
        return Split(Q=U, S=s, C=sk[:, None] * Vt, n=n, trunc_err=err)     # A = U, C = S V^T
    return Split(Q=Vt, S=s, C=U * sk[None, :], n=n, trunc_err=err)         # B = V^T, C = U S


def psi_matrix(psi: np.ndarray) -> np.ndarray:
    """psi[a, s1, s2, b] -> Psi[(a s1), (s2 b)] (row-major reshape; no data movement)."""
    mL, d1, d2, mR = psi.shape
    return np.ascontiguousarray(psi).reshape(mL * d1, d2 * mR)


@dataclass
class SplitQN:
    Q: np.ndarray        # dir 0: U [M, n]; dir 1: V^T [n, N] -- new bond sector-sorted
    S: np.ndarray        # all singular values of all sector blocks, descending, zero-padded to min(M, N)
    Sk: np.ndarray       # kept singular values in new-bond order
    qk: np.ndarray       # charge of each new-bond index (nondecreasing)
    C: np.ndarray        # dir 0: S V^T [n, N]; dir 1: U S [M, n]
    n: int
    trunc_err: float


def svd_split_qn(psi_mat: np.ndarray, qrow, qcol, cutoff: float = 0.0, maxdim: int = 0, mindim: int = 1,
                 direction: int = 0) -> SplitQN:
    """Two-site split of a charge-conserving Psi (U(1), Sec. 7): Psi[r][c]
    is nonzero only if qrow[r] == qcol[c] (the charge carried by the centre bond), so Psi is
    block diagonal over the charge sectors; factorizations of block-sparse ITensors treat
    the nonzero blocks independently.  Every block gets its own
    SVD (numpy/LAPACK, a library step); one truncation (reading R20/R21) runs over the union
    of all blocks' singular values ("independent SVD per flux-sector block,
    single global sorted truncation across sectors"); the new bond index is ordered by
    charge, then by descending singular value within a charge (reading R24), and carries
    the block's charge.  Gauge per vector as in svd_split (R22)."""
    Psi = np.asarray(psi_mat, dtype=np.float64)
    M, N = Psi.shape
    qrow, qcol = np.asarray(qrow), np.asarray(qcol)
    if qrow.shape != (M,) or qcol.shape != (N,):
        raise ValueError("charge arrays must match Psi's shape")
    allowed = qrow[:, None] == qcol[None, :]
    if np.any(Psi[~allowed] != 0.0):
        raise ValueError("Psi has entries outside its charge blocks")
    sectors = sorted(set(qrow.tolist()) & set(qcol.tolist()))
    cand = []        # (value, sector position, index in block)
    blocks = {}
    for si, c in enumerate(sectors):
        rows, cols = np.nonzero(qrow == c)[0], np.nonzero(qcol == c)[0]
        U, s, Vt = np.linalg.svd(Psi[np.ix_(rows, cols)], full_matrices=False)
        blocks[c] = (rows, cols, U, s, Vt)
        cand += [(float(v), si, j) for j, v in enumerate(s)]
    if not cand:
        raise ValueError("no charge sector is present in both rows and columns")
    cand.sort(key=lambda e: (-e[0], e[1], e[2]))
    S = np.zeros(min(M, N))
    S[: len(cand)] = [e[0] for e in cand]
    n, err = truncate_spectrum(S, cutoff, maxdim, mindim)
    kept = sorted(cand[:n], key=lambda e: (e[1], -e[0], e[2]))    # new bond: charge, then value
    Q = np.zeros((M, n)) if direction == 0 else np.zeros((n, N))
    C = np.zeros((n, N)) if direction == 0 else np.zeros((M, n))
    Sk, qk = np.zeros(n), np.zeros(n, dtype=int)
    for k, (v, si, j) in enumerate(kept):
        c = sectors[si]
        rows, cols, U, s, Vt = blocks[c]
        u, vt = U[:, j].copy(), Vt[j, :].copy()
        vec = u if direction == 0 else vt
        if vec[np.argmax(np.abs(vec))] < 0:                          # gauge (R22)
            u, vt = -u, -vt
        Sk[k], qk[k] = s[j], c
        if direction == 0:
            Q[rows, k] = u
            C[k, cols] = s[j] * vt
        else:
            Q[k, cols] = vt
            C[rows, k] = u * s[j]
    return SplitQN(Q=Q, S=S, Sk=Sk, qk=qk, C=C, n=n, trunc_err=err)


def qn_row_col_charges(qa, qs1, qs2, qb):
    """Charges of Psi's rows (a s1) and columns (s2 b) for the U(1) convention of reading R18
    (a bond carries the total charge to its left): qrow = q(a) + q(s1), qcol = q(b) - q(s2)."""
    qa, qs1, qs2, qb = (np.asarray(v) for v in (qa, qs1, qs2, qb))
    return (qa[:, None] + qs1[None, :]).reshape(-1), (qb[None, :] - qs2[:, None]).reshape(-1)
