"""Hand-written finite-state-machine MPOs for the three workload models.

Seeded-input module shared by the oracle tests and the CUDA path: it builds inputs
only and holds none of the H_eff / Lanczos arithmetic.

Conventions (readings R2-R6):
  * W[w, s', s, w1] = <s'| O_{w -> w1} |s>: s' is the output (primed) leg, s the input,
    w the left MPO bond, w1 the right one (north_star's W1[w,s1',s1,w1]).
  * channel k-1 = "start" (nothing placed yet), channel 0 = "done" (term complete);
    left boundary vector selects k-1, right boundary selects 0.
"""
from __future__ import annotations

import numpy as np

# ---- S = 1/2: basis (Up, Dn) = (0, 1); operators of Eq. (1)
SZ = np.array([[0.5, 0.0], [0.0, -0.5]])
SP = np.array([[0.0, 1.0], [0.0, 0.0]])   # S+ |Dn> = |Up>
SM = SP.T.copy()
I2 = np.eye(2)


def heisenberg_chain_W() -> np.ndarray:
    """Bulk W of H = sum_i Sz_i Sz_{i+1} + 1/2 S+_i S-_{i+1} + 1/2 S-_i S+_{i+1}  (Eq. 1).

    Bond dimension 5.  Returns shape (5, 2, 2, 5).
    """
    k = 5
    W = np.zeros((k, 2, 2, k))
    start, done = k - 1, 0
    W[start, :, :, start] = I2
    W[done, :, :, done] = I2
    W[start, :, :, 1] = 0.5 * SM
    W[start, :, :, 2] = 0.5 * SP
    W[start, :, :, 3] = SZ
    W[1, :, :, done] = SP
    W[2, :, :, done] = SM
    W[3, :, :, done] = SZ
    return W


def dm_chain_W(D: float = 0.5) -> np.ndarray:
    """Complex Hermitian MPO (k = 5): Eq. (1) plus a Dzyaloshinskii-Moriya term
    D (Sx_i Sy_{i+1} - Sy_i Sx_{i+1}) = (iD/2)(S+_i S-_{i+1} - S-_i S+_{i+1}), i.e. bond
    1/2 (1 + iD) S+_i S-_{i+1} + 1/2 (1 - iD) S-_i S+_{i+1} + Sz_i Sz_{i+1}
    (the NEXT-4 complex workload; reading R19)."""
    k = 5
    W = np.zeros((k, 2, 2, k), dtype=np.complex128)
    start, done = k - 1, 0
    W[start, :, :, start] = I2
    W[done, :, :, done] = I2
    W[start, :, :, 1] = 0.5 * (1 - 1j * D) * SM
    W[start, :, :, 2] = 0.5 * (1 + 1j * D) * SP
    W[start, :, :, 3] = SZ
    W[1, :, :, done] = SP
    W[2, :, :, done] = SM
    W[3, :, :, done] = SZ
    return W


def heisenberg_zz_W() -> np.ndarray:
    """The Sz Sz part of Eq. (1) alone (k = 3): one term of an MPO sum."""
    k = 3
    W = np.zeros((k, 2, 2, k))
    W[2, :, :, 2] = I2
    W[0, :, :, 0] = I2
    W[2, :, :, 1] = SZ
    W[1, :, :, 0] = SZ
    return W


def heisenberg_flip_W() -> np.ndarray:
    """The 1/2 (S+S- + S-S+) part of Eq. (1) alone (k = 4)."""
    k = 4
    W = np.zeros((k, 2, 2, k))
    W[3, :, :, 3] = I2
    W[0, :, :, 0] = I2
    W[3, :, :, 1] = 0.5 * SM
    W[3, :, :, 2] = 0.5 * SP
    W[1, :, :, 0] = SP
    W[2, :, :, 0] = SM
    return W


CYL_WIDTH = 6


def cylinder_bond(i: int, j: int, width: int = CYL_WIDTH) -> float:
    """J1 coupling between snake sites i < j of a width-`width` cylinder (periodic in y, open in x)."""
    t = j - i
    if t == 1:
        return 1.0 if i % width != width - 1 else 0.0           # within a column
    if t == width - 1:
        return 1.0 if i % width == 0 else 0.0                   # the y-wrap bond (y=0, y=width-1)
    if t == width:
        return 1.0                                              # x bond
    return 0.0


def cylinder_W(j: int, width: int = CYL_WIDTH) -> np.ndarray:
    """Per-site W at snake site j of the J1 Heisenberg cylinder (reading R5).

    Channels: done=0, (op, t) = 1 + op*width + (t-1) for op in (S+, S-, Sz), t = 1..width
    sites since the first operator was placed, start = 3*width + 1.  k = 3*width + 2 = 20.
    """
    k = 3 * width + 2
    start, done = k - 1, 0
    ops_open = (SP, SM, SZ)
    ops_close = (0.5 * SM, 0.5 * SP, SZ)
    W = np.zeros((k, 2, 2, k))
    W[start, :, :, start] = I2
    W[done, :, :, done] = I2
    for op in range(3):
        W[start, :, :, 1 + op * width] = ops_open[op]
        for t in range(1, width + 1):
            ch = 1 + op * width + (t - 1)
            if t < width:
                W[ch, :, :, ch + 1] = I2
            J = cylinder_bond(j - t, j, width) if j - t >= 0 else 0.0
            if J != 0.0:
                W[ch, :, :, done] = J * ops_close[op]
    return W


# ---- Hubbard: local basis (0, up, dn, updn) = (0,1,2,3); Jordan-Wigner with up before dn (reading R6)
CUP = np.zeros((4, 4)); CUP[0, 1] = 1.0; CUP[2, 3] = 1.0          # a_up
CDN = np.zeros((4, 4)); CDN[0, 2] = 1.0; CDN[1, 3] = -1.0         # (-1)^{n_up} a_dn
FJW = np.diag([1.0, -1.0, -1.0, 1.0])
NUPDN = np.diag([0.0, 0.0, 0.0, 1.0])
I4 = np.eye(4)


def hubbard_W(t: float = 1.0, U: float = 4.0) -> np.ndarray:
    """Bulk W of H = -t sum_{i,s}(c+_{is} c_{i+1,s} + h.c.) + U sum_i n_{i,up} n_{i,dn}; k = 6.

    The model appears in the paper only as an application; the
    operator string ordering is DESIGN.md reading R6.
    """
    k = 6
    start, done = k - 1, 0
    W = np.zeros((k, 4, 4, k))
    W[start, :, :, start] = I4
    W[done, :, :, done] = I4
    W[start, :, :, done] = U * NUPDN
    # c+_{i s} c_{i+1 s} = (C_s^T F)_i (C_s)_{i+1};  h.c. = (F C_s)_i (C_s^T)_{i+1}
    for n, C in enumerate((CUP, CDN)):
        W[start, :, :, 1 + 2 * n] = C.T @ FJW
        W[1 + 2 * n, :, :, done] = -t * C
        W[start, :, :, 2 + 2 * n] = FJW @ C
        W[2 + 2 * n, :, :, done] = -t * C.T
    return W


def hubbard_cylinder_W(j: int, width: int = CYL_WIDTH, t: float = 1.0, U: float = 4.0) -> np.ndarray:
    """Per-site W at snake site j of the Hubbard model on a width-`width` cylinder (periodic in
    y, open in x, snake i = x*width + y; hopping -t on the J1 bonds of cylinder_bond, on-site
    U n_up n_dn).  Jordan-Wigner as in hubbard_W: c+_i c_j (i < j) = (C^T F)_i F..F (C)_j and
    its h.c. (F C)_i F..F (C^T)_j, so channels passing a site carry the string F.

    Channels: done = 0, (op, t) = 1 + op*width + (t-1) for the four openers
    op = (C_up^T F, F C_up, C_dn^T F, F C_dn) and t = 1..width sites since the opener,
    start = 4*width + 1: k = 4*width + 2 (26 at width 6).  d = 4.  The quasi-2D Hubbard
    workload of the paper's applications; reading R26."""
    k = 4 * width + 2
    start, done = k - 1, 0
    opens = (CUP.T @ FJW, FJW @ CUP, CDN.T @ FJW, FJW @ CDN)
    closes = (CUP, CUP.T, CDN, CDN.T)
    W = np.zeros((k, 4, 4, k))
    W[start, :, :, start] = I4
    W[done, :, :, done] = I4
    W[start, :, :, done] = U * NUPDN
    for op in range(4):
        W[start, :, :, 1 + op * width] = opens[op]
        for tt in range(1, width + 1):
            ch = 1 + op * width + (tt - 1)
            if tt < width:
                W[ch, :, :, ch + 1] = FJW
            J = cylinder_bond(j - tt, j, width) if j - tt >= 0 else 0.0
            if J != 0.0:
                W[ch, :, :, done] = -t * J * closes[op]
    return W


def boundary_vectors(k: int) -> tuple[np.ndarray, np.ndarray]:
    """(left, right) MPO boundary vectors: left selects start = k-1, right selects done = 0."""
    l = np.zeros(k); l[k - 1] = 1.0
    r = np.zeros(k); r[0] = 1.0
    return l, r
