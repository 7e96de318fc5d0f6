"""Dense / sparse Hamiltonians built by Kronecker products, independently of heffgen's MPOs.

Pin infrastructure for tests (exact diagonalisation = the textbook special case of the
local eigenproblem at full bond dimension).  numpy/scipy only.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

SZ = sp.csr_matrix(np.array([[0.5, 0.0], [0.0, -0.5]]))
SP = sp.csr_matrix(np.array([[0.0, 1.0], [0.0, 0.0]]))
SM = sp.csr_matrix(np.array([[0.0, 0.0], [1.0, 0.0]]))


def _site_op(op, i, N, d=2):
    left = sp.identity(d ** i, format="csr")
    right = sp.identity(d ** (N - i - 1), format="csr")
    return sp.kron(sp.kron(left, op, format="csr"), right, format="csr")


def heisenberg(N: int, bonds) -> sp.csr_matrix:
    """H = sum_{(i,j) in bonds} J (Sz Sz + 1/2 S+S- + 1/2 S-S+), site 0 most significant."""
    H = sp.csr_matrix((2 ** N, 2 ** N))
    for i, j, J in bonds:
        H = H + J * (_site_op(SZ, i, N) @ _site_op(SZ, j, N)
                     + 0.5 * _site_op(SP, i, N) @ _site_op(SM, j, N)
                     + 0.5 * _site_op(SM, i, N) @ _site_op(SP, j, N))
    return H.tocsr()


def chain_bonds(N):
    return [(i, i + 1, 1.0) for i in range(N - 1)]


def cylinder_bonds(Lx, Ly=6):
    """J1 bonds of an Lx x Ly cylinder, open in x, periodic in y, sites numbered x*Ly + y."""
    b = []
    for x in range(Lx):
        for y in range(Ly):
            i = x * Ly + y
            b.append((i, x * Ly + (y + 1) % Ly, 1.0))
            if x + 1 < Lx:
                b.append((i, i + Ly, 1.0))
    return [(min(i, j), max(i, j), J) for i, j, J in b]


def hubbard(N: int, t=1.0, U=4.0, bonds=None) -> sp.csr_matrix:
    """Hubbard model on 2N fermionic modes p = 2i + sigma (up=0, dn=1), Jordan-Wigner
    strings over all modes q < p.  Mode basis |n> with n=1 occupied; a = [[0,1],[0,0]].
    bonds: hopping pairs (i, j, J) (default: the open chain, J = 1); hopping -t J."""
    if bonds is None:
        bonds = chain_bonds(N)
    M = 2 * N
    a = sp.csr_matrix(np.array([[0.0, 1.0], [0.0, 0.0]]))
    Z = sp.csr_matrix(np.diag([1.0, -1.0]))
    I = sp.identity(2, format="csr")

    def c(p):
        ops = [Z] * p + [a] + [I] * (M - p - 1)
        out = ops[0]
        for o in ops[1:]:
            out = sp.kron(out, o, format="csr")
        return out

    cs = [c(p) for p in range(M)]
    H = sp.csr_matrix((2 ** M, 2 ** M))
    for i, j, J in bonds:
        for s in range(2):
            p, q = 2 * i + s, 2 * j + s
            hop = cs[p].T @ cs[q]
            H = H - t * J * (hop + hop.T)
    for i in range(N):
        H = H + U * (cs[2 * i].T @ cs[2 * i]) @ (cs[2 * i + 1].T @ cs[2 * i + 1])
    return H.tocsr()


def mpo_dense(Ws, l, r) -> np.ndarray:
    """Densify an MPO chain: H[(s'_0..),(s_0..)] = l . W_0 ... W_{N-1} . r (tiny N only)."""
    d = Ws[0].shape[1]
    H = np.einsum("w,wpsv->psv", l, Ws[0])            # [s',s,w]
    for W in Ws[1:]:
        n = H.shape[0]
        H = np.einsum("abw,wpsv->apbsv", H, W).reshape(n * d, n * d, W.shape[3])
    return np.einsum("abw,w->ab", H, r)


def mpo_apply(Ws, l, r, x) -> np.ndarray:
    """y = H x for the MPO chain, sweeping site by site (no dense H)."""
    N = len(Ws)
    d = Ws[0].shape[1]
    T = np.einsum("w,...->w...", l, x.reshape((d,) * N))
    for j, W in enumerate(Ws):
        # T[w, s0'..s_{j-1}', s_j, ...] -> [w', ..., s_j', ...]
        T = np.tensordot(W, T, axes=([0, 2], [0, 1 + j]))   # [s_j', w', rest...]
        T = np.moveaxis(T, 1, 0)                           # [w', s_j', rest...]
        T = np.moveaxis(T, 1, 1 + j)
    return np.tensordot(r, T, axes=([0], [0])).reshape(-1)
