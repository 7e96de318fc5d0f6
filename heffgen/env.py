"""Seeded random orthonormal MPS blocks and their MPO environments L, R.

Seeded-input module shared by the oracle tests and the CUDA path: it builds inputs
only and holds none of the H_eff / Lanczos arithmetic.  The environment contraction
below is setup (ProjMPO), not the measured path; it runs in torch
fp64 so the m = 4096 / 8192 inputs can be made on the GPU in seconds.

Recipe (reading R7): numpy default_rng(seed) (PCG64) draws every site tensor
in C order from N(0,1) -- left block from the left edge inwards, then right block from
the right edge inwards -- so the draws do not depend on the torch device.  Bond dims
grow as min(d^j, m) from each edge.  Left tensors are left-orthonormalised by thin QR
of A reshaped (a s) x b; right tensors are right-orthonormalised by thin QR of the
transpose of B reshaped a x (s b).
"""
from __future__ import annotations

import numpy as np
import torch


def _qr_left(A: torch.Tensor) -> torch.Tensor:
    mi, d, mo = A.shape
    Q, _ = torch.linalg.qr(A.reshape(mi * d, mo), mode="reduced")
    return Q.reshape(mi, d, mo)


def _qr_right(B: torch.Tensor) -> torch.Tensor:
    """Rows orthonormal: B B^dagger = I (conjugate transpose for complex tensors)."""
    mo, d, mi = B.shape
    Q, _ = torch.linalg.qr(B.reshape(mo, d * mi).conj().T, mode="reduced")
    return Q.conj().T.reshape(mo, d, mi)


def left_bond_dims(nsites: int, d: int, m: int) -> list[int]:
    return [min(d ** j, m) for j in range(nsites + 1)]


def _draw(rng, shape, complex_):
    x = rng.standard_normal(shape)
    if complex_:
        x = x + 1j * rng.standard_normal(shape)
    return x


def draw_left_block(rng: np.random.Generator, nsites: int, d: int, m: int, device, complex_: bool = False):
    dims = left_bond_dims(nsites, d, m)
    out = []
    for j in range(nsites):
        mi, mo = dims[j], min(dims[j + 1], dims[j] * d)
        A = torch.from_numpy(_draw(rng, (mi, d, mo), complex_)).to(device)
        out.append(_qr_left(A))
    return out


def draw_right_block(rng: np.random.Generator, nsites: int, d: int, m: int, device, complex_: bool = False):
    """Right block tensors listed left-to-right; drawn from the right edge inwards."""
    dims = left_bond_dims(nsites, d, m)  # dims counted from the right edge
    rev = []
    for j in range(nsites):
        mi, mo = dims[j], min(dims[j + 1], dims[j] * d)   # mi: bond towards the edge
        B = torch.from_numpy(_draw(rng, (mo, d, mi), complex_)).to(device)
        rev.append(_qr_right(B))
    return rev[::-1]


def grow_left(L: torch.Tensor, A: torch.Tensor, W: torch.Tensor) -> torch.Tensor:
    """L'[a',w',a] = sum conj(A[x',s',a']) L[x',w,x] W[w,s',s,w'] A[x,s,a] (conj: bra side)."""
    mi, k, _ = L.shape
    _, d, mo = A.shape
    k2 = W.shape[3]
    X = (L.reshape(mi * k, mi) @ A.reshape(mi, d * mo)).reshape(mi, k, d, mo)           # [x',w,s,a]
    Y = torch.einsum("xwsa,wpsv->xpva", X, W)                                             # [x',s',w',a]
    return (A.reshape(mi * d, mo).conj().T @ Y.reshape(mi * d, k2 * mo)).reshape(mo, k2, mo)


def grow_right(R: torch.Tensor, B: torch.Tensor, W: torch.Tensor) -> torch.Tensor:
    """R'[b',w,b] = sum conj(B[b',s',y']) R[y',w',y] W[w,s',s,w'] B[b,s,y] (conj: bra side)."""
    mi, k2, _ = R.shape
    mo, d, _ = B.shape
    k = W.shape[0]
    X = (B.reshape(mo * d, mi).conj() @ R.reshape(mi, k2 * mi)).reshape(mo, d, k2, mi)  # [b',s',w',y]
    Y = torch.einsum("bpvy,wpsv->bwsy", X, W)                                             # [b',w,s,y]
    return (Y.reshape(mo * k, d * mi) @ B.reshape(mo, d * mi).T).reshape(mo, k, mo)


def build_left_env(As: list[torch.Tensor], Ws: list[torch.Tensor], k: int, device) -> torch.Tensor:
    L = torch.zeros((1, k, 1), dtype=As[0].dtype if As else torch.float64, device=device)
    L[0, k - 1, 0] = 1.0
    for A, W in zip(As, Ws):
        L = grow_left(L, A, W)
    return L


def build_right_env(Bs: list[torch.Tensor], Ws: list[torch.Tensor], k: int, device) -> torch.Tensor:
    R = torch.zeros((1, k, 1), dtype=Bs[0].dtype if Bs else torch.float64, device=device)
    R[0, 0, 0] = 1.0
    for B, W in zip(reversed(Bs), reversed(Ws)):
        R = grow_right(R, B, W)
    return R
