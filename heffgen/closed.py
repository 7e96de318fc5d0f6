"""Inputs whose H_eff.psi has a closed form at ANY size (full-size pins of the oracle and
full-output checks of the CUDA path; the closed form itself lives in the tests).

Seeded-input module: it builds inputs only and holds none of the H_eff / Lanczos
arithmetic.  The MPO is a k = 2 finite-state machine (channel 1 = start, 0 = done, as in
heffgen.mpo) of one arbitrary (non-symmetric) single-site operator per site,
    W[1,:,:,1] = I,  W[1,:,:,0] = O,  W[0,:,:,0] = I,
the left environment has the identity in its start channel and a weighted permutation in
its done channel, L[a',1,a] = delta(a',a), L[a',0,a] = eL[a] delta(a', pi(a)), and the right
environment the identity in its done channel and a weighted permutation in its start
channel, R[b',0,b] = delta(b',b), R[b',1,b] = eR[b] delta(b', rho(b)).  Summing (D) over the
four FSM paths gives
    out[a',s1',s2',b'] = eL[pi^-1 a'] psi[pi^-1 a', s1', s2', b'] + eR[rho^-1 b'] psi[a', s1', s2', rho^-1 b']
                       + sum_s1 O1[s1',s1] psi[a', s1, s2', b'] + sum_s2 O2[s2',s2] psi[a', s1', s2, b'],
which is what the tests evaluate (meta holds pi, rho, eL, eR, O1, O2).
"""
from __future__ import annotations

import numpy as np
import torch

from .configs import HeffInputs, random_psi


def permuted_diagonal(m: int, d: int, seed: int, device="cpu", mR: int | None = None) -> HeffInputs:
    rng = np.random.default_rng(seed)
    mR = m if mR is None else mR
    pi, rho = rng.permutation(m), rng.permutation(mR)
    eL, eR = rng.standard_normal(m), rng.standard_normal(mR)
    O1, O2 = rng.standard_normal((d, d)), rng.standard_normal((d, d))
    L = np.zeros((m, 2, m))
    L[np.arange(m), 1, np.arange(m)] = 1.0
    L[pi, 0, np.arange(m)] = eL
    R = np.zeros((mR, 2, mR))
    R[np.arange(mR), 0, np.arange(mR)] = 1.0
    R[rho, 1, np.arange(mR)] = eR

    def W(O):
        w = np.zeros((2, d, d, 2))
        w[1, :, :, 1] = np.eye(d)
        w[1, :, :, 0] = O
        w[0, :, :, 0] = np.eye(d)
        return w

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
    psi = random_psi(seed + 1, (m, d, d, mR), device)
    return HeffInputs(t(L), t(W(O1)), t(W(O2)), t(R), psi,
                      dict(model="permuted_diagonal", seed=seed, pi=pi, rho=rho, eL=eL, eR=eR, O1=O1, O2=O2))


def separable(m: int, d: int, seed: int, device="cpu", mR: int | None = None) -> HeffInputs:
    """The Hermitian member of the family: pi = rho = identity, symmetric site operators, so
    H_eff = diag(eL) + O1 + O2 + diag(eR) acting on separate legs and its ground energy is
    min eL + min eig O1 + min eig O2 + min eR, with the product ground state
    e_{argmin eL} x u1 x u2 x e_{argmin eR}.  eL and eR have one value -1 (at a random index)
    and the rest in [0, 1], and the site operators' eigenvalues are >= 0.5 apart, so the
    spectral gap is >= 0.5 and Lanczos converges in tens of steps at any m (full-size pins of
    lanczos_ground).  meta["E0"], meta["x0"] are not stored: the tests derive them."""
    rng = np.random.default_rng(seed)
    mR = m if mR is None else mR

    def levels(n):
        v = rng.uniform(0.0, 1.0, n)
        v[rng.integers(n)] = -1.0
        return v

    def sym(n):
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.cumsum(rng.uniform(0.5, 1.0, n)) - 1.0
        return (q * lam) @ q.T

    eL, eR, O1, O2 = levels(m), levels(mR), sym(d), sym(d)
    L = np.zeros((m, 2, m))
    L[np.arange(m), 1, np.arange(m)] = 1.0
    L[np.arange(m), 0, np.arange(m)] = eL
    R = np.zeros((mR, 2, mR))
    R[np.arange(mR), 0, np.arange(mR)] = 1.0
    R[np.arange(mR), 1, np.arange(mR)] = eR

    def W(O):
        w = np.zeros((2, d, d, 2))
        w[1, :, :, 1] = np.eye(d)
        w[1, :, :, 0] = O
        w[0, :, :, 0] = np.eye(d)
        return w

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
    psi = random_psi(seed + 1, (m, d, d, mR), device)
    return HeffInputs(t(L), t(W(O1)), t(W(O2)), t(R), psi,
                      dict(model="separable", seed=seed, pi=np.arange(m), rho=np.arange(mR), eL=eL, eR=eR, O1=O1,
                           O2=O2))
