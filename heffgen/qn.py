"""U(1)-symmetric (Sz-conserving) inputs for the block-sparse H_eff.

Seeded-input module shared by the oracle tests and the CUDA path: it builds inputs only
and holds none of the H_eff / Lanczos arithmetic.

Quantum numbers (Sec. 7; QN with arrows), reading
R18 of DESIGN.md:
  * site charge q(s) = 2 Sz: Up = +1, Dn = -1 (basis order of R3);
  * a bond index carries the total charge of everything to its LEFT; an MPS tensor
    A[a,s,b] may be nonzero only if q(b) = q(a) + q(s);
  * MPO channel charge c(w): W[w,s',s,w1] may be nonzero only if
    q(s') - q(s) = c(w1) - c(w) (start and done channels carry 0);
  * then L[a',w,a] != 0 only if q(a') - q(a) = c(w), R[b',w,b] != 0 only if
    q(b') - q(b) = c(w), and psi[a,s1,s2,b] != 0 only if q(b) = q(a) + q(s1) + q(s2);
    H_eff maps that sector to itself.
Bond indices are sorted by charge so every sector is a contiguous range.  The tensors are
stored dense (zeros outside the allowed blocks); the random MPS blocks are drawn from
numpy default_rng(seed) in a fixed order and QR-orthonormalised per sector.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import env, mpo
from .configs import HeffInputs

SPIN_Q = np.array([1, -1])


def heisenberg_channel_charges() -> np.ndarray:
    # done, after S- (lowers 2Sz by 2), after S+, after Sz, start
    return np.array([0, -2, 2, 0, 0])


def cylinder_channel_charges(width: int = mpo.CYL_WIDTH) -> np.ndarray:
    c = np.zeros(3 * width + 2, dtype=int)
    for op, q in enumerate((2, -2, 0)):          # opened with S+, S-, Sz
        c[1 + op * width: 1 + (op + 1) * width] = q
    return c


def check_mpo_charges(W: np.ndarray, c: np.ndarray, qs: np.ndarray) -> bool:
    k, d, _, k2 = W.shape
    for w in range(k):
        for sp in range(d):
            for s in range(d):
                for w1 in range(k2):
                    if W[w, sp, s, w1] != 0.0 and qs[sp] - qs[s] != c[w1] - c[w]:
                        return False
    return True


def _cap(avail: dict, m: int) -> dict:
    """Sector dims <= avail with total <= m (proportional, largest remainders)."""
    tot = sum(avail.values())
    if tot <= m:
        return dict(avail)
    qs = sorted(avail)
    raw = {q: avail[q] * m / tot for q in qs}
    dims = {q: min(avail[q], int(np.floor(raw[q]))) for q in qs}
    rem = m - sum(dims.values())
    for q in sorted(qs, key=lambda q: -(raw[q] - np.floor(raw[q]))):
        if rem == 0:
            break
        if dims[q] < avail[q]:
            dims[q] += 1
            rem -= 1
    return {q: d for q, d in dims.items() if d > 0}


@dataclass
class Bond:
    charges: np.ndarray  # per index, sorted nondecreasing

    @property
    def dim(self):
        return len(self.charges)


def _bond_from(dims: dict) -> Bond:
    return Bond(np.concatenate([np.full(dims[q], q, dtype=int) for q in sorted(dims)]) if dims else np.zeros(0, int))


def draw_left_block_qn(rng, nsites: int, qs: np.ndarray, m: int, device):
    """Left-orthonormal U(1) site tensors from the trivial left edge (charge 0)."""
    bond = Bond(np.array([0]))
    As = []
    for _ in range(nsites):
        rows = [(a, s) for a in range(bond.dim) for s in range(len(qs))]
        avail = {}
        for a, s in rows:
            q = bond.charges[a] + qs[s]
            avail[q] = avail.get(q, 0) + 1
        new = _bond_from(_cap(avail, m))
        A = np.zeros((bond.dim, len(qs), new.dim))
        for q in sorted(set(new.charges)):
            cols = np.nonzero(new.charges == q)[0]
            rr = [(a, s) for a, s in rows if bond.charges[a] + qs[s] == q]
            blk = rng.standard_normal((len(rr), len(cols)))
            Q, _ = np.linalg.qr(blk)
            for i, (a, s) in enumerate(rr):
                A[a, s, cols] = Q[i]
        As.append(torch.from_numpy(A).to(device))
        bond = new
    return As, bond


def draw_right_block_qn(rng, nsites: int, qs: np.ndarray, m: int, Q: int, device):
    """Right-orthonormal U(1) site tensors from the right edge; returned left-to-right.
    Internally charges count what lies to the RIGHT (r); the bond's left-counted charge is
    Q - r, and the returned bond is sorted by that."""
    r_bond = np.array([0])                 # right edge: nothing to the right
    Bs_rev = []
    for _ in range(nsites):
        cols = [(s, y) for s in range(len(qs)) for y in range(len(r_bond))]
        avail = {}
        for s, y in cols:
            r = r_bond[y] + qs[s]
            avail[r] = avail.get(r, 0) + 1
        dims = _cap(avail, m)
        # order new indices by left-counted charge Q - r ascending = r descending
        new_r = np.concatenate([np.full(dims[r], r, dtype=int) for r in sorted(dims, reverse=True)])
        B = np.zeros((len(new_r), len(qs), len(r_bond)))
        for r in sorted(dims, reverse=True):
            rowsb = np.nonzero(new_r == r)[0]
            cc = [(s, y) for s, y in cols if r_bond[y] + qs[s] == r]
            blk = rng.standard_normal((len(rowsb), len(cc)))
            Qm, _ = np.linalg.qr(blk.T)        # orthonormal rows of the (rows x cc) block
            for j, (s, y) in enumerate(cc):
                B[rowsb, s, y] = Qm[j]
        Bs_rev.append(torch.from_numpy(B).to(device))
        r_bond = new_r
    return Bs_rev[::-1], Bond(Q - r_bond)


@dataclass
class QNInputs:
    x: HeffInputs
    qa: np.ndarray     # [mL]
    qb: np.ndarray     # [mR]
    qs1: np.ndarray
    qs2: np.ndarray
    cL: np.ndarray
    cM: np.ndarray
    cR: np.ndarray

    def mask(self) -> np.ndarray:
        """Allowed entries of psi / out: q(b) = q(a) + q(s1) + q(s2)."""
        return (self.qb[None, None, None, :] ==
                self.qa[:, None, None, None] + self.qs1[None, :, None, None] + self.qs2[None, None, :, None])

    def qn_dict(self) -> dict:
        return dict(qa=self.qa, qb=self.qb, qs1=self.qs1, qs2=self.qs2, cL=self.cL, cM=self.cM, cR=self.cR)


def model_inputs_qn(Ws: list, charges: list, window: int, m: int, seed: int, Q: int = 0, device="cpu") -> QNInputs:
    """U(1) analogue of configs.model_inputs: sector-sorted, block-sparse L, R, psi in the
    total-charge-Q sector.  charges[j] = channel charges of the MPO bond to the right of
    site j (charges[j][w1] for W_j[..., w1]); the left edge channel is the start (0)."""
    N = len(Ws)
    qs = SPIN_Q
    rng = np.random.default_rng(seed)
    As, bl = draw_left_block_qn(rng, window, qs, m, device)
    Bs, br = draw_right_block_qn(rng, N - window - 2, qs, m, Q, device)
    tW = [torch.from_numpy(np.ascontiguousarray(W)).to(device) for W in Ws]
    k = Ws[0].shape[0]
    L = env.build_left_env(As, tW[:window], k, device)
    R = env.build_right_env(Bs, tW[window + 2:], k, device)
    qa, qb = bl.charges, br.charges
    mask = (qb[None, None, None, :] == qa[:, None, None, None] + qs[None, :, None, None] + qs[None, None, :, None])
    psi = np.random.default_rng(seed + 1).standard_normal(mask.shape) * mask
    psi /= np.linalg.norm(psi)
    x = HeffInputs(L.contiguous(), tW[window].contiguous(), tW[window + 1].contiguous(), R.contiguous(),
                   torch.from_numpy(psi).to(device), dict(N=N, window=window, m_cap=m, seed=seed, Q=Q, qn=True))
    return QNInputs(x, qa, qb, qs, qs, np.asarray(charges[window - 1] if window > 0 else np.zeros(k, int)),
                    np.asarray(charges[window]), np.asarray(charges[window + 1]))


def heisenberg_chain_qn(N: int, window: int, m: int, seed: int, Q: int = 0, device="cpu") -> QNInputs:
    W = mpo.heisenberg_chain_W()
    c = heisenberg_channel_charges()
    return model_inputs_qn([W] * N, [c] * N, window, m, seed, Q, device)


def cylinder_qn(Lx: int, window: int, m: int, seed: int, Q: int = 0, device="cpu") -> QNInputs:
    N = Lx * mpo.CYL_WIDTH
    Ws = [mpo.cylinder_W(j) for j in range(N)]
    c = cylinder_channel_charges()
    return model_inputs_qn(Ws, [c] * N, window, m, seed, Q, device)
