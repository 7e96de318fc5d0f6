"""Named workload presets C1..C5 (BASELINE.json configs[0..4]) and generic builders.

Seeded-input module shared by the oracle tests and the CUDA path: it builds inputs
only and holds none of the H_eff / Lanczos arithmetic.  DESIGN.md section "Input
recipe" states each preset; seeds are 1000 + c for config c.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import env, mpo


@dataclass
class HeffInputs:
    L: torch.Tensor      # [mL, kL, mL]
    W1: torch.Tensor     # [kL, d1, d1, kM]
    W2: torch.Tensor     # [kM, d2, d2, kR]
    R: torch.Tensor      # [mR, kR, mR]
    psi: torch.Tensor    # [mL, d1, d2, mR], unit 2-norm
    meta: dict = field(default_factory=dict)

    @property
    def dims(self) -> dict:
        mL, kL, _ = self.L.shape
        _, d1, _, kM = self.W1.shape
        _, d2, _, kR = self.W2.shape
        mR = self.R.shape[0]
        return dict(mL=mL, d1=d1, d2=d2, mR=mR, kL=kL, kM=kM, kR=kR)

    def numpy(self):
        return tuple(t.detach().cpu().numpy() for t in (self.L, self.W1, self.W2, self.R, self.psi))

    def to(self, device):
        return HeffInputs(*(t.to(device) for t in (self.L, self.W1, self.W2, self.R, self.psi)), meta=dict(self.meta))


def random_psi(seed: int, shape, device="cpu") -> torch.Tensor:
    """psi ~ N(0,1) from default_rng(seed), divided by its 2-norm (reading R8)."""
    x = np.random.default_rng(seed).standard_normal(shape)
    x /= np.linalg.norm(x)
    return torch.from_numpy(x).to(device)


def graded_matrix(M: int, N: int, seed: int, decades: float = 12.0) -> np.ndarray:
    """Synthetic two-site matrix with a DMRG-like decaying spectrum: Q1 diag(s) Q2^T with
    Q1, Q2 the orthonormal factors of N(0,1) matrices (default_rng(seed)) and
    s_i = 10^(-decades * i / (k-1)), k = min(M, N), then unit Frobenius norm."""
    rng = np.random.default_rng(seed)
    k = min(M, N)
    Q1, _ = np.linalg.qr(rng.standard_normal((M, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((N, k)))
    s = 10.0 ** (-decades * np.arange(k) / max(1, k - 1))
    A = (Q1 * s[None, :]) @ Q2.T
    return A / np.linalg.norm(A)


def model_inputs(Ws: list[np.ndarray], window: int, m: int, seed: int, device="cpu", meta=None) -> HeffInputs:
    """Environments of a random orthonormal MPS around the two-site window (window, window+1).

    Ws[j] is the MPO tensor of site j (len(Ws) = N).  L is built over sites < window,
    R over sites > window+1, both with bond cap m.
    """
    N = len(Ws)
    d = Ws[0].shape[1]
    k = Ws[0].shape[0]
    rng = np.random.default_rng(seed)
    tW = [torch.from_numpy(np.ascontiguousarray(W)).to(device) for W in Ws]
    As = env.draw_left_block(rng, window, d, m, device)
    Bs = env.draw_right_block(rng, N - window - 2, d, m, device)
    L = env.build_left_env(As, tW[:window], k, device)
    R = env.build_right_env(Bs, tW[window + 2:], k, device)
    psi = random_psi(seed + 1, (L.shape[0], d, d, R.shape[0]), device)
    m_ = dict(meta or {})
    m_.update(N=N, window=window, m_cap=m, seed=seed)
    return HeffInputs(L.contiguous(), tW[window].contiguous(), tW[window + 1].contiguous(), R.contiguous(),
                      psi.contiguous(), m_)


def model_inputs_complex(Ws: list, window: int, m: int, seed: int, device="cpu") -> HeffInputs:
    """Complex analogue of model_inputs: random complex orthonormal MPS (real and imaginary
    parts N(0,1) from default_rng(seed)), environments with the bra side conjugated, psi
    complex N(0,1) from default_rng(seed+1), unit norm."""
    N = len(Ws)
    d = Ws[0].shape[1]
    k = Ws[0].shape[0]
    rng = np.random.default_rng(seed)
    tW = [torch.from_numpy(np.ascontiguousarray(W, dtype=np.complex128)).to(device) for W in Ws]
    As = env.draw_left_block(rng, window, d, m, device, complex_=True)
    Bs = env.draw_right_block(rng, N - window - 2, d, m, device, complex_=True)
    L = env.build_left_env(As, tW[:window], k, device)
    R = env.build_right_env(Bs, tW[window + 2:], k, device)
    r2 = np.random.default_rng(seed + 1)
    shape = (L.shape[0], d, d, R.shape[0])
    x = r2.standard_normal(shape) + 1j * r2.standard_normal(shape)
    x /= np.linalg.norm(x)
    return HeffInputs(L.contiguous(), tW[window].contiguous(), tW[window + 1].contiguous(), R.contiguous(),
                      torch.from_numpy(x).to(device), dict(N=N, window=window, m_cap=m, seed=seed, complex=True))


def dm_chain(N: int, window: int, m: int, seed: int, D: float = 0.5, device="cpu") -> HeffInputs:
    return model_inputs_complex([mpo.dm_chain_W(D)] * N, window, m, seed, device)


def model_inputs_terms(Ws_terms: list, window: int, m: int, seed: int, device="cpu") -> list:
    """Environments of ONE random orthonormal MPS for several MPOs (an MPO sum,
    P:L739-750).  Ws_terms[t][j] is term t's MPO tensor at site j.  The MPS draws are the
    same as model_inputs' for the same seed; psi is shared."""
    N = len(Ws_terms[0])
    d = Ws_terms[0][0].shape[1]
    rng = np.random.default_rng(seed)
    As = env.draw_left_block(rng, window, d, m, device)
    Bs = env.draw_right_block(rng, N - window - 2, d, m, device)
    out = []
    psi = None
    for Ws in Ws_terms:
        k = Ws[0].shape[0]
        tW = [torch.from_numpy(np.ascontiguousarray(W)).to(device) for W in Ws]
        L = env.build_left_env(As, tW[:window], k, device)
        R = env.build_right_env(Bs, tW[window + 2:], k, device)
        if psi is None:
            psi = random_psi(seed + 1, (L.shape[0], d, d, R.shape[0]), device)
        out.append(HeffInputs(L.contiguous(), tW[window].contiguous(), tW[window + 1].contiguous(), R.contiguous(),
                              psi, dict(N=N, window=window, m_cap=m, seed=seed, k=k)))
    return out


def heisenberg_chain_split(N: int, window: int, m: int, seed: int, device="cpu") -> list:
    """Eq. (1) as the MPO sum [Sz Sz terms, flip terms] (SPEC.md:771's dmrg([H1,H2]) example)."""
    return model_inputs_terms([[mpo.heisenberg_zz_W()] * N, [mpo.heisenberg_flip_W()] * N], window, m, seed, device)


def heisenberg_chain(N: int, window: int, m: int, seed: int, device="cpu") -> HeffInputs:
    W = mpo.heisenberg_chain_W()
    return model_inputs([W] * N, window, m, seed, device, dict(model="heisenberg_chain"))


def trivial_two_site(model: str = "heisenberg") -> HeffInputs:
    """N = 2 with the trivial boundary environments: L = left vector, R = right vector (1 x k x 1)."""
    W = mpo.heisenberg_chain_W() if model == "heisenberg" else mpo.hubbard_W()
    k, d = W.shape[0], W.shape[1]
    l, r = mpo.boundary_vectors(k)
    L = torch.from_numpy(l.reshape(1, k, 1).copy())
    R = torch.from_numpy(r.reshape(1, k, 1).copy())
    psi = random_psi(7, (1, d, d, 1))
    tW = torch.from_numpy(W)
    return HeffInputs(L, tW, tW.clone(), R, psi, dict(model=model, N=2, window=0))


def n_side_for(m: int, d: int) -> int:
    """Sites per side so that the edge-grown bond reaches m: ceil(log_d m) + 1."""
    return int(math.ceil(math.log(m, d) - 1e-12)) + 1


def random_dense(dims: dict, seed: int, device="cpu") -> HeffInputs:
    """Unstructured N(0,1) tensors of arbitrary dims (kernel parity at ragged shapes;
    not Hermitian, so never used for Lanczos)."""
    rng = np.random.default_rng(seed)
    mL, d1, d2, mR, kL, kM, kR = (dims[k] for k in ("mL", "d1", "d2", "mR", "kL", "kM", "kR"))
    t = lambda *s: torch.from_numpy(rng.standard_normal(s)).to(device)
    L, W1, W2, R = t(mL, kL, mL), t(kL, d1, d1, kM), t(kM, d2, d2, kR), t(mR, kR, mR)
    psi = random_psi(seed + 1, (mL, d1, d2, mR), device)
    return HeffInputs(L, W1, W2, R, psi, dict(model="random", seed=seed))


# ---------------------------------------------------------------- the five presets
CONFIGS = {
    # C1: BASELINE configs[0] -- m = 16 from a full-rank N = 10 chain, window (4,5) 0-based
    "c1": dict(model="heisenberg_chain", N=10, window=4, m=16, seed=1001),
    # C1's brute-force check: N = 8, window (2,3) -> mL = 4, mR = 16, spectrum of the 256x256 H
    "c1_n8": dict(model="heisenberg_chain", N=8, window=2, m=16, seed=1001),
    "c2": dict(model="heisenberg_chain", m=256, seed=1002),
    "c3": dict(model="heisenberg_chain", m=1024, seed=1003),
    # C4: 6x6 width-6 cylinder snaked into 36 sites, window (17,18) 0-based
    "c4": dict(model="cylinder", Lx=6, window=17, m=4096, seed=1004),
    # C5: Hubbard U=4 t=1 chain
    "c5": dict(model="hubbard", m=8192, seed=1005),
    # beyond BASELINE.json: Hubbard U=4 t=1 on a width-6 cylinder (d = 4, k = 26; reading R26),
    # 4 x 6 sites snaked into 24, window (11,12) -- the k d1 d2 = 416 MPO of the quasi-2D
    # Hubbard studies; a parity / throughput case of the MPO kernel's
    # narrow column tiles
    "hcyl6": dict(model="hubbard_cylinder", Lx=4, window=11, m=256, seed=1006),
}


def make(name: str, device="cpu", m: int | None = None) -> HeffInputs:
    """Build preset `name`; `m` overrides the bond cap (small stand-ins in tests)."""
    c = dict(CONFIGS[name])
    mm = m if m is not None else c["m"]
    if c["model"] == "heisenberg_chain":
        if "N" in c:
            return heisenberg_chain(c["N"], c["window"], mm, c["seed"], device)
        ns = n_side_for(mm, 2)
        return model_inputs([mpo.heisenberg_chain_W()] * (2 * ns + 2), ns, mm, c["seed"], device,
                            dict(model="heisenberg_chain", config=name))
    if c["model"] == "cylinder":
        N = c["Lx"] * mpo.CYL_WIDTH
        Ws = [mpo.cylinder_W(j) for j in range(N)]
        return model_inputs(Ws, c["window"], mm, c["seed"], device, dict(model="cylinder", config=name))
    if c["model"] == "hubbard_cylinder":
        N = c["Lx"] * mpo.CYL_WIDTH
        Ws = [mpo.hubbard_cylinder_W(j) for j in range(N)]
        return model_inputs(Ws, c["window"], mm, c["seed"], device, dict(model="hubbard_cylinder", config=name))
    if c["model"] == "hubbard":
        ns = n_side_for(mm, 4)
        return model_inputs([mpo.hubbard_W()] * (2 * ns + 2), ns, mm, c["seed"], device,
                            dict(model="hubbard", config=name))
    raise KeyError(name)


def flops_per_matvec(d: dict) -> float:
    """Algorithmic flops of one H_eff.psi (reading R16): the two GEMM steps plus the
    two dense MPO steps, 2 flop per multiply-add."""
    mL, d1, d2, mR, kL, kM, kR = (d[k] for k in ("mL", "d1", "d2", "mR", "kL", "kM", "kR"))
    g1 = 2.0 * mL * kL * mL * d1 * d2 * mR
    s2 = 2.0 * mL * d1 * kM * d2 * mR * kL * d1
    s3 = 2.0 * mL * d1 * d2 * kR * mR * kM * d2
    g4 = 2.0 * mL * d1 * d2 * mR * kR * mR
    return g1 + s2 + s3 + g4


def gemm_flops_per_matvec(d: dict) -> float:
    mL, d1, d2, mR, kL, kR = (d[k] for k in ("mL", "d1", "d2", "mR", "kL", "kR"))
    return 2.0 * mL * kL * mL * d1 * d2 * mR + 2.0 * mL * d1 * d2 * mR * kR * mR
