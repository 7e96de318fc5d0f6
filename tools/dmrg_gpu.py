"""Two-site DMRG sweeps assembled from libheff's kernels -- an integration check that the
hot path composes into the paper's algorithm (Sec. 6.2): at every bond the
local eigensolve is libheff's lanczos_ground on H_eff (heff_create / heff_apply), the
environments move with heff_env_update_left/right, and the two-site tensor is formed with
heff_gemm, and the two-site split is libheff's heff_svd_split (block one-sided Jacobi SVD,
SURVEY 8(f) NEXT-2).  Every step of the sweep runs in libheff's kernels; this script only
sequences them.

    python tools/dmrg_gpu.py --N 20 --maxdim 64 --sweeps 4
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from heffgen import mpo  # noqa: E402
from paper_2007_14822_b200 import Heff, env_update_left, env_update_right, svd_split  # noqa: E402
from paper_2007_14822_b200.heff import gemm  # noqa: E402


def random_right_mps(rng, N, d, m, device):
    """Right-orthonormal random MPS with bond dims min(d^j, d^(N-j), m) (boundary bonds 1)."""
    D = [min(d ** j, d ** (N - j), m) for j in range(N + 1)]
    As = []
    for j in range(N):
        X = torch.from_numpy(rng.standard_normal((D[j], d * D[j + 1]))).to(device)
        Q, _ = torch.linalg.qr(X.T, mode="reduced")          # orthonormal rows of the block
        As.append(Q.T.reshape(D[j], d, D[j + 1]).contiguous())
    return As


def two_site(A, B):
    """psi[a,s1,s2,b] = sum_k A[a,s1,k] B[k,s2,b] on libheff's GEMM."""
    a, d1, k = A.shape
    _, d2, b = B.shape
    return gemm(A.reshape(a * d1, k), B.reshape(k, d2 * b)).reshape(a, d1, d2, b)


SPLIT_STATS = {"calls": 0, "sweeps": 0, "max_sweeps": 0, "ms": 0.0}

# DMRG_PHASES=1: per-sweep wall time of each step of a bond update (synchronising after each)
PHASES: dict = {}
_PHASES_ON = os.environ.get("DMRG_PHASES") == "1"


def _phase_clock():
    if _PHASES_ON:
        torch.cuda.synchronize()
    return time.perf_counter()


def _phase(name, t0):
    if not _PHASES_ON:
        return t0
    torch.cuda.synchronize()
    t = time.perf_counter()
    PHASES[name] = PHASES.get(name, 0.0) + (t - t0)
    return t


def split(psi, maxdim, cutoff, direction):
    """Truncated SVD of psi reshaped (a s1) x (s2 b) on libheff (heff_svd_split): keeps the
    largest singular values with relative discarded weight <= cutoff and at most maxdim
    (P:L521-546).  Moving right returns (U, S V^T), moving left (U S, V^T)."""
    a, d1, d2, b = psi.shape
    t0 = time.perf_counter()
    r = svd_split(psi, cutoff=cutoff, maxdim=maxdim, direction=0 if direction == "right" else 1)
    SPLIT_STATS["calls"] += 1
    SPLIT_STATS["sweeps"] += r.sweeps
    SPLIT_STATS["max_sweeps"] = max(SPLIT_STATS["max_sweeps"], r.sweeps)
    SPLIT_STATS["ms"] += 1e3 * (time.perf_counter() - t0)
    k = r.n
    if direction == "right":
        return r.Q.reshape(a, d1, k).contiguous(), r.C.reshape(k, d2, b).contiguous(), r.trunc_err
    return r.C.reshape(a, d1, k).contiguous(), r.Q.reshape(k, d2, b).contiguous(), r.trunc_err


def dmrg(Ws, maxdims, cutoff=1e-11, seed=0, lanczos_iter=40, init_dim=8, device="cuda", log=print, capture=None):
    """capture: optional dict; receives the converged two-site wavefunction of the centre
    bond (bond N/2-1, last left-to-right half sweep) under key "psi"."""
    N = len(Ws)
    d = Ws[0].shape[1]
    k = Ws[0].shape[0]
    tW = [torch.from_numpy(np.ascontiguousarray(W)).to(device) for W in Ws]
    # random right-orthonormal initial MPS (site tensors [a, s, b])
    rng = np.random.default_rng(seed)
    As = random_right_mps(rng, N, d, init_dim, device)
    # environments: Ls[j] = left of site j, Rs[j] = right of site j-1 (Rs[N] = boundary)
    Ls = [None] * (N + 1)
    Rs = [None] * (N + 2)
    Ls[0] = torch.zeros((1, k, 1), dtype=torch.float64, device=device)
    Ls[0][0, k - 1, 0] = 1.0
    Rs[N] = torch.zeros((1, k, 1), dtype=torch.float64, device=device)
    Rs[N][0, 0, 0] = 1.0
    for j in range(N - 1, 1, -1):
        Rs[j] = env_update_right(Rs[j + 1], As[j], tW[j])
    energy = None
    for sw, maxdim in enumerate(maxdims):
        t0 = time.perf_counter()
        maxdisc = 0.0
        # left-to-right then right-to-left half sweeps
        for direction, bonds in (("right", range(N - 1)), ("left", range(N - 2, -1, -1))):
            for j in bonds:
                tp = _phase_clock()
                psi = two_site(As[j], As[j + 1]).contiguous()
                tp = _phase("two_site", tp)
                with Heff(Ls[j], tW[j], tW[j + 1], Rs[j + 2]) as h:
                    tp = _phase("create", tp)
                    r = h.lanczos_ground(psi, max_iter=lanczos_iter, tol=1e-12, converge=True)
                    tp = _phase("lanczos", tp)
                tp = _phase("destroy", tp)
                energy = r.energy
                if capture is not None and direction == "right" and j == N // 2 - 1 and sw == len(maxdims) - 1:
                    capture["psi"] = psi.clone()
                A, B, disc = split(psi, maxdim, cutoff, direction)
                tp = _phase("split", tp)
                maxdisc = max(maxdisc, disc)
                As[j], As[j + 1] = A, B
                if direction == "right":
                    Ls[j + 1] = env_update_left(Ls[j], As[j], tW[j])
                else:
                    Rs[j + 1] = env_update_right(Rs[j + 2], As[j + 1], tW[j + 1])
                _phase("env", tp)
        if PHASES:
            log("  phases (s): " + ", ".join(f"{k} {v:.2f}" for k, v in PHASES.items()))
            PHASES.clear()
        log(f"After sweep {sw + 1} energy={energy:.12f} maxlinkdim={max(a.shape[2] for a in As[:-1])} "
            f"maxtrunc={maxdisc:.2e} time={time.perf_counter() - t0:.2f} split: {SPLIT_STATS['calls']} calls, "
            f"{SPLIT_STATS['sweeps'] / max(1, SPLIT_STATS['calls']):.1f} Jacobi sweeps avg "
            f"(max {SPLIT_STATS['max_sweeps']}), {SPLIT_STATS['ms'] / 1e3:.2f} s")
        SPLIT_STATS.update(calls=0, sweeps=0, max_sweeps=0, ms=0.0)
    return energy, As


def dmrg_qn(Ws, chan_q, maxdims, cutoff=1e-11, lanczos_iter=40, device="cuda", log=print):
    """U(1) (Sz-conserving) two-site DMRG in the Sz = 0 sector (reading R18 conventions):
    the start is the Neel product state; every bond declares its charges to the matvec
    (heff_set_qn: block-sparse GEMM schedules, Lanczos on the sector's entries), splits with
    heff_svd_split_qn (one SVD per centre-bond charge block), records the new bond's charges
    and grows the environments with heff_env_update_*_qn (block-sparse GEMM schedules).
    chan_q[j]: MPO channel charges of the bond right of site j."""
    from paper_2007_14822_b200.heff import psi_row_col_charges, svd_split_qn
    N = len(Ws)
    k = Ws[0].shape[0]
    qs = np.array([1, -1])
    tW = [torch.from_numpy(np.ascontiguousarray(W)).to(device) for W in Ws]
    As, bq = [], [np.array([0])]
    for j in range(N):                                   # Neel state: Up, Dn, Up, ...
        A = torch.zeros((1, 2, 1), dtype=torch.float64, device=device)
        A[0, j % 2, 0] = 1.0
        As.append(A)
        bq.append(bq[-1] + qs[j % 2])
    chan = [np.zeros(k, dtype=int)] + [np.asarray(c) for c in chan_q]   # chan[j] = bond left of site j
    Ls = [None] * (N + 1)
    Rs = [None] * (N + 2)
    Ls[0] = torch.zeros((1, k, 1), dtype=torch.float64, device=device)
    Ls[0][0, k - 1, 0] = 1.0
    Rs[N] = torch.zeros((1, k, 1), dtype=torch.float64, device=device)
    Rs[N][0, 0, 0] = 1.0
    def env_qn(j):  # charges of the site-j environment updates (heff_env_update_*_qn)
        return dict(qs=qs, cl=chan[j], cr=chan[j + 1])

    for j in range(N - 1, 1, -1):
        Rs[j] = env_update_right(Rs[j + 1], As[j], tW[j], qn=dict(q_in=bq[j + 1], q_out=bq[j], **env_qn(j)))
    energy = None
    for sw, maxdim in enumerate(maxdims):
        t0 = time.perf_counter()
        t_split = 0.0
        for direction, bonds in (("right", range(N - 1)), ("left", range(N - 2, -1, -1))):
            for j in bonds:
                psi = two_site(As[j], As[j + 1]).contiguous()
                with Heff(Ls[j], tW[j], tW[j + 1], Rs[j + 2]) as h:
                    h.set_qn(dict(qa=bq[j], qb=bq[j + 2], qs1=qs, qs2=qs, cL=chan[j], cM=chan[j + 1], cR=chan[j + 2]))
                    r = h.lanczos_ground(psi, max_iter=lanczos_iter, tol=1e-12, converge=True)
                energy = r.energy
                a, d1, d2, b = psi.shape
                qrow, qcol = psi_row_col_charges(bq[j], qs, qs, bq[j + 2])
                ts = time.perf_counter()
                sp = svd_split_qn(psi, qrow, qcol, cutoff=cutoff, maxdim=maxdim,
                                  direction=0 if direction == "right" else 1)
                t_split += time.perf_counter() - ts
                kk = sp.n
                bq[j + 1] = np.asarray(sp.qk)
                if direction == "right":
                    As[j], As[j + 1] = sp.Q.reshape(a, d1, kk).contiguous(), sp.C.reshape(kk, d2, b).contiguous()
                    Ls[j + 1] = env_update_left(Ls[j], As[j], tW[j], qn=dict(q_in=bq[j], q_out=bq[j + 1], **env_qn(j)))
                else:
                    As[j], As[j + 1] = sp.C.reshape(a, d1, kk).contiguous(), sp.Q.reshape(kk, d2, b).contiguous()
                    Rs[j + 1] = env_update_right(Rs[j + 2], As[j + 1], tW[j + 1],
                                                 qn=dict(q_in=bq[j + 2], q_out=bq[j + 1], **env_qn(j + 1)))
        log(f"After sweep {sw + 1} energy={energy:.12f} maxlinkdim={max(a.shape[2] for a in As[:-1])} "
            f"time={time.perf_counter() - t0:.2f} split {t_split:.2f} s")
    return energy, As, bq


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=20)
    ap.add_argument("--maxdim", type=int, default=64)
    ap.add_argument("--sweeps", type=int, default=4)
    ap.add_argument("--model", default="chain", choices=["chain", "cylinder"])
    ap.add_argument("--lanczos", type=int, default=40)
    ap.add_argument("--qn", action="store_true", help="U(1)-conserving sweeps in the Sz = 0 sector")
    ap.add_argument("--paper-a2", action="store_true",
                    help="the paper's App. A.2 run (PAPER.md:1498-1517): N = 100 S=1/2 Heisenberg chain, random "
                         "MPS of bond dimension 10, 5 sweeps with maxdim 10,20,100,100,200 and cutoff 1e-11")
    args = ap.parse_args()
    if args.paper_a2:
        t0 = time.perf_counter()
        e, As = dmrg([mpo.heisenberg_chain_W()] * 100, [10, 20, 100, 100, 200], cutoff=1e-11, init_dim=10,
                     lanczos_iter=args.lanczos)
        print(f"G.S. energy = {e:.12f}  E0/N = {e / 100:.8f}  ({time.perf_counter() - t0:.1f} s)")
        return
    if args.model == "chain":
        Ws = [mpo.heisenberg_chain_W()] * args.N
    else:
        Ws = [mpo.cylinder_W(j) for j in range(args.N)]
    maxdims = [min(args.maxdim, 10 * 2 ** s) for s in range(args.sweeps)]
    if args.qn:
        from heffgen import qn as hqn
        c = hqn.heisenberg_channel_charges() if args.model == "chain" else hqn.cylinder_channel_charges()
        e, _, _ = dmrg_qn(Ws, [c] * args.N, maxdims, lanczos_iter=args.lanczos)
        print(f"E0 = {e:.12f}  E0/N = {e / args.N:.8f}")
        return
    e, _ = dmrg(Ws, maxdims, lanczos_iter=args.lanczos)
    print(f"E0 = {e:.12f}  E0/N = {e / args.N:.8f}")


if __name__ == "__main__":
    main()
