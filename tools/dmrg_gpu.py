"""Two-site DMRG sweeps assembled from libheff's kernels -- an integration check that the
hot path composes into the paper's algorithm (Sec. 6.2): at every bond the
local eigensolve is libheff's lanczos_ground on H_eff (heff_create / heff_apply), the
environments move with heff_env_update_left/right, and the two-site tensor is formed with
heff_gemm.  The SVD split (not built in libheff yet) uses
torch.linalg.svd (cuSOLVER) here, so this script is a test harness, not a product path.

    python tools/dmrg_gpu.py --N 20 --maxdim 64 --sweeps 4
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from heffgen import mpo  # noqa: E402
from paper_2007_14822_b200 import Heff, env_update_left, env_update_right  # noqa: E402
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


def split(psi, maxdim, cutoff, direction):
    """Truncated SVD of psi reshaped (a s1) x (s2 b); keeps the largest singular values with
    discarded weight <= cutoff (relative) and at most maxdim."""
    a, d1, d2, b = psi.shape
    U, S, Vh = torch.linalg.svd(psi.reshape(a * d1, d2 * b), full_matrices=False)
    w = S * S
    tot = w.sum()
    tail = torch.flip(torch.cumsum(torch.flip(w, [0]), 0), [0])   # tail[i] = sum_{j >= i} w_j
    keep = int((tail / tot > cutoff).sum().item())
    keep = max(1, min(keep, maxdim))
    U, S, Vh = U[:, :keep], S[:keep], Vh[:keep]
    disc = float((tot - w[:keep].sum()) / tot)
    if direction == "right":
        return U.reshape(a, d1, keep).contiguous(), (S[:, None] * Vh).reshape(keep, d2, b).contiguous(), disc
    return (U * S[None, :]).reshape(a, d1, keep).contiguous(), Vh.reshape(keep, d2, b).contiguous(), disc


def dmrg(Ws, maxdims, cutoff=1e-11, seed=0, lanczos_iter=40, init_dim=8, device="cuda", log=print):
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
                psi = two_site(As[j], As[j + 1]).contiguous()
                with Heff(Ls[j], tW[j], tW[j + 1], Rs[j + 2]) as h:
                    r = h.lanczos_ground(psi, max_iter=lanczos_iter, tol=1e-12, converge=True)
                energy = r.energy
                A, B, disc = split(psi, maxdim, cutoff, direction)
                maxdisc = max(maxdisc, disc)
                As[j], As[j + 1] = A, B
                if direction == "right":
                    Ls[j + 1] = env_update_left(Ls[j], As[j], tW[j])
                else:
                    Rs[j + 1] = env_update_right(Rs[j + 2], As[j + 1], tW[j + 1])
        log(f"After sweep {sw + 1} energy={energy:.12f} maxlinkdim={max(a.shape[2] for a in As[:-1])} "
            f"maxtrunc={maxdisc:.2e} time={time.perf_counter() - t0:.2f}")
    return energy, As


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=20)
    ap.add_argument("--maxdim", type=int, default=64)
    ap.add_argument("--sweeps", type=int, default=4)
    args = ap.parse_args()
    W = mpo.heisenberg_chain_W()
    maxdims = [min(args.maxdim, 10 * 2 ** s) for s in range(args.sweeps)]
    e, _ = dmrg([W] * args.N, maxdims)
    print(f"E0 = {e:.12f}  E0/N = {e / args.N:.8f}")


if __name__ == "__main__":
    main()
