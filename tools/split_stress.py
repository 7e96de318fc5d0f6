"""Stress: heff_svd_split on random shapes and spectra (Gaussian, graded over many decades,
rank-deficient, repeated values, tiny and huge scales), both directions, against
numpy's singular values (R23 tolerance) and the reconstruction Q C."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2007_14822_b200 import heff  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(11)
t_end = time.time() + float(sys.argv[1] if len(sys.argv) > 1 else 60)
n = bad = 0
while time.time() < t_end:
    M, N = (int(rng.integers(1, 600)) for _ in range(2))
    k = min(M, N)
    kind = rng.integers(0, 5)
    U, _ = np.linalg.qr(rng.standard_normal((M, k)))
    V, _ = np.linalg.qr(rng.standard_normal((N, k)))
    if kind == 0:
        s = np.abs(rng.standard_normal(k))
    elif kind == 1:
        s = 10.0 ** (-rng.uniform(0, 14, k))
    elif kind == 2:
        s = np.where(rng.random(k) < 0.5, 0.0, rng.random(k))
    elif kind == 3:
        s = np.repeat(rng.random(max(1, k // 4)), 4)[:k]
        s = np.pad(s, (0, k - s.size))
    else:
        s = rng.random(k) * 10.0 ** rng.uniform(-100, 100)
    if not np.any(s > 0):
        s[0] = 1.0
    Psi = (U * s) @ V.T
    for d in (0, 1):
        r = heff.svd_split(torch.from_numpy(Psi).to(dev).view(M, 1, 1, N), direction=d)
        ref = np.linalg.svd(Psi, compute_uv=False)
        S = r.S.cpu().numpy()[: ref.size]
        fro = np.linalg.norm(Psi)
        Q, C = r.Q.cpu().numpy(), r.C.cpu().numpy()
        rec = (Q.reshape(M, -1) @ C.reshape(-1, N)) if d == 0 else (C.reshape(M, -1) @ Q.reshape(-1, N))
        # defaults keep every value above the numerical-rank threshold (R21), so Q C = Psi up to
        # the discarded values below 1e-12 s_1
        ok = np.max(np.abs(S - ref)) <= 1e-12 * fro and np.linalg.norm(rec - Psi) <= 1e-11 * fro
        if not ok:
            bad += 1
            print("MISMATCH", M, N, kind, d, np.max(np.abs(S - ref)) / fro, np.linalg.norm(rec - Psi) / fro, flush=True)
        n += 1
print(f"stress: {n} splits, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
