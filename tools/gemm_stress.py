"""Stress: many back-to-back libheff GEMMs of random shapes (stream-K in-kernel reduction,
PDL, both tiles, accumulate) checked against torch.matmul -- looks for rare races."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2007_14822_b200.heff import gemm  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator().manual_seed(7)
t_end = time.time() + float(sys.argv[1] if len(sys.argv) > 1 else 60)
n = bad = 0
while time.time() < t_end:
    M, N, K = (int(torch.randint(1, 1500, (1,), generator=g)) for _ in range(3))
    bk = bool(torch.randint(0, 2, (1,), generator=g))
    acc = bool(torch.randint(0, 2, (1,), generator=g))
    A = torch.randn(M, K, dtype=torch.float64, device=dev)
    B = torch.randn((N, K) if bk else (K, N), dtype=torch.float64, device=dev)
    C0 = torch.randn(M, N, dtype=torch.float64, device=dev)
    outs = [gemm(A, B, bk, C=C0.clone(), accumulate=acc) for _ in range(4)]
    ref = (C0 if acc else 0) + A @ (B.T if bk else B)
    tol = 1e-12 * max(1.0, ref.abs().max().item()) * max(1.0, K ** 0.5)
    for o in outs:
        if not (o - ref).abs().max().item() <= tol or not torch.equal(o, outs[0]):
            bad += 1
            print("MISMATCH", M, N, K, bk, acc, flush=True)
    n += len(outs)
torch.cuda.synchronize()
print(f"stress: {n} GEMMs, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
