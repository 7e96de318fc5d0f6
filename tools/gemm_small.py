"""Small-GEMM latency probe: the C2 matvec's GEMM shapes under the tile / stream-K knobs
(HEFF_GEMM_TILE, HEFF_NO_STREAMK read per launch)."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2007_14822_b200.heff import gemm  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
shapes = {"c2_gemm1": (1280, 1024, 256, False), "c2_gemm4": (1024, 256, 1280, True)}
for name, (M, N, K, bk) in shapes.items():
    A = torch.randn(M, K, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn((N, K) if bk else (K, N), dtype=torch.float64, device=dev, generator=g)
    C = torch.empty(M, N, dtype=torch.float64, device=dev)
    for tile in ("64", "128"):
        for sk in (None, "1"):
            os.environ["HEFF_GEMM_TILE"] = tile
            if sk:
                os.environ["HEFF_NO_STREAMK"] = sk
            else:
                os.environ.pop("HEFF_NO_STREAMK", None)
            for _ in range(20):
                gemm(A, B, bk, C=C)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                gemm(A, B, bk, C=C)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 200 * 1e3
            print(f"{name} tile={tile} streamk={'off' if sk else 'on'}: {us:.1f} us = {2*M*N*K/us/1e6:.1f} TF/s", flush=True)
