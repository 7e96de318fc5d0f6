"""Matvec latency at small bonds (chain, k = 5; cylinder, k = 20): the fused small-bond
kernel vs the GEMM path (run twice, with and without HEFF_NO_SMALL_MATVEC=1)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402

dev = torch.device("cuda:0")
for cfg, ms in (("c1", (8, 16, 24, 32, 40, 48, 64)), ("c4", (8, 16, 24, 32))):
    for m in ms:
        x = C.make(cfg, m=m, device=dev)
        with Heff(x.L, x.W1, x.W2, x.R) as h:
            out = torch.empty_like(x.psi)
            for _ in range(20):
                h.apply(x.psi, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                h.apply(x.psi, out)
            e1.record()
            torch.cuda.synchronize()
        print(f"{cfg} m={m} k={x.dims['kL']}: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us", flush=True)
