"""Plan creation/destruction cost and converge-mode Lanczos latency vs bond dimension
(the per-bond overheads of a DMRG sweep that builds one plan per bond)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402

dev = torch.device("cuda:0")
for cfg, m in (("c1", 10), ("c1", 100), ("c1", 200), ("c4", 256), ("c4", 512), ("c4", 1024)):
    x = C.make(cfg, m=m, device=dev)
    for _ in range(3):
        with Heff(x.L, x.W1, x.W2, x.R) as h:
            h.lanczos_ground(x.psi.clone(), max_iter=4)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        with Heff(x.L, x.W1, x.W2, x.R) as h:
            h.lanczos_ground(x.psi.clone(), max_iter=4)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        h.lanczos_ground(x.psi.clone(), max_iter=4)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            h.lanczos_ground(x.psi.clone(), max_iter=4)
        torch.cuda.synchronize()
        tl = (time.perf_counter() - t0) / 10
    ts.sort()
    print(f"{cfg} m={m} k={x.dims['kL']}: create+4-step lanczos+destroy median {ts[5]*1e3:.2f} ms "
          f"(min {ts[0]*1e3:.2f}, max {ts[-1]*1e3:.2f}); reused plan {tl*1e3:.2f} ms", flush=True)
