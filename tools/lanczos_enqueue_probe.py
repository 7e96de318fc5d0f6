"""Host enqueue time against device time of fixed-step lanczos_ground (is the Krylov loop
host-bound at small bonds?).  Prints, per config, the per-step device time (CUDA events
around the call) and the HEFF_LANCZOS_TIMING=1 enqueue / wait split from libheff."""
import os
import sys
from pathlib import Path

os.environ.setdefault("HEFF_LANCZOS_TIMING", "1")
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402

steps = 20
for name, kw in (("c1", {}), ("c2", dict(m=64)), ("c2", dict(m=128)), ("c2", {}), ("c4", dict(m=64)),
                 ("c4", dict(m=128))):
    x = C.make(name, device=torch.device("cuda:0"), **kw)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        for _ in range(3):
            h.lanczos_ground(x.psi.clone(), max_iter=steps)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            p = x.psi.clone()
            torch.cuda.synchronize()
            e0.record()
            h.lanczos_ground(p, max_iter=steps)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    print(f"PROBE {name} {kw} us/step {sorted(ts)}", flush=True)
