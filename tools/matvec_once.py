"""A few H_eff.psi matvecs at one config (profiling driver for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "c2"   # "c4:128" = preset c4 at bond cap m = 128
name, _, mm = spec.partition(":")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
x = C.make(name, device=torch.device("cuda:0"), m=int(mm) if mm else None)
with Heff(x.L, x.W1, x.W2, x.R) as h:
    out = torch.empty_like(x.psi)
    for _ in range(reps):
        h.apply(x.psi, out)
    torch.cuda.synchronize()
print("ok", name)
