"""One fixed-step lanczos_ground at one config (profiling driver for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
x = C.make(name, device=torch.device("cuda:0"))
with Heff(x.L, x.W1, x.W2, x.R) as h:
    r = h.lanczos_ground(x.psi.clone(), max_iter=steps)
    torch.cuda.synchronize()
print("ok", name, r.energy)
