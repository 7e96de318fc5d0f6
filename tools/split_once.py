"""One heff_svd_split call at a config size (profiling driver for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import heff  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = sys.argv[2] if len(sys.argv) > 2 else "random"
dev = torch.device("cuda:0")
if kind == "random":
    psi = C.random_psi(1000 + m, (m, 2, 2, m), dev)
else:
    psi = torch.from_numpy(C.graded_matrix(2 * m, 2 * m, 7, 12.0)).to(dev).view(m, 2, 2, m)
r = heff.svd_split(psi, maxdim=m)
torch.cuda.synchronize()
print(f"m={m} kind={kind} sweeps={r.sweeps} n={r.n} err={r.trunc_err:.3e}")
