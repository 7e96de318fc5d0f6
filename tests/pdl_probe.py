"""Helper for tests/test_gpu_gemm.py::test_pdl_on_off_bitwise: runs a fixed sequence of
libheff calls (GEMMs, a C2 Lanczos run, a split) and saves the outputs."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff, heff  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(3)
A = torch.randn(1280, 256, dtype=torch.float64, device=dev, generator=g)
B = torch.randn(256, 1024, dtype=torch.float64, device=dev, generator=g)
outs = {"gemm": heff.gemm(A, B).cpu().numpy()}
x = C.make("c2", device=dev)
with Heff(x.L, x.W1, x.W2, x.R) as h:
    v = x.psi.clone()
    r = h.lanczos_ground(v, max_iter=12)
    outs["lanczos_v"] = v.cpu().numpy()
    outs["lanczos_e"] = np.array([r.energy])
sp = heff.svd_split(x.psi, maxdim=200)
outs["split_S"] = sp.S.cpu().numpy()
outs["split_Q"] = sp.Q.cpu().numpy()
np.savez(sys.argv[1], **outs)
