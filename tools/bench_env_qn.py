"""U(1) environment update (heff_env_update_left/right_qn) vs dense at C4-QN size (6x6 cylinder,
m = 4096, Sz = 0) on one GPU."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from heffgen import mpo  # noqa: E402
from heffgen import qn as hqn  # noqa: E402
from paper_2007_14822_b200 import heff  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


dev = torch.device("cuda:0")
m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
z = hqn.cylinder_qn(6, 17, m, 1105, device=dev)
qs = np.array([1, -1])
c = hqn.cylinder_channel_charges()
W = torch.from_numpy(mpo.cylinder_W(17)).to(dev)
rng = np.random.default_rng(3)
qa_new = np.sort(np.asarray((z.qa[:, None] + qs[None, :]).ravel()))[np.linspace(0, 2 * m - 1, m).round().astype(int)]
mask = qa_new[None, None, :] == z.qa[:, None, None] + qs[None, :, None]
A = torch.from_numpy(rng.standard_normal(mask.shape) * mask).to(dev)
qn = dict(q_in=z.qa, q_out=qa_new, qs=qs, cl=c, cr=c)
td, Ld = timed(lambda: heff.env_update_left(z.x.L, A, W))
tq, Lq = timed(lambda: heff.env_update_left(z.x.L, A, W, qn=qn))
row = dict(m=m, dense_ms=td, qn_ms=tq, speedup=td / tq, rel_diff=float((Ld - Lq).norm() / Ld.norm()))
print(json.dumps(row))
