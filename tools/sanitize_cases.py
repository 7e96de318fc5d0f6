"""Small invocations of every libheff kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from heffgen import configs as C  # noqa: E402
from heffgen import mpo  # noqa: E402
from paper_2007_14822_b200 import Heff, HeffSum, env_update_left, env_update_right  # noqa: E402
from paper_2007_14822_b200.heff import relayout_blocked  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    # order A: TMA path (c1, c2 with split-K), plain path (ragged), trivial two-site
    for x, path in ((C.make("c1"), 0), (C.make("c2", m=128), 0), (C.make("c2", m=128), 1),
                    (C.random_dense(dict(mL=37, d1=3, d2=2, mR=29, kL=4, kM=3, kR=5), seed=1), 0),
                    (C.trivial_two_site(), 0), (C.make("c5", m=32), 2)):
        xd = x.to(dev)
        with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
            h.set_option(1, path)
            h.apply(xd.psi)
            h.lanczos_ground(xd.psi.clone(), max_iter=4)
    # unfused Lanczos BLAS-1 kernels
    os.environ["HEFF_NO_FUSED_STEP"] = "1"
    xd = C.make("c1").to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.lanczos_ground(xd.psi.clone(), max_iter=5, tol=1e-8, converge=True)
    del os.environ["HEFF_NO_FUSED_STEP"]
    # order B virtual shards
    xd = C.make("c2", m=64).to(dev)
    for g in range(2):
        lo, hi = 32 * g, 32 * (g + 1)
        with Heff(xd.L, xd.W1, xd.W2, xd.R[lo:hi].contiguous(), dist=dict(nranks=2, rank=g, b_lo=lo, b_hi=hi)) as h:
            h.apply(xd.psi)
    # penalty and MPO sum
    terms = [t.to(dev) for t in C.heisenberg_chain_split(12, 5, 32, seed=3)]
    plans = [Heff(t.L, t.W1, t.W2, t.R) for t in terms]
    hs = HeffSum(plans)
    hs.set_penalty(torch.randn((2,) + tuple(terms[0].psi.shape), dtype=torch.float64, device=dev), 3.0)
    hs.apply(terms[0].psi)
    hs.lanczos_ground(terms[0].psi.clone(), max_iter=4)
    hs.close()
    for p in plans:
        p.close()
    # environment updates and the relayout map
    rng = np.random.default_rng(0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for mi, d, mo, W in ((16, 2, 32, mpo.heisenberg_chain_W()), (7, 4, 9, mpo.hubbard_W())):
        k = W.shape[0]
        env_update_left(t(rng.standard_normal((mi, k, mi))), t(rng.standard_normal((mi, d, mo))), t(W))
        env_update_right(t(rng.standard_normal((mi, k, mi))), t(rng.standard_normal((mo, d, mi))), t(W))
    relayout_blocked(torch.randn(3, 5, 7, dtype=torch.float64, device=dev), 3)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
