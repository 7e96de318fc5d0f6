"""P ranks of the b'-sharded libheff path as P host threads of one process on ONE GPU,
communicating through the NCCL test double tests/fake_nccl/fake_nccl.cc (loaded by libheff
via HEFF_NCCL_PATH).  Started as a subprocess by tests/test_gpu_fake_nccl.py:

    python tests/fake_nccl_worker.py <fake .so> <outdir> <config> <P> <steps> [<mode>]

mode "run": every rank builds its communicating plan (order B on b' in [r nb, (r+1) nb)),
runs heff_apply on the full psi and a fixed-step lanczos_ground through the all-gather +
re-layout exchange and the all-reduced CGS2 scalars; the shards are written to outdir.
mode "peer_missing": rank P-1 never calls lanczos_ground; the others must fail with
HEFF_ENCCL (the double's barrier timeout) instead of hanging.
All waiting happens on the host (no kernel waits for another rank).
"""
from __future__ import annotations

import json
import os
import sys
import threading
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def main(fake: str, outdir: str, config: str, P: int, steps: int, mode: str = "run") -> int:
    os.environ["HEFF_NCCL_PATH"] = fake          # before libheff loads any NCCL
    import numpy as np
    import torch

    from heffgen import configs as C
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200 import dist as hdist
    from paper_2007_14822_b200.heff import HeffError, OPT_COMM_STATE, OPT_FUSED_GATHER, nccl_unique_id

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    x = C.make(config)
    mR = x.dims["mR"]
    xd = x.to(dev)
    uid = nccl_unique_id()
    torch.cuda.synchronize()
    res: list = [None] * P

    def rank_fn(r: int):
        try:
            torch.cuda.set_device(dev)
            lo, hi = hdist.shard_range(mR, P, r)
            st = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(st):
                Rg = xd.R[lo:hi].contiguous()
                with Heff(xd.L, xd.W1, xd.W2, Rg, dist=dict(nranks=P, rank=r, b_lo=lo, b_hi=hi, uid=uid),
                          stream=st) as h:
                    assert h.get_option(OPT_COMM_STATE) == 1
                    out = h.apply(xd.psi, stream=st)
                    v = xd.psi[..., lo:hi].contiguous()
                    if mode == "peer_missing":
                        if r == P - 1:
                            res[r] = dict(skipped=True)
                            return
                        try:
                            h.lanczos_ground(v, max_iter=steps, stream=st)
                            res[r] = dict(error=None)
                        except HeffError as e:
                            res[r] = dict(error=str(e), code=e.code)
                        return
                    # the gather-fused path needs symmetric windows: the double has none, so
                    # the request must fail cleanly on every rank (before any collective)
                    h.set_option(OPT_FUSED_GATHER, 1)
                    try:
                        h.lanczos_ground(v.clone(), max_iter=steps, stream=st)
                        fused_err = None
                    except HeffError as e:
                        fused_err = str(e)
                    h.set_option(OPT_FUSED_GATHER, 0)
                    rr = h.lanczos_ground(v, max_iter=steps, stream=st)
                    st.synchronize()
                    np.save(Path(outdir) / f"out_{r}.npy", out.cpu().numpy())
                    np.save(Path(outdir) / f"ritz_{r}.npy", v.cpu().numpy())
                    res[r] = dict(energy=rr.energy, iters=rr.iters, alpha=list(rr.alpha), beta=list(rr.beta),
                                  fused_err=fused_err)
        except Exception as e:  # noqa: BLE001 -- reported to the parent test
            res[r] = dict(exception=repr(e))

    threads = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    (Path(outdir) / "result.json").write_text(json.dumps(res))
    return 0


if __name__ == "__main__":
    a = sys.argv[1:]
    sys.exit(main(a[0], a[1], a[2], int(a[3]), int(a[4]), *(a[5:6])))
