"""Per-CTA timelines of the small-bond order-A kernels (heff_debug_fused_timestamps, %globaltimer
stamps written by consumer thread 0), back-to-back matvecs at one config:
  gemm1_mpo_fused_kernel: entry, after the dependency wait, after the main loop, after the T1
    staging, the first epilogue unit (CSR read, done), exit;
  gemm_cluster_splitk_kernel (GEMM4): entry, first stage ready, end of the main loop, after the
    partial push (ranks > 0) / the reduction wait (rank 0), exit.
    python tools/fused_timeline.py c2     (or c4:128 = preset c4 at m = 128)"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from heffgen import configs as C  # noqa: E402
from paper_2007_14822_b200 import Heff, heff  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
lib = heff.lib()
lib.heff_debug_fused_timestamps.argtypes = [ctypes.c_int, ctypes.c_void_p]
cfg, _, mm = name.partition(":")
x = C.make(cfg, device=torch.device("cuda:0"), m=int(mm) if mm else None)
n = 512
buf = np.zeros(8 * n, dtype=np.uint64)
with Heff(x.L, x.W1, x.W2, x.R) as h:
    out = torch.empty_like(x.psi)
    for _ in range(5):
        h.apply(x.psi, out)
    lib.heff_debug_fused_timestamps(n, None)
    for _ in range(5):
        h.apply(x.psi, out)
    torch.cuda.synchronize()
    lib.heff_debug_fused_timestamps(n, buf.ctypes.data)
    lib.heff_debug_fused_timestamps(0, None)
allt = buf.reshape(n, 8).astype(np.int64)
f = allt[: n // 2][:, [0, 1, 2, 4, 5, 6, 3]]
f = f[f[:, 0] > 0]
g = allt[n // 2:][:, [0, 1, 2, 3, 4]]
g = g[g[:, 0] > 0]
t0 = f[:, 0].min()


def show(t, labels, steps, title):
    rel = (t - t0) / 1e3
    print(f"{title}: {len(t)} CTAs; microseconds from the fused kernel's first entry")
    for k, lab in enumerate(labels):
        print(f"  {lab:22s} min {rel[:, k].min():7.2f}  median {np.median(rel[:, k]):7.2f}  max {rel[:, k].max():7.2f}")
    d = np.diff(t, axis=1) / 1e3
    for k, lab in enumerate(steps):
        print(f"  [{lab:20s}] min {d[:, k].min():7.2f}  median {np.median(d[:, k]):7.2f}  max {d[:, k].max():7.2f}")


if (allt[: n // 2, 5] == 0).all() and (allt[: n // 2, 4] > 0).any():
    # matvec_cluster_kernel (one launch): entry, GEMM1 done, MPO done, GEMM4 done, reduction done
    m = allt[: n // 2][:, [0, 1, 2, 3, 4]]
    m = m[m[:, 0] > 0]
    t0 = m[:, 0].min()
    show(m, ("entry", "GEMM1 done", "MPO -> T3 done", "GEMM4 done", "reduction done"),
         ("GEMM1 (incl. wait)", "MPO epilogue", "GEMM4 passes", "cluster reduction"), f"{name} matvec_cluster")
    sys.exit(0)
show(f, ("entry", "after pdl_wait", "after main loop", "after T1 staging", "1st unit CSR", "1st unit done", "exit"),
     ("wait", "main loop", "T1 -> smem", "to 1st unit", "1st unit", "other units"), f"{name} gemm1_mpo_fused")
if len(g):
    show(g, ("entry", "first stage", "after main loop", "after push/reduce wait", "exit"),
         ("ramp", "main loop", "push / wait", "sum + store"), f"{name} cluster GEMM4")
