"""Per-CTA timeline of the fused small-bond kernel (heff_debug_fused_timestamps): entry,
after the dependency wait, after the main loop, exit -- back-to-back matvecs at one config."""
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
n = 148
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
t = buf.reshape(n, 8).astype(np.int64)[:, [0, 1, 2, 4, 3]]
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print(f"{name}: {len(t)} CTAs (last matvec); microseconds from the first CTA's entry")
for k, lab in enumerate(("entry", "after pdl_wait", "after main loop", "after T1 staging", "exit")):
    print(f"  {lab:16s} min {rel[:, k].min():7.2f}  median {np.median(rel[:, k]):7.2f}  max {rel[:, k].max():7.2f}")
d = np.diff(t, axis=1) / 1e3
for k, lab in enumerate(("wait", "main loop", "T1 -> smem", "MPO + T3 store")):
    print(f"  {lab:16s} min {d[:, k].min():7.2f}  median {np.median(d[:, k]):7.2f}  max {d[:, k].max():7.2f}")
