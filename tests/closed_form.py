"""Closed-form H_eff.psi of heffgen.closed.permuted_diagonal inputs (the four FSM paths of
(D); derivation in heffgen/closed.py).  Test infrastructure: plain numpy / torch indexing and
a 2x2-or-4x4 contraction over the site legs, evaluated on chosen output rows or columns."""
from __future__ import annotations

import numpy as np


def expected_rows(meta: dict, psi: np.ndarray, rows) -> np.ndarray:
    """out[a', :, :, :] for a' in rows (order-A row samples)."""
    rows = np.asarray(rows)
    pinv = np.argsort(meta["pi"])
    rinv = np.argsort(meta["rho"])
    src = pinv[rows]
    out = meta["eL"][src][:, None, None, None] * psi[src]
    out = out + meta["eR"][rinv][None, None, None, :] * psi[rows][:, :, :, rinv]
    out = out + np.einsum("ij,ajkb->aikb", meta["O1"], psi[rows])
    out = out + np.einsum("kl,ajlb->ajkb", meta["O2"], psi[rows])
    return out


def expected_cols(meta: dict, psi: np.ndarray, cols) -> np.ndarray:
    """out[:, :, :, b'] for b' in cols (order-B column samples), shape [mL, d1, d2, len(cols)]."""
    cols = np.asarray(cols)
    pinv = np.argsort(meta["pi"])
    rinv = np.argsort(meta["rho"])
    src = rinv[cols]
    out = meta["eL"][pinv][:, None, None, None] * psi[pinv][:, :, :, cols]
    out = out + meta["eR"][src][None, None, None, :] * psi[:, :, :, src]
    out = out + np.einsum("ij,ajkb->aikb", meta["O1"], psi[:, :, :, cols])
    out = out + np.einsum("kl,ajlb->ajkb", meta["O2"], psi[:, :, :, cols])
    return out


def expected_full_torch(meta: dict, psi):
    """The whole output with torch ops (GPU full-size check; no libheff kernel involved)."""
    import torch
    dev = psi.device
    pinv = torch.from_numpy(np.argsort(meta["pi"])).to(dev)
    rinv = torch.from_numpy(np.argsort(meta["rho"])).to(dev)
    eL = torch.from_numpy(meta["eL"]).to(dev)
    eR = torch.from_numpy(meta["eR"]).to(dev)
    O1 = torch.from_numpy(meta["O1"]).to(dev)
    O2 = torch.from_numpy(meta["O2"]).to(dev)
    out = eL[pinv][:, None, None, None] * psi[pinv]
    out += eR[rinv][None, None, None, :] * psi[:, :, :, rinv]
    out += torch.einsum("ij,ajkb->aikb", O1, psi)
    out += torch.einsum("kl,ajlb->ajkb", O2, psi)
    return out
