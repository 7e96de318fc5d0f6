"""The communicating b'-sharded path with P > 1 ranks, executed on ONE
GPU through an NCCL test double (tests/fake_nccl/fake_nccl.cc): P host threads of one
process, one libheff plan per rank, collectives with host-side rendezvous (no kernel waits
for another rank).  This runs the P > 1 branches that a single-GPU box otherwise never
reaches -- ncclAllGather of the Krylov shard into the blocked buffer, the re-layout, the
all-reduced CGS2 dot products and norms, equal-shard checks, the fused-gather refusal
without symmetric windows, and the error return when a peer never arrives -- and checks
them against the CPU oracle.  It is a correctness test of libheff's orchestration, not of
NCCL's transport (tests/test_gpu_multirank.py does that on P GPUs).
"""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
MATVEC_TOL = 1e-12
ENERGY_TOL = 1e-10
STEPS = 6


@pytest.fixture(scope="module")
def fake_nccl(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__ as g
    g.build()
    from paper_2007_14822_b200.build import nccl_include
    so = tmp_path_factory.mktemp("fake_nccl") / "libfakenccl.so"
    subprocess.run(["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-I", "/usr/local/cuda/include", "-I",
                    nccl_include(), str(ROOT / "tests" / "fake_nccl" / "fake_nccl.cc"), "-o", str(so),
                    "-L", "/usr/local/cuda/lib64/stubs", "-lcuda"], check=True)
    return so


def _run(so, outdir, cfg, P, mode="run", env_extra=None, timeout=600):
    import os
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "fake_nccl_worker.py"), str(so), str(outdir), cfg,
                        str(P), str(STEPS), mode], env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads((Path(outdir) / "result.json").read_text())


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_lanczos_fake_nccl(fake_nccl, P, tmp_path):
    from heffgen import configs as C
    from oracle import oracle

    cfg = "c2"                                   # m = 256: nb = 128 / 64 / 32
    res = _run(fake_nccl, tmp_path, cfg, P)
    for r in res:
        assert "exception" not in r, r
    oracle.build()
    x = C.make(cfg)
    L, W1, W2, R, psi = x.numpy()
    ref = oracle.heff_apply(L, W1, W2, R, psi)
    out = np.concatenate([np.load(tmp_path / f"out_{r}.npy") for r in range(P)], axis=-1)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= MATVEC_TOL
    o = oracle.lanczos_heff(L, W1, W2, R, psi, max_iter=STEPS)
    for r in res:
        # every rank forms the same all-reduced scalars: identical tridiagonals and energies
        assert r["alpha"] == res[0]["alpha"] and r["beta"] == res[0]["beta"]
        assert r["iters"] == o.iters
        assert abs(r["energy"] - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy)), (r["energy"], o.energy)
        assert r["fused_err"] is not None and "symmetric-memory windows" in r["fused_err"]
    v = np.concatenate([np.load(tmp_path / f"ritz_{r}.npy") for r in range(P)], axis=-1).reshape(-1)
    assert abs(np.linalg.norm(v) - 1.0) <= 1e-12
    assert abs(abs(float(np.dot(v, o.x.reshape(-1)))) - 1.0) <= 1e-10


def test_missing_peer_fails_instead_of_hanging(fake_nccl, tmp_path):
    """Rank P-1 never enters lanczos_ground: the other ranks' first collective must come back
    with HEFF_ENCCL (the double's 3 s barrier timeout), not block forever."""
    from paper_2007_14822_b200.heff import HEFF_ENCCL

    P = 2
    res = _run(fake_nccl, tmp_path, "c1", P, mode="peer_missing", env_extra={"FAKE_NCCL_TIMEOUT_S": "3"},
               timeout=300)
    assert res[P - 1] == {"skipped": True}
    for r in res[:-1]:
        assert "exception" not in r, r
        assert r["error"] is not None and r["code"] == HEFF_ENCCL, r
