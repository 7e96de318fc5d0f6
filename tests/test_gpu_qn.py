"""GPU parity of the U(1) block-sparse H_eff (heff_set_qn; NEXT-3) against the dense
oracle on the same sector-structured inputs."""
import numpy as np
import pytest
import torch

from heffgen import qn
from tests import ed_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


CASES = {
    "chain_m256": lambda: qn.heisenberg_chain_qn(20, 9, 256, seed=11),
    "chain_m1024": lambda: qn.heisenberg_chain_qn(24, 11, 1024, seed=12),
    "chain_Q2": lambda: qn.heisenberg_chain_qn(20, 9, 200, seed=13, Q=2),
    "cylinder_m256": lambda: qn.cylinder_qn(3, 8, 256, seed=14),
    "n10_full": lambda: qn.heisenberg_chain_qn(10, 4, 16, seed=15),
}


@pytest.mark.parametrize("force", [True, False])
@pytest.mark.parametrize("case", sorted(CASES))
def test_qn_matvec_parity(dev, orc, case, force, monkeypatch):
    if force:
        monkeypatch.setenv("HEFF_QN_FORCE_SPARSE", "1")   # exercise the sparse kernel path at every size
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200.heff import OPT_SPARSE_KBLOCKS
    z = CASES[case]()
    L, W1, W2, R, psi = z.x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = z.x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        dense = h.apply(xd.psi).cpu().numpy()
        h.set_qn(z.qn_dict())
        nkb = h.get_option(OPT_SPARSE_KBLOCKS)
        out = h.apply(xd.psi).cpu().numpy()
        out2 = h.apply(xd.psi).cpu().numpy()
    assert rel(out, ref) <= 1e-12
    assert rel(dense, ref) <= 1e-12
    assert np.array_equal(out, out2)
    assert np.abs(out[~z.mask()]).max() == 0.0
    d = z.x.dims
    dense_kb = (-(-d["mL"] * d["kL"] // 128) * -(-d["d1"] * d["d2"] * d["mR"] // 128) * -(-d["mL"] // 16) +
                -(-d["mL"] * d["d1"] * d["d2"] // 128) * -(-d["mR"] // 128) * -(-d["kR"] * d["mR"] // 16))
    assert 0 < nkb <= dense_kb
    if force and d["mL"] >= 256:
        assert nkb < 0.8 * dense_kb     # the symmetry actually removes work


def test_qn_lanczos_sector_ED(dev):
    from paper_2007_14822_b200 import Heff
    H = ed_ref.heisenberg(10, ed_ref.chain_bonds(10)).toarray()
    sz2 = np.array([sum(1 if (i >> (9 - k)) & 1 == 0 else -1 for k in range(10)) for i in range(1024)])
    for Q in (0, 2):
        z = qn.heisenberg_chain_qn(10, 4, 16, seed=16, Q=Q)
        xd = z.x.to(dev)
        with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
            h.set_qn(z.qn_dict())
            r = h.lanczos_ground(xd.psi.clone(), max_iter=300, tol=1e-10, converge=True)
        e = np.linalg.eigvalsh(H[np.ix_(sz2 == Q, sz2 == Q)])[0]
        assert abs(r.energy - e) <= 1e-10


def test_qn_errors(dev):
    from paper_2007_14822_b200 import Heff, HeffError
    z = qn.heisenberg_chain_qn(20, 9, 64, seed=17)
    xd = z.x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        bad = z.qn_dict()
        bad["qa"] = bad["qa"][::-1].copy()
        with pytest.raises(HeffError):
            h.set_qn(bad)
        h.set_qn(z.qn_dict())
        h.set_qn(None)                      # back to dense
        h.apply(xd.psi)


@pytest.mark.parametrize("case", ["chain_m256", "cylinder_m256"])
def test_qn_lanczos_fixed_steps_parity(dev, orc, case):
    """Sector-compact Lanczos on the GPU vs the oracle's dense Lanczos on the same inputs."""
    from paper_2007_14822_b200 import Heff
    z = CASES[case]()
    L, W1, W2, R, psi = z.x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=12)
    xd = z.x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_qn(z.qn_dict())
        v = xd.psi.clone()
        r = h.lanczos_ground(v, max_iter=12)
    assert r.iters == o.iters == 12
    assert abs(r.energy - o.energy) <= 1e-10 * max(1.0, abs(o.energy))
    vc = v.cpu().numpy()
    assert np.abs(vc[~z.mask()]).max() == 0.0
    assert abs(abs(np.vdot(vc, o.x)) - 1.0) < 1e-8


def test_plan_lifecycle_returns_device_memory(dev):
    """Creating and destroying U(1), complex and plain plans (with Lanczos runs, which add
    the Krylov basis and the sector scatter buffers) leaves no device memory behind once
    heff_release_caches has emptied the workspace cache; before that, the cache reuses the
    destroyed plans' blocks instead of growing."""
    from heffgen import configs as C
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200.heff import release_caches
    z = CASES["chain_m256"]()
    xd = z.x.to(dev)
    xc = C.make("c2", device=dev)
    Lz = torch.complex(xc.L, 0.1 * xc.L).contiguous()
    W1z = torch.complex(xc.W1, torch.zeros_like(xc.W1)).contiguous()
    W2z = torch.complex(xc.W2, torch.zeros_like(xc.W2)).contiguous()
    Rz = torch.complex(xc.R, 0.1 * xc.R).contiguous()

    def cycle():
        with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
            h.set_qn(z.qn_dict())
            h.lanczos_ground(xd.psi.clone(), max_iter=6)
        with Heff(Lz, W1z, W2z, Rz) as hz:
            hz.apply(torch.complex(xc.psi, xc.psi).contiguous())
        with Heff(xc.L, xc.W1, xc.W2, xc.R) as h:
            h.lanczos_ground(xc.psi.clone(), max_iter=6)
        torch.cuda.synchronize()

    cycle()
    release_caches()
    torch.cuda.empty_cache()
    free0 = torch.cuda.mem_get_info()[0]
    cycle()
    free_cached = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        cycle()
    torch.cuda.empty_cache()
    assert torch.cuda.mem_get_info()[0] >= free_cached - (64 << 20)   # blocks reused, not re-allocated
    release_caches()
    torch.cuda.empty_cache()
    assert torch.cuda.mem_get_info()[0] >= free0 - (16 << 20)          # nothing leaked


def test_qn_c4qn_full_size_sampled_rows(dev, orc):
    """C4-QN (6x6 cylinder, m = 4096, Sz = 0 sector; the configuration of tools/sweep_qn.py)
    on the block-sparse schedules, against the dense oracle on sampled output rows."""
    from paper_2007_14822_b200 import Heff
    z = qn.cylinder_qn(6, 17, 4096, seed=2004, device=dev)
    xd = z.x
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_qn(z.qn_dict())
        out = h.apply(xd.psi)
        torch.cuda.synchronize()
    rows = [0, 1000, 2048, 4095]
    outc = out[rows].cpu().numpy()
    del out
    L, W1, W2, R, psi = xd.numpy()
    for i, a in enumerate(rows):
        ref = orc.heff_apply(L, W1, W2, R, psi, rows=(a, a + 1))[0]
        nrm = max(np.linalg.norm(ref), 1e-300)
        assert np.linalg.norm(outc[i] - ref) / nrm <= 1e-12, a
