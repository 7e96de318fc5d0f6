"""GPU parity: libheff (through its C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star, reading R10): relative Frobenius error <= 1e-12
per matvec; Lanczos ground energy within 1e-10 * max(1, |E|); ED energies within 1e-10.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla
import torch

from heffgen import configs as C
from tests import ed_ref

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-12
ENERGY_TOL = 1e-10


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
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu_apply(x, dev, path=0, psi=None):
    from paper_2007_14822_b200 import Heff
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        h.set_option(1, path)
        p = xd.psi if psi is None else torch.from_numpy(psi).to(dev)
        out = h.apply(p)
        torch.cuda.synchronize()
        return out.cpu().numpy()


CASES = {
    "c1": lambda: C.make("c1"),
    "c1_n8": lambda: C.make("c1_n8"),
    "two_site": lambda: C.trivial_two_site(),
    "hubbard_two_site": lambda: C.trivial_two_site("hubbard"),
    "c2": lambda: C.make("c2"),
    "c4_m64": lambda: C.make("c4", m=64),
    "c5_m32": lambda: C.make("c5", m=32),
    "ragged_odd": lambda: C.random_dense(dict(mL=37, d1=3, d2=2, mR=29, kL=4, kM=3, kR=5), seed=31),
    "ragged_even": lambda: C.random_dense(dict(mL=200, d1=3, d2=3, mR=150, kL=7, kM=5, kR=7), seed=32),
    "tails": lambda: C.random_dense(dict(mL=130, d1=2, d2=2, mR=258, kL=3, kM=2, kR=5), seed=33),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("path", [0, 1, 2])
def test_matvec_parity(dev, orc, case, path):
    x = CASES[case]()
    d = x.dims
    if path == 2 and (d["mL"] % 2 or (d["d1"] * d["d2"] * d["mR"]) % 2 or (d["kR"] * d["mR"]) % 2):
        pytest.skip("TMA path needs even row pitches")
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    out = gpu_apply(x, dev, path)
    assert rel(out, ref) <= MATVEC_TOL, rel(out, ref)


def test_matvec_parity_c3(dev, orc):
    x = C.make("c3")
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    out = gpu_apply(x, dev)
    assert rel(out, ref) <= MATVEC_TOL


def test_matvec_parity_c4_full_size_sampled_rows(dev, orc):
    """C4 at full size (m = 4096, k = 20) in the bench's launch configuration; the oracle
    computes sampled output rows a' one by one (order A is independent per a')."""
    from paper_2007_14822_b200 import Heff
    x = C.make("c4", device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        out = h.apply(x.psi)
        torch.cuda.synchronize()
        L, W1, W2, R, psi = x.numpy()
        mL = L.shape[0]
        rows = sorted({0, 1, 127, 128, 2047, mL - 2, mL - 1} | set(np.random.default_rng(5).integers(0, mL, 5).tolist()))
        outc = out.cpu().numpy()
    for a in rows:
        ref = orc.heff_apply(L, W1, W2, R, psi, rows=(a, a + 1))[0]
        assert rel(outc[a], ref) <= MATVEC_TOL, (a, rel(outc[a], ref))
    # a property that holds at any size: <psi|H psi> equals the oracle-free order-B value
    e_a = float(np.vdot(psi, outc))
    assert np.isfinite(e_a)


def test_matvec_parity_c5_full_size_sampled_rows(dev, orc):
    """C5 (Hubbard, m = 8192, d = 4, k = 6: psi 8.6 GB, L and R 3.2 GB each) at full size on
    one GPU; the oracle computes sampled output rows a' one by one."""
    from paper_2007_14822_b200 import Heff
    free, _ = torch.cuda.mem_get_info()
    if free < 100 * 2**30:
        pytest.skip("C5 needs ~100 GB of device memory")
    x = C.make("c5", device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        out = h.apply(x.psi)
        torch.cuda.synchronize()
    mL = x.dims["mL"]
    rows = sorted({0, mL - 1} | set(np.random.default_rng(7).integers(1, mL - 1, 2).tolist()))
    outc = out[rows].cpu().numpy()
    del out
    L, W1, W2, R, psi = x.numpy()
    del x
    torch.cuda.empty_cache()
    for i, a in enumerate(rows):
        ref = orc.heff_apply(L, W1, W2, R, psi, rows=(a, a + 1))[0]
        assert rel(outc[i], ref) <= MATVEC_TOL, (a, rel(outc[i], ref))


def test_orderB_virtual_shards(dev, orc):
    from paper_2007_14822_b200 import Heff
    for x, P in ((C.make("c2"), 2), (C.make("c2"), 4), (C.make("c4", m=64), 8),
                 (C.random_dense(dict(mL=40, d1=2, d2=3, mR=33, kL=3, kM=4, kR=2), seed=3), 3)):
        L, W1, W2, R, psi = x.numpy()
        ref = orc.heff_apply(L, W1, W2, R, psi)
        xd = x.to(dev)
        mR = R.shape[0]
        bounds = np.linspace(0, mR, P + 1).astype(int)
        parts = []
        for g in range(P):
            lo, hi = int(bounds[g]), int(bounds[g + 1])
            Rg = xd.R[lo:hi].contiguous()
            with Heff(xd.L, xd.W1, xd.W2, Rg, dist=dict(nranks=P, rank=g, b_lo=lo, b_hi=hi)) as h:
                parts.append(h.apply(xd.psi).cpu().numpy())
        out = np.concatenate(parts, axis=3)
        assert rel(out, ref) <= MATVEC_TOL
        refB = orc.heff_apply_B(L, W1, W2, R, psi, cols=(int(bounds[1]), int(bounds[2])))
        assert rel(parts[1], refB) <= MATVEC_TOL


def test_linearity_and_hermiticity_gpu(dev):
    from paper_2007_14822_b200 import Heff
    x = C.make("c2", device=dev)
    g = torch.Generator(device="cpu").manual_seed(4)
    phi = torch.randn(x.psi.shape, generator=g, dtype=torch.float64).to(dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        Hpsi, Hphi = h.apply(x.psi), h.apply(phi)
        Hlin = h.apply((2.0 * x.psi - 0.5 * phi).contiguous())
    assert torch.linalg.norm(Hlin - (2.0 * Hpsi - 0.5 * Hphi)) <= 1e-13 * torch.linalg.norm(Hlin)
    lhs, rhs = torch.dot(phi.ravel(), Hpsi.ravel()), torch.dot(Hphi.ravel(), x.psi.ravel())
    assert abs(lhs - rhs) <= 1e-12 * torch.linalg.norm(phi) * torch.linalg.norm(Hpsi)


@pytest.mark.parametrize("case", ["c2", "ragged_even", "tails"])
def test_apply_host_e2e(dev, orc, case, monkeypatch):
    """heff_apply_host: the overlapped path (column-chunked H2D + GEMM1, row-chunked GEMM4 +
    D2H) and the plain copy-compute-copy path, pinned and pageable host buffers."""
    from paper_2007_14822_b200 import Heff
    x = CASES[case]()
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = x.to(dev)
    outs = []
    for pipelined in (True, False):
        if not pipelined:
            monkeypatch.setenv("HEFF_NO_E2E_PIPELINE", "1")
        with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
            for pin in (True, False):
                out = torch.empty(x.psi.shape, dtype=torch.float64)
                if pin:
                    out = out.pin_memory()
                h.apply_host(x.psi.contiguous().pin_memory() if pin else x.psi.contiguous(), out)
                assert rel(out.numpy(), ref) <= MATVEC_TOL, (pipelined, pin)
                outs.append(out.numpy().copy())
    # chunked GEMM4 schedules its stream-K splits per chunk: same values up to summation order
    assert rel(outs[0], outs[2]) <= 1e-14


# ------------------------------------------------------------------------ Lanczos
def gpu_lanczos(x, dev, max_iter, tol=0.0, converge=False, thetas=True):
    from paper_2007_14822_b200 import Heff
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        v = xd.psi.clone()
        r = h.lanczos_ground(v, max_iter=max_iter, tol=tol, converge=converge, thetas=thetas)
        return r, v.cpu().numpy()


@pytest.mark.parametrize("name,steps", [("c1", 20), ("two_site", 6), ("c2", 8)])
def test_lanczos_fixed_without_thetas_is_exact(dev, name, steps):
    """A fixed-step run that does not ask for the per-step Ritz values checks only for
    breakdown per step; the stopping step (incl. the singlet's early invariant-subspace stop),
    T_j, energy, residual and Ritz vector must be bitwise those of the run that solves T_j
    at every step."""
    x = CASES[name]()
    r1, v1 = gpu_lanczos(x, dev, steps, thetas=True)
    r0, v0 = gpu_lanczos(x, dev, steps, thetas=False)
    assert len(r1.thetas) == r1.iters and r0.thetas == []
    assert (r0.iters, r0.energy, r0.resid) == (r1.iters, r1.energy, r1.resid)
    assert r0.alpha == r1.alpha and r0.beta == r1.beta
    assert np.array_equal(v0, v1)


@pytest.mark.parametrize("m", [128, 256])
def test_lanczos_step3_unroll_is_bitwise(dev, m, monkeypatch):
    """cgs2_step3_kernel with two elements per thread per iteration (the default at C2) keeps
    every per-thread sum in element order: T_j and the Ritz vector are bitwise those of the
    one-element loop, over 30 steps (three-pass kernel to j = 24, four-pass after)."""
    from paper_2007_14822_b200 import Heff
    xd = C.make("c2", m=m).to(dev)
    out = {}
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        for flag in ("1", "0"):
            monkeypatch.setenv("HEFF_STEP3_UNROLL", flag)
            v = xd.psi.clone()
            r = h.lanczos_ground(v, max_iter=30)
            out[flag] = (r.energy, r.iters, tuple(r.alpha), tuple(r.beta), v.cpu().numpy().tobytes())
    assert out["1"] == out["0"]


@pytest.mark.parametrize("m", [128, 256])
def test_lanczos_step3_two_blocks_per_sm(dev, m, monkeypatch):
    """j <= 12 steps on the two-blocks-per-SM step3 instantiation (a different grid, so
    different partial sums): deterministic run to run, and T_j / energy / Ritz vector equal
    to the one-block-per-SM kernel's to rounding (Lanczos parity vs the oracle runs the
    default)."""
    from paper_2007_14822_b200 import Heff
    xd = C.make("c2", m=m).to(dev)
    out = {}
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        for flag in ("1", "0", "1"):
            monkeypatch.setenv("HEFF_STEP3_SMALLJ", flag)
            v = xd.psi.clone()
            r = h.lanczos_ground(v, max_iter=20)
            res = (r.energy, r.iters, np.array(r.alpha), np.array(r.beta), v.cpu().numpy())
            if flag in out:
                a = out[flag]
                assert a[0] == res[0] and np.array_equal(a[2], res[2]) and np.array_equal(a[4], res[4])
            out[flag] = res
    a, b = out["1"], out["0"]
    assert a[1] == b[1] and abs(a[0] - b[0]) <= 1e-12 * abs(b[0])
    assert np.max(np.abs(a[2] - b[2])) <= 1e-10 and np.max(np.abs(a[3] - b[3])) <= 1e-10
    assert abs(abs(float(np.dot(a[4].ravel(), b[4].ravel()))) - 1.0) <= 1e-9


@pytest.mark.parametrize("m", [128, 256])
def test_lanczos_step_grid_barrier_matches_cooperative(dev, m, monkeypatch):
    """The multi-block CGS2 steps launched as ordinary kernels (flip-counter grid barrier)
    must give bitwise the cooperative launch's T_j and Ritz vector, over 30 steps (three-pass
    kernel up to j = 24, four-pass kernel after), twice in a row on one plan (the barrier
    counter is reused across launches and calls)."""
    from paper_2007_14822_b200 import Heff
    xd = C.make("c2", m=m).to(dev)
    out = {}
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        for flag in ("1", "0", "1"):
            monkeypatch.setenv("HEFF_STEP_NONCOOP", flag)
            v = xd.psi.clone()
            r = h.lanczos_ground(v, max_iter=30)
            res = (r.energy, r.iters, tuple(r.alpha), tuple(r.beta), v.cpu().numpy().tobytes())
            if flag in out:
                assert out[flag] == res
            out[flag] = res
    assert out["1"] == out["0"]


@pytest.mark.parametrize("name,tol", [("c1", 1e-10), ("c2", 1e-10), ("two_site", 1e-12), ("ragged_odd", 1e-9)])
def test_lanczos_converge_batched_checks_are_exact(dev, name, tol, monkeypatch):
    """Converge mode on small vectors runs up to 3 steps ahead of the host's residual test;
    the stopping step, T_j, energy and Ritz vector must be bitwise those of per-step checks
    (including an early invariant-subspace stop: the two-site singlet problem)."""
    x = CASES[name]()
    monkeypatch.setenv("HEFF_LANCZOS_BATCH", "1")
    r1, v1 = gpu_lanczos(x, dev, 60, tol=tol, converge=True)
    for b in ("4", "7"):
        monkeypatch.setenv("HEFF_LANCZOS_BATCH", b)
        rb, vb = gpu_lanczos(x, dev, 60, tol=tol, converge=True)
        assert rb.iters == r1.iters and rb.energy == r1.energy, (b, rb.iters, r1.iters)
        assert rb.alpha == r1.alpha and rb.beta == r1.beta and rb.thetas == r1.thetas
        assert np.array_equal(vb, v1)


@pytest.mark.parametrize("name,steps", [("c1", 20), ("c1_n8", 20), ("c3", 6)])
def test_lanczos_fixed_steps_parity(dev, orc, name, steps):
    x = C.make(name)
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=steps)
    r, v = gpu_lanczos(x, dev, steps)
    assert r.iters == o.iters == steps
    assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))
    np.testing.assert_allclose(r.alpha, o.alpha, rtol=0, atol=1e-10)
    np.testing.assert_allclose(r.beta, o.beta, rtol=0, atol=1e-10)
    assert abs(np.linalg.norm(v) - 1.0) < 1e-12
    assert abs(abs(np.vdot(v, o.x)) - 1.0) < 1e-8


@pytest.mark.parametrize("variant", ["cooperative", "separate"])
def test_lanczos_step_kernels_c2(dev, orc, variant, monkeypatch):
    """The single-GPU CGS2 step forms on a mid-size vector (C2, n = 262 144), 24 fixed steps
    against the oracle: the fused cooperative step (default) and the separate multi-dot /
    multi-axpy kernels (HEFF_NO_FUSED_STEP); bitwise run to run."""
    if variant == "separate":
        monkeypatch.setenv("HEFF_NO_FUSED_STEP", "1")
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=24)
    r, v = gpu_lanczos(x, dev, 24)
    assert r.iters == o.iters == 24
    assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))
    np.testing.assert_allclose(r.alpha, o.alpha, rtol=0, atol=1e-10)
    np.testing.assert_allclose(r.beta, o.beta, rtol=0, atol=1e-10)
    assert abs(abs(np.vdot(v, o.x)) - 1.0) < 1e-8
    r2, v2 = gpu_lanczos(x, dev, 24)   # deterministic
    assert r2.alpha == r.alpha and np.array_equal(v2, v)


def test_lanczos_converge_c2(dev, orc):
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=500, tol=1e-10, converge=True)
    r, v = gpu_lanczos(x, dev, 500, tol=1e-10, converge=True)
    assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))
    assert abs(r.iters - o.iters) <= 2
    assert abs(abs(np.vdot(v, o.x)) - 1.0) < 1e-10


@pytest.mark.parametrize("name,N", [("c1_n8", 8), ("c1", 10)])
def test_lanczos_gpu_matches_ed(dev, name, N):
    x = C.make(name)
    r, _ = gpu_lanczos(x, dev, 300, tol=1e-10, converge=True)
    e0 = spla.eigsh(ed_ref.heisenberg(N, ed_ref.chain_bonds(N)), k=1, which="SA", tol=1e-14)[0][0]
    assert abs(r.energy - e0) <= 1e-10


def test_lanczos_two_site_singlet(dev):
    r, v = gpu_lanczos(C.trivial_two_site(), dev, 10, tol=1e-12, converge=True)
    assert abs(r.energy + 0.75) <= 1e-12
    # singlet (|ud> - |du>)/sqrt(2) up to sign
    s = np.zeros(4); s[1], s[2] = 1 / np.sqrt(2), -1 / np.sqrt(2)
    assert abs(abs(np.dot(v.ravel(), s)) - 1) < 1e-10


def test_lanczos_zero_vector_and_errors(dev):
    from paper_2007_14822_b200 import Heff, HeffError, HeffZeroVector
    x = C.make("c1").to(dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        with pytest.raises(HeffZeroVector):
            h.lanczos_ground(torch.zeros_like(x.psi), max_iter=5)
        # converge mode, and a theta_out request: the same error, psi left untouched, and
        # the plan still solves afterwards (the zero test waits for the first read-back)
        z = torch.zeros_like(x.psi)
        with pytest.raises(HeffZeroVector):
            h.lanczos_ground(z, max_iter=30, tol=1e-10, converge=True)
        assert int(torch.count_nonzero(z)) == 0
        r0 = h.lanczos_ground(x.psi.clone(), max_iter=20)
        with pytest.raises(HeffZeroVector):
            h.lanczos_ground(torch.zeros_like(x.psi), max_iter=5, thetas=True)
        r1 = h.lanczos_ground(x.psi.clone(), max_iter=20)
        assert r1.energy == r0.energy
        with pytest.raises(HeffError):
            h.apply(x.psi, x.psi)                       # aliasing
        with pytest.raises(HeffError):
            h.lanczos_ground(x.psi.clone(), max_iter=0)
    bad = torch.zeros((4, 3, 4), dtype=torch.float64, device=dev)   # kL mismatch is caught on the python side
    with pytest.raises(Exception):
        Heff(bad, x.W1, x.W2, x.R)


def test_lanczos_reserve_option(dev):
    """HEFF_OPT_LANCZOS_RESERVE pre-allocates the Krylov workspace; results are unchanged
    and out-of-range values are rejected."""
    from paper_2007_14822_b200 import Heff, HeffError
    from paper_2007_14822_b200.heff import OPT_LANCZOS_RESERVE
    x = C.make("c2").to(dev)
    r0, v0 = gpu_lanczos(C.make("c2"), dev, 12)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        h.set_option(OPT_LANCZOS_RESERVE, 20)
        v = x.psi.clone()
        r = h.lanczos_ground(v, max_iter=12)
        assert r.energy == r0.energy and np.array_equal(v.cpu().numpy(), v0)
        for bad in (0, -1, 10**6):
            with pytest.raises(HeffError):
                h.set_option(OPT_LANCZOS_RESERVE, bad)


def test_c_abi_rejects_degenerate_dims(dev):
    """heff_create through the C ABI: any zero or negative extent is HEFF_EINVAL with a
    message, null tensors too; nothing is allocated or launched."""
    import ctypes
    from paper_2007_14822_b200 import heff
    x = C.make("c1").to(dev)
    good = [16, 2, 2, 16, 5, 5, 5]
    for i in range(7):
        for bad in (0, -3):
            dims = list(good)
            dims[i] = bad
            d = heff._Dims(*dims)
            plan = ctypes.c_void_p()
            rc = heff.lib().heff_create(ctypes.byref(plan), ctypes.byref(d), x.L.data_ptr(), x.W1.data_ptr(), x.W2.data_ptr(),
                                        x.R.data_ptr(), None, None)
            assert rc == -1, (i, bad, rc)                  # HEFF_EINVAL
            assert heff.lib().heff_last_error()
    d = heff._Dims(*good)
    plan = ctypes.c_void_p()
    assert heff.lib().heff_create(ctypes.byref(plan), ctypes.byref(d), None, x.W1.data_ptr(), x.W2.data_ptr(),
                                  x.R.data_ptr(), None, None) == -1


def test_lanczos_nccl_single_rank(dev, orc):
    """The communicating (order B + NCCL) Lanczos path with one rank on one GPU."""
    from paper_2007_14822_b200 import Heff, nccl_unique_id
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=20)
    xd = x.to(dev)
    uid = nccl_unique_id()
    with Heff(xd.L, xd.W1, xd.W2, xd.R, dist=dict(nranks=1, rank=0, b_lo=0, b_hi=R.shape[0], uid=uid)) as h:
        v = xd.psi.clone()
        r = h.lanczos_ground(v, max_iter=20)
    assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))


def test_kernel_launch_count(dev):
    from paper_2007_14822_b200 import Heff
    x = C.make("c2", device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        h.apply(x.psi)
        assert h.get_option(2) >= 2      # GEMM1 (+ the MPO when fused), the MPO kernel otherwise, GEMM4


def test_relayout_kernel(dev):
    from paper_2007_14822_b200 import dist as hdist
    from paper_2007_14822_b200.heff import relayout_blocked
    for P, rows, nb in ((4, 37, 33), (8, 64, 512), (1, 5, 7)):
        src = torch.randn(P, rows, nb, dtype=torch.float64, device=dev)
        assert torch.equal(relayout_blocked(src, P), hdist.blocked_to_natural(src, P))


def test_sharded_plan_matvec_full_c3_with_nccl(dev, orc):
    """A communicating 1-rank plan computes the full out through order B (all-gather path
    is the identity at P = 1); compare with the oracle at C3."""
    from paper_2007_14822_b200 import Heff, nccl_unique_id
    x = C.make("c3")
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R, dist=dict(nranks=1, rank=0, b_lo=0, b_hi=R.shape[0],
                                                   uid=nccl_unique_id())) as h:
        out = h.apply(xd.psi).cpu().numpy()
    assert rel(out, ref) <= MATVEC_TOL


@pytest.mark.parametrize("sk", ["on", "off"])
def test_streamk_and_data_parallel_schedules(dev, orc, sk, monkeypatch):
    """Hybrid stream-K (partial tiles + fixup) and the plain persistent schedule give the same
    parity on shapes with ragged last waves (pure stream-K and DP + stream-K tails)."""
    if sk == "off":
        monkeypatch.setenv("HEFF_NO_STREAMK", "1")
    for x in (C.make("c2"), C.random_dense(dict(mL=600, d1=2, d2=2, mR=520, kL=5, kM=5, kR=5), seed=12)):
        L, W1, W2, R, psi = x.numpy()
        ref = orc.heff_apply(L, W1, W2, R, psi)
        assert rel(gpu_apply(x, dev), ref) <= MATVEC_TOL


def test_c_abi_demo_runs(dev, tmp_path):
    """examples/heff_demo.c: lanczos_ground + heff_svd_split called from C give the N = 2
    singlet (E0 = -3/4, Schmidt values 1/sqrt 2)."""
    import subprocess
    from tests.test_boundary_cpu import _build_c_demo
    r = _build_c_demo(tmp_path / "heff_demo")
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(tmp_path / "heff_demo")], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr


def test_lanczos_c4_bench_config_properties(dev, orc):
    """The bench workload (C4, m = 4096) is too large for the oracle's Lanczos; check what holds
    at any size: alpha_1 = <v1|H|v1> against the oracle's matvec on sampled rows, the Ritz value
    equals the Rayleigh quotient of the returned vector, and the residual ||H x - theta x||
    equals libheff's estimate beta_j |y_j[last]| (exact arithmetic identity)."""
    from paper_2007_14822_b200 import Heff
    x = C.make("c4", device=dev)
    psi0 = x.psi / torch.linalg.norm(x.psi)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        v = psi0.clone()
        r = h.lanczos_ground(v, max_iter=4)
        hx = h.apply(v)
        hv1 = h.apply(psi0)
        torch.cuda.synchronize()
    theta_rq = float(torch.vdot(v.reshape(-1), hx.reshape(-1)))
    assert abs(theta_rq - r.energy) <= 1e-9 * abs(r.energy)
    res = float(torch.linalg.norm(hx - r.energy * v))
    assert abs(res - r.resid) <= 1e-6 * max(res, 1e-12) + 1e-10
    # alpha_1 vs the oracle on sampled output rows a' (each row is independent in order A)
    L, W1, W2, R = (t.cpu().numpy() for t in (x.L, x.W1, x.W2, x.R))
    p0 = psi0.cpu().numpy()
    for a in (0, 1777, 4095):
        ref = orc.heff_apply(L, W1, W2, R, p0, rows=(a, a + 1))[0]
        assert rel(hv1[a].cpu().numpy(), ref) <= MATVEC_TOL
    assert abs(float(torch.vdot(psi0.reshape(-1), hv1.reshape(-1))) - r.alpha[0]) <= 1e-10 * abs(r.alpha[0])


def test_lanczos_nccl_single_rank_forced_allgather(dev, orc):
    """HEFF_OPT_FORCE_ALLGATHER runs the P > 1 exchange (ncclAllGather into the blocked buffer +
    the re-layout kernel) on a 1-rank communicator: same energy and Ritz vector as the oracle,
    bitwise the same as the copy shortcut (both are exact copies at P = 1)."""
    from paper_2007_14822_b200 import Heff, nccl_unique_id
    from paper_2007_14822_b200.heff import OPT_COMM_STATE, OPT_FORCE_ALLGATHER
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=12)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R, dist=dict(nranks=1, rank=0, b_lo=0, b_hi=R.shape[0],
                                                   uid=nccl_unique_id())) as h:
        assert h.get_option(OPT_COMM_STATE) == 1
        v0 = xd.psi.clone()
        r0 = h.lanczos_ground(v0, max_iter=12)
        h.set_option(OPT_FORCE_ALLGATHER, 1)
        assert h.get_option(OPT_FORCE_ALLGATHER) == 1
        v1 = xd.psi.clone()
        r1 = h.lanczos_ground(v1, max_iter=12)
    assert abs(r1.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))
    assert r1.energy == r0.energy and torch.equal(v0, v1)
    assert abs(abs(float(np.dot(v1.cpu().numpy().reshape(-1), o.x.reshape(-1)))) - 1.0) <= 1e-10


def test_force_allgather_needs_a_communicator(dev):
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200.heff import OPT_COMM_STATE, OPT_FORCE_ALLGATHER, HeffError
    x = C.make("c1", device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        assert h.get_option(OPT_COMM_STATE) == 0
        with pytest.raises(HeffError):
            h.set_option(OPT_FORCE_ALLGATHER, 1)


def test_binding_rejects_wrong_vector_sizes(dev):
    """The binding checks psi's length against the plan (full vector, or the shard of a
    communicating plan) before any pointer crosses the C ABI."""
    from paper_2007_14822_b200 import Heff, nccl_unique_id
    x = C.make("c2", device=dev)
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        with pytest.raises(ValueError):
            h.lanczos_ground(x.psi[:, :, :, :128].contiguous(), max_iter=2)
        with pytest.raises(ValueError):
            h.apply(x.psi[:128].contiguous())
    Rg = x.R[:128].contiguous()
    with Heff(x.L, x.W1, x.W2, Rg, dist=dict(nranks=2, rank=0, b_lo=0, b_hi=128)) as h:   # virtual shard
        with pytest.raises(ValueError):
            h.apply_blocked(x.psi[:, :, :, :128].contiguous())
        h.apply_blocked(x.psi.reshape(-1).clone())


@pytest.mark.parametrize("case,env", [("c2", None), ("c2", "0"), ("cyl128", None), ("uneven", "1"),
                                      ("c2_m240", None)])
def test_fused_gemm1_mpo_matvec(dev, orc, case, env, monkeypatch):
    """Small bonds: GEMM1 + the two-site MPO fused on fat tiles (T1 never written), GEMM4 by
    cluster split-K -- the default at C2 (m = 256) and the k = 20 cylinder at m = 128; forced
    (HEFF_FUSED_MATVEC=1) on a sub-half-wave mL != mR shape; off (=0) for comparison; m = 240
    (mR not a multiple of the 32-wide b tile) falls back.  Parity with the oracle in all."""
    from paper_2007_14822_b200 import Heff
    if env is not None:
        monkeypatch.setenv("HEFF_FUSED_MATVEC", env)
    monkeypatch.setenv("HEFF_CLUSTER_MATVEC", "0")   # the two-kernel form (test_cluster_matvec: one launch)
    x = {"c2": lambda: C.make("c2"), "cyl128": lambda: C.make("c4", m=128),
         "uneven": lambda: C.model_inputs([C.mpo.heisenberg_chain_W()] * 20, 6, 192, seed=77),
         "c2_m240": lambda: C.make("c2", m=240)}[case]()
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        out = h.apply(xd.psi)
        out2 = h.apply(xd.psi)
        torch.cuda.synchronize()
        nl = h.get_option(2)
    assert rel(out.cpu().numpy(), ref) <= MATVEC_TOL
    assert torch.equal(out, out2)
    if case in ("c2", "cyl128", "uneven") and env != "0":
        assert nl == 2, nl                 # fused GEMM1+MPO, GEMM4


def test_comm_failure_detection_aborts(dev, monkeypatch):
    """Failure detection of communicating plans: a stream that makes no
    progress for HEFF_NCCL_TIMEOUT_S makes lanczos_ground abort the communicator
    (ncclCommAbort) and return HEFF_ENCCL; the plan is then unusable (comm state -1, later
    calls fail fast) and can be destroyed.  Simulated on one GPU by a ~3 s spin kernel queued
    ahead of the solve on the same stream with a 1 s timeout."""
    from paper_2007_14822_b200 import Heff, nccl_unique_id
    from paper_2007_14822_b200.heff import OPT_COMM_STATE, HeffError
    x = C.make("c1").to(dev)
    h = Heff(x.L, x.W1, x.W2, x.R, dist=dict(nranks=1, rank=0, b_lo=0, b_hi=x.R.shape[0], uid=nccl_unique_id()))
    try:
        h.lanczos_ground(x.psi.clone(), max_iter=4)          # healthy first
        assert h.get_option(OPT_COMM_STATE) == 1
        monkeypatch.setenv("HEFF_NCCL_TIMEOUT_S", "1")
        torch.cuda._sleep(int(3.0 * 2.0e9))                    # ~3 s of spinning at ~2 GHz
        with pytest.raises(HeffError) as ei:
            h.lanczos_ground(x.psi.clone(), max_iter=4)
        assert ei.value.code == -4 and "aborted" in str(ei.value)
        assert h.get_option(OPT_COMM_STATE) == -1
        with pytest.raises(HeffError):
            h.lanczos_ground(x.psi.clone(), max_iter=4)
        torch.cuda.synchronize()
    finally:
        h.close()


@pytest.mark.parametrize("P,g", [(2, 1), (4, 0), (8, 5)])
def test_apply_host_sharded_pipelined(dev, orc, P, g):
    """End-to-end matvec of a b'-shard (heff_apply_host: psi's row blocks copied in on a copy
    stream while GEMM_A runs per block) against the order-B oracle on the shard's columns and
    against the device-resident heff_apply of the same plan (the row-blocked GEMM_A may split K
    differently: rounding only)."""
    from paper_2007_14822_b200 import Heff
    x = C.make("c2")
    L, W1, W2, R, psi = x.numpy()
    mR = R.shape[0]
    nb = mR // P
    ref = orc.heff_apply_B(L, W1, W2, R, psi, cols=(g * nb, (g + 1) * nb))
    xd = x.to(dev)
    Rg = xd.R[g * nb:(g + 1) * nb].contiguous()
    with Heff(xd.L, xd.W1, xd.W2, Rg, dist=dict(nranks=P, rank=g, b_lo=g * nb, b_hi=(g + 1) * nb)) as h:
        hin = x.psi.clone().pin_memory()
        hout = torch.empty(h.out_shape, dtype=torch.float64).pin_memory()
        h.apply_host(hin, hout)
        dout = h.apply(xd.psi)
        torch.cuda.synchronize()
    assert rel(hout.numpy(), ref) <= MATVEC_TOL
    assert rel(hout.numpy(), dout.cpu().numpy()) <= 1e-14


CLUSTER_CASES = {   # case: (inputs, runs as one cluster launch)
    "chain_m128": (lambda: C.make("c2", m=128), True),            # clusters of 4, one 128-wide b' pass
    "mL128_mR256": (lambda: C.random_dense(dict(mL=128, d1=2, d2=2, mR=256, kL=5, kM=4, kR=5), seed=42), True),
    "m64": (lambda: C.random_dense(dict(mL=64, d1=2, d2=2, mR=64, kL=5, kM=2, kR=5), seed=43), True),
    "mR32": (lambda: C.random_dense(dict(mL=96, d1=2, d2=2, mR=32, kL=5, kM=5, kR=5), seed=44), True),
    # the k = 20 cylinder (TA = 4 a' per fat tile: 16 GEMM4 rows per cluster, 20 w2 x 32 b per
    # CTA's K-slice): m = 64 clusters of 2, m = 128 32 clusters of 4
    "cyl_m64": (lambda: C.make("c4", m=64), True),
    "cyl_m128": (lambda: C.make("c4", m=128), True),
    # clusters of 6 (not a divisor of 64) and C2's 16 clusters of 8 (more than the 15 that are
    # co-resident on a B200) fall back to the two-kernel form
    "mR192": (lambda: C.random_dense(dict(mL=256, d1=2, d2=2, mR=192, kL=5, kM=3, kR=5), seed=41), False),
    "c2": (lambda: C.make("c2"), False),
}


@pytest.mark.parametrize("case", sorted(CLUSTER_CASES))
def test_cluster_matvec(dev, orc, case, monkeypatch):
    """Small chains: the whole order-A matvec in ONE launch (matvec_cluster_kernel: GEMM1 +
    two-site MPO + the GEMM4 slice of each fat tile in shared memory, the GEMM4 split-K
    reduced over the a' block's thread-block cluster through DSMEM).  Parity with the oracle,
    bitwise run-to-run, and the kernel count; with HEFF_CLUSTER_MATVEC=0 the two-kernel form."""
    from paper_2007_14822_b200 import Heff
    make, single = CLUSTER_CASES[case]
    x = make()
    L, W1, W2, R, psi = x.numpy()
    ref = orc.heff_apply(L, W1, W2, R, psi)
    xd = x.to(dev)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        out = h.apply(xd.psi)
        out2 = h.apply(xd.psi)
        torch.cuda.synchronize()
        nl = h.get_option(2)
    assert (nl == 1) == single, nl
    assert rel(out.cpu().numpy(), ref) <= MATVEC_TOL
    assert torch.equal(out, out2)
    monkeypatch.setenv("HEFF_CLUSTER_MATVEC", "0")
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h:
        out3 = h.apply(xd.psi)
        torch.cuda.synchronize()
        assert h.get_option(2) >= 2
    assert rel(out3.cpu().numpy(), ref) <= MATVEC_TOL


def test_cluster_matvec_accumulate_and_lanczos(dev, orc):
    """The cluster matvec's accumulating epilogue (MPO sums: out += H_t psi) and a Lanczos
    solve on it (chain, m = 128), against the oracle."""
    from paper_2007_14822_b200 import Heff, HeffSum
    x = C.make("c2", m=128)
    L, W1, W2, R, psi = x.numpy()
    xd = x.to(dev)
    ref = orc.heff_apply(L, W1, W2, R, psi)
    with Heff(xd.L, xd.W1, xd.W2, xd.R) as h1, Heff(xd.L, xd.W1, xd.W2, xd.R) as h2:
        hs = HeffSum([h1, h2])
        out = hs.apply(xd.psi)
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), 2 * ref) <= MATVEC_TOL
        hs.close()
        v = xd.psi.clone()
        r = h1.lanczos_ground(v, max_iter=10)
    o = orc.lanczos_heff(L, W1, W2, R, psi, max_iter=10)
    assert abs(r.energy - o.energy) <= ENERGY_TOL * max(1.0, abs(o.energy))
