"""Kernel-level tests of libheff's FP64 DMMA GEMM (heff_gemm) against torch.matmul in fp64:
odd shapes, both B layouts, accumulate, both load paths, stream-K on/off, and bitwise
run-to-run determinism (which also exposes shared-memory reuse races)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1, 1), (7, 5, 3), (64, 64, 16), (80, 64, 16), (129, 130, 17), (1280, 1024, 256), (1024, 256, 1280),
          (640, 512, 128), (300, 900, 2000), (20, 4096, 4096)]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build()
    return torch.device("cuda:0")


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bk", [False, True])
@pytest.mark.parametrize("tile", [None, "64", "128"])
def test_gemm_vs_torch(dev, shape, bk, tile, monkeypatch):
    """tile: the automatic choice, or the 64x64 / 128x128 TMA tile forced (HEFF_GEMM_TILE)."""
    from paper_2007_14822_b200.heff import gemm
    if tile:
        monkeypatch.setenv("HEFF_GEMM_TILE", tile)
    M, N, K = shape
    g = torch.Generator(device=dev).manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn((N, K) if bk else (K, N), dtype=torch.float64, device=dev, generator=g)
    ref = A @ (B.T if bk else B)
    tol = 1e-13 * max(1.0, K ** 0.5) * ref.abs().max().item()
    paths = [0, 1] + ([2] if (K % 2 == 0 and (K if bk else N) % 2 == 0) else [])
    for path in paths:
        C1 = gemm(A, B, bk, path=path)
        C2 = gemm(A, B, bk, path=path)
        torch.cuda.synchronize()
        assert (C1 - ref).abs().max().item() <= tol, path
        assert torch.equal(C1, C2), f"path {path}: not bitwise reproducible"
        # accumulate
        C0 = torch.randn(M, N, dtype=torch.float64, device=dev, generator=g)
        C3 = gemm(A, B, bk, C=C0.clone(), accumulate=True, path=path)
        assert (C3 - (C0 + ref)).abs().max().item() <= tol + 1e-15 * C0.abs().max().item()


@pytest.mark.parametrize("sk", ["1", None])
@pytest.mark.parametrize("tile", ["64", "128"])
def test_gemm_streamk_toggle_identical_results_tolerance(dev, sk, tile, monkeypatch):
    from paper_2007_14822_b200.heff import gemm
    monkeypatch.setenv("HEFF_GEMM_TILE", tile)
    if sk:
        monkeypatch.setenv("HEFF_NO_STREAMK", sk)
    g = torch.Generator(device=dev).manual_seed(1)
    for (M, N, K) in ((1280, 1024, 256), (1024, 256, 1280), (5120, 4096, 1024)):
        A = torch.randn(M, K, dtype=torch.float64, device=dev, generator=g)
        B = torch.randn(K, N, dtype=torch.float64, device=dev, generator=g)
        ref = A @ B
        outs = [gemm(A, B) for _ in range(3)]
        torch.cuda.synchronize()
        assert all(torch.equal(outs[0], o) for o in outs[1:])
        assert (outs[0] - ref).abs().max().item() <= 1e-12 * ref.abs().max().item()


STREAMK_SHAPES = [(1280, 1024, 256), (1024, 256, 1280), (640, 512, 128), (300, 900, 2000), (20, 4096, 4096),
                  (5120, 4096, 1024), (129, 130, 1700)]


@pytest.mark.parametrize("tile", ["64", "128"])
def test_streamk_inkernel_fixup_bitwise_equals_fixup_kernel(dev, tile, monkeypatch):
    """The in-kernel stream-K reduction (highest contributor waits on release/acquire flags)
    sums the partial tiles in the fixup kernel's order: bitwise the same C, also in
    accumulate mode and across repeated launches (epoch-tagged flags, ticket reset)."""
    from paper_2007_14822_b200.heff import gemm
    monkeypatch.setenv("HEFF_GEMM_TILE", tile)
    g = torch.Generator(device=dev).manual_seed(11)
    for (M, N, K) in STREAMK_SHAPES:
        for bk in (False, True):
            A = torch.randn(M, K, dtype=torch.float64, device=dev, generator=g)
            B = torch.randn((N, K) if bk else (K, N), dtype=torch.float64, device=dev, generator=g)
            C0 = torch.randn(M, N, dtype=torch.float64, device=dev, generator=g)
            monkeypatch.delenv("HEFF_SK_FIXUP_KERNEL", raising=False)
            ink = [gemm(A, B, bk) for _ in range(3)]
            inka = gemm(A, B, bk, C=C0.clone(), accumulate=True)
            monkeypatch.setenv("HEFF_SK_FIXUP_KERNEL", "1")
            ref = gemm(A, B, bk)
            refa = gemm(A, B, bk, C=C0.clone(), accumulate=True)
            torch.cuda.synchronize()
            assert all(torch.equal(ref, x) for x in ink), (M, N, K, bk)
            assert torch.equal(refa, inka), (M, N, K, bk)
            exact = A @ (B.T if bk else B)
            assert (ref - exact).abs().max().item() <= 1e-12 * exact.abs().max().item()


def test_streamk_concurrent_streams_no_deadlock(dev):
    """Stream-K GEMMs from two host threads on two streams share the SMs; reducers only wait
    on CTAs that hold earlier tickets, so this finishes (a wait past ~10 s would trap)."""
    import threading
    from paper_2007_14822_b200.heff import gemm
    g = torch.Generator(device=dev).manual_seed(5)
    A = torch.randn(1024, 1280, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn(256, 1280, dtype=torch.float64, device=dev, generator=g)
    ref = A @ B.T
    errs = []

    def work():
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            outs = [gemm(A, B, True) for _ in range(50)]
        s.synchronize()
        errs.append(max((o - ref).abs().max().item() for o in outs))

    ts = [threading.Thread(target=work) for _ in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert len(errs) == 2 and max(errs) <= 1e-12 * ref.abs().max().item()


def test_streamk_one_thread_two_streams(dev):
    """One host thread enqueues stream-K GEMMs on two streams without synchronising: each
    stream gets its own partial-tile workspace and ticket counter, so the concurrently
    running kernels neither mix partial tiles nor wait on each other's CTAs."""
    from paper_2007_14822_b200.heff import gemm
    g = torch.Generator(device=dev).manual_seed(9)
    A = torch.randn(1024, 1280, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn(256, 1280, dtype=torch.float64, device=dev, generator=g)
    A2 = torch.randn(1280, 256, dtype=torch.float64, device=dev, generator=g)
    B2 = torch.randn(256, 1024, dtype=torch.float64, device=dev, generator=g)
    ref1, ref2 = A @ B.T, A2 @ B2
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    torch.cuda.synchronize()
    for _ in range(30):
        with torch.cuda.stream(s1):          # C allocated, zeroed and written on s1
            outs.append((1, gemm(A, B, True)))
        with torch.cuda.stream(s2):
            outs.append((2, gemm(A2, B2, False)))
    torch.cuda.synchronize()
    for k, o in outs:
        ref = ref1 if k == 1 else ref2
        assert (o - ref).abs().max().item() <= 1e-12 * ref.abs().max().item()


def test_pdl_on_off_bitwise(dev, tmp_path):
    """Programmatic dependent launch changes only when kernels start, never the arithmetic:
    GEMM, Lanczos and split outputs are bitwise the same with HEFF_NO_PDL=1 (separate
    processes: the switch is read once per process)."""
    import os
    import subprocess
    import sys
    import numpy as np
    probe = os.path.join(os.path.dirname(__file__), "pdl_probe.py")
    files = []
    for off in ("", "1"):
        env = dict(os.environ)
        env.pop("HEFF_NO_PDL", None)
        if off:
            env["HEFF_NO_PDL"] = off
        f = str(tmp_path / f"out{off or '0'}.npz")
        subprocess.run([sys.executable, probe, f], check=True, env=env, timeout=600)
        files.append(np.load(f))
    for k in files[0].files:
        assert np.array_equal(files[0][k], files[1][k]), k


# shapes whose 64x64 tile count x CS fills 60..100% of the SMs in one wave: the cluster
# split-K kernel (CS = 2 or 4 CTAs per tile, DSMEM reduction) runs them
CLUSTER_SHAPES = [(1024, 256, 1280), (512, 256, 2048), (1000, 250, 1100), (448, 320, 999), (200, 1200, 600)]


@pytest.mark.parametrize("shape", CLUSTER_SHAPES)
@pytest.mark.parametrize("bk", [False, True])
def test_gemm_cluster_splitk(dev, shape, bk, monkeypatch):
    """Cluster split-K against torch.matmul, bitwise run-to-run, with accumulate; and against
    the stream-K schedule (HEFF_NO_CLUSTER_SPLITK) within rounding."""
    from paper_2007_14822_b200.heff import gemm
    M, N, K = shape
    if (K if bk else N) % 2 or K % 2:
        pytest.skip("TMA path needs even row pitches")
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    A = torch.randn(M, K, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn((N, K) if bk else (K, N), dtype=torch.float64, device=dev, generator=g)
    ref = A @ (B.T if bk else B)
    tol = 1e-13 * max(1.0, K ** 0.5) * ref.abs().max().item()
    C1 = gemm(A, B, bk)
    C2 = gemm(A, B, bk)
    C0 = torch.randn(M, N, dtype=torch.float64, device=dev, generator=g)
    C3 = gemm(A, B, bk, C=C0.clone(), accumulate=True)
    monkeypatch.setenv("HEFF_NO_CLUSTER_SPLITK", "1")
    Csk = gemm(A, B, bk)
    torch.cuda.synchronize()
    assert (C1 - ref).abs().max().item() <= tol
    assert torch.equal(C1, C2), "cluster split-K not bitwise reproducible"
    assert (C3 - (C0 + ref)).abs().max().item() <= tol + 1e-15 * C0.abs().max().item()
    assert (C1 - Csk).abs().max().item() <= tol
