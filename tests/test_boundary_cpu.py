"""CPU-side checks of the C-ABI boundary: libheff builds for sm_100a, loads without a GPU,
and exports every function include/heff.h declares.  No compute calls (no GPU here)."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "heff.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|size_t|char\s*\*|const char\s*\*)\s*\*?\s*(heff_\w+|lanczos_ground)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_north_star_calls():
    fns = header_functions()
    for name in ("heff_create", "heff_apply", "lanczos_ground", "heff_destroy", "heff_last_error"):
        assert name in fns, fns


def test_library_builds_and_exports_every_symbol():
    import __graft_entry__ as g
    g.build()
    from paper_2007_14822_b200 import heff
    L = heff.lib()
    fns = header_functions()
    assert set(fns) <= set(heff.EXPORTED), set(fns) - set(heff.EXPORTED)
    for name in fns:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(heff.LIB_PATH)], capture_output=True, text=True).stdout
    for name in fns:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_with_dmma_and_tma():
    from paper_2007_14822_b200 import heff
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(heff.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass
    assert "DMMA.8x8x4" in sass          # FP64 tensor-core MMA
    assert "UTMALDG" in sass             # TMA loads


def test_product_path_does_not_import_oracle():
    pkg = ROOT / "paper_2007_14822_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("*.h")):
        t = f.read_text()
        assert "oracle" not in re.sub(r"#.*|//.*", "", t).replace("oracle/", ""), f


def test_binding_errors_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2007_14822_b200 import Heff
    t = torch.zeros(2, 2, 2, dtype=torch.float64)
    with pytest.raises(TypeError):
        Heff(t, t.reshape(2, 1, 2, 2), t.reshape(2, 1, 2, 2), t)


def test_library_tridiagonal_ql_vs_oracle_bisection_and_numpy(oracle_lib):
    """P10: libheff's host QL (used by lanczos_ground) vs the oracle's Sturm bisection vs
    numpy.linalg.eigh, no GPU needed."""
    import numpy as np
    from paper_2007_14822_b200 import heff
    rng = np.random.default_rng(11)
    for j in (1, 2, 5, 20, 150, 400):
        a = rng.standard_normal(j) * 3.0
        b = np.abs(rng.standard_normal(j - 1))
        th_q, y_q = heff.tridiag_lowest(a, b)
        th_b, y_b = oracle_lib.tridiag_lowest(a, b)
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        ev = np.linalg.eigvalsh(T)[0]
        scale = max(1.0, np.abs(a).max() + 2 * (b.max() if j > 1 else 0))
        assert abs(th_q - ev) <= 1e-14 * scale * 4
        assert abs(th_q - th_b) <= 1e-14 * scale * 4
        assert np.linalg.norm(T @ y_q - th_q * y_q) <= 1e-12 * scale
        assert abs(abs(np.dot(y_q, y_b)) - 1.0) <= 1e-9
        assert y_q[np.argmax(np.abs(y_q))] > 0
    # split matrix (a zero off-diagonal) and a 1x1
    th, y = heff.tridiag_lowest([2.0, -1.0, 3.0], [0.0, 0.5])
    assert abs(th - np.linalg.eigvalsh(np.diag([2.0, -1.0, 3.0]) + np.diag([0.0, 0.5], 1) + np.diag([0.0, 0.5], -1))[0]) < 1e-15


def test_library_tridiagonal_per_step_check_vs_numpy():
    """lanczos_ground's O(j) per-step check (Sturm bisection + inverse iteration) against
    numpy.linalg.eigh: the lowest eigenvalue to machine precision and |y[last]| of its unit
    eigenvector -- random T, Lanczos-like T of a Heisenberg-chain Hamiltonian (clustered
    low end), a split T (zero off-diagonal), 1x1 and 2x2 closed forms; no GPU needed."""
    import numpy as np
    from paper_2007_14822_b200 import heff
    rng = np.random.default_rng(12)
    cases = []
    for j in (3, 5, 20, 64, 150):
        cases.append((rng.standard_normal(j) * 3.0, np.abs(rng.standard_normal(j - 1))))
    # T_j of a Lanczos run on a random symmetric matrix with a clustered low spectrum
    n = 300
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([[-5.0, -4.999, -4.99], np.linspace(-4, 4, n - 3)])
    H = (Q * lam) @ Q.T
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    V, al, be = [v], [], []
    for k in range(60):
        w = H @ V[-1]
        al.append(V[-1] @ w)
        for _ in range(2):
            w -= np.array(V).T @ (np.array(V) @ w)
        be.append(np.linalg.norm(w))
        V.append(w / be[-1])
    for j in (10, 30, 60):
        cases.append((np.array(al[:j]), np.array(be[:j - 1])))
    for a, b in cases:
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        ev, U = np.linalg.eigh(T)
        scale = max(1.0, np.abs(a).max() + 2 * b.max())
        th, yl = heff.tridiag_lowest_check(a, b)
        assert abs(th - ev[0]) <= 8e-16 * scale * 4, (len(a), th, ev[0])
        if ev[1] - ev[0] > 1e-6 * scale:   # the eigenvector is well defined
            assert abs(yl - abs(U[-1, 0])) <= 1e-9 * max(1.0, 1.0 / (ev[1] - ev[0])), (len(a), yl, U[-1, 0])
    # closed forms: 1x1; 2x2 [[a, b], [b, c]]
    th, yl = heff.tridiag_lowest_check([1.5], [])
    assert th == 1.5 and yl == 1.0
    a0, c0, b0 = 1.0, 3.0, 0.5
    lo = 0.5 * (a0 + c0) - np.hypot(0.5 * (a0 - c0), b0)
    th, yl = heff.tridiag_lowest_check([a0, c0], [b0])
    y = np.array([b0, lo - a0])
    assert abs(th - lo) <= 1e-15 * 4 and abs(yl - abs(y[1]) / np.linalg.norm(y)) <= 1e-12
    # split matrix: the lowest eigenvalue sits in the first block, its last component is 0
    th, yl = heff.tridiag_lowest_check([-2.0, 1.0, 3.0], [0.3, 0.0])
    ev, U = np.linalg.eigh(np.diag([-2.0, 1.0, 3.0]) + np.diag([0.3, 0.0], 1) + np.diag([0.3, 0.0], -1))
    assert abs(th - ev[0]) <= 1e-14 and yl <= 1e-12


def test_host_truncation_rule_matches_oracle_and_brute_force():
    """heff_truncate_spectrum (the rule heff_svd_split applies on the host, readings R20/R21)
    against the oracle's rule and SPEC.md's brute-force cut scan, host-only."""
    import numpy as np
    from oracle import split as osplit
    from paper_2007_14822_b200 import heff
    from tests.test_oracle_split import _brute_kept
    assert heff.truncate_spectrum([1.0, 0, 0, 0]) == (1, 0.0)
    n, e = heff.truncate_spectrum(np.array([1.0, 1, 1, 1]) / 2, maxdim=2)
    assert n == 2 and abs(e - 0.5) < 1e-15
    rng = np.random.default_rng(12)
    for trial in range(400):
        k = int(rng.integers(1, 50))
        s = np.sort(np.exp(rng.uniform(-35, 0, k)))[::-1]
        if rng.random() < 0.2 and k > 1:
            s[rng.integers(1, k):] = 0.0
        cutoff = float(10 ** rng.uniform(-16, -1)) if rng.random() < 0.9 else 0.0
        maxdim, mindim = int(rng.integers(0, k + 3)), int(rng.integers(1, k + 2))
        got = heff.truncate_spectrum(s, cutoff, maxdim, mindim)
        ref = osplit.truncate_spectrum(s, cutoff, maxdim, mindim)
        assert got[0] == ref[0] == _brute_kept(s, cutoff, maxdim, mindim), (trial, got, ref)
        assert abs(got[1] - ref[1]) <= 1e-14 * max(1.0, ref[1])
    with pytest.raises(heff.HeffError):
        heff.truncate_spectrum([1.0, 2.0])
    with pytest.raises(heff.HeffError):
        heff.truncate_spectrum([1.0], cutoff=-1.0)
    with pytest.raises(heff.HeffZeroVector):
        heff.truncate_spectrum([0.0, 0.0])


def _build_c_demo(out):
    cmd = ["gcc", "-O2", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
           str(ROOT / "examples" / "heff_demo.c"), "-L", str(ROOT / "paper_2007_14822_b200"), "-lheff",
           f"-Wl,-rpath,{ROOT / 'paper_2007_14822_b200'}", "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", "-o", str(out)]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_abi_demo_compiles_and_links(tmp_path):
    """examples/heff_demo.c uses include/heff.h from plain C and links libheff.so -- the
    boundary is a C ABI, not a Python one."""
    import __graft_entry__ as g
    g.build()
    r = _build_c_demo(tmp_path / "heff_demo")
    assert r.returncode == 0, r.stderr
