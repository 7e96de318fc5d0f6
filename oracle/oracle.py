"""ctypes front end of the CPU oracle (oracle/heff_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(paper_2007_14822_b200) never imports it, and this module imports nothing from the
product path.

Every function here is marshalling around the C oracle; the arithmetic and its paper
citations live in heff_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "heff_oracle.c"
_LIB = _HERE / "liboracle.so"

# x86-64-v3 = AVX2 + FMA: present on every Xeon this runs on (build here, run on the GPU box host)
CFLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> Path:
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        cmd = ["gcc", *CFLAGS, "-o", str(_LIB), str(_SRC), "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class _Dims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("mL", "d1", "d2", "mR", "kL", "kM", "kR")]


MATVEC_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double))

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(_LIB))
        dp = ctypes.POINTER(ctypes.c_double)
        _lib.ref_heff_direct.argtypes = [ctypes.POINTER(_Dims), dp, dp, dp, dp, dp, dp]
        _lib.ref_heff_direct.restype = None
        for f in (_lib.ref_heff_apply_A, _lib.ref_heff_apply_B):
            f.argtypes = [ctypes.POINTER(_Dims), dp, dp, dp, dp, dp, ctypes.c_int64, ctypes.c_int64, dp]
            f.restype = ctypes.c_int
        _lib.ref_tridiag_lowest.argtypes = [ctypes.c_int, dp, dp, dp, dp]
        _lib.ref_tridiag_lowest.restype = ctypes.c_int
        _lib.ref_lanczos.argtypes = [MATVEC_FN, ctypes.c_void_p, ctypes.c_int64, dp, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_int, dp, dp, ctypes.POINTER(ctypes.c_int), dp, dp, dp]
        _lib.ref_lanczos.restype = ctypes.c_int
        _lib.ref_lanczos_heff.argtypes = [ctypes.POINTER(_Dims), dp, dp, dp, dp, dp, ctypes.c_int, ctypes.c_double,
                                          ctypes.c_int, dp, dp, ctypes.POINTER(ctypes.c_int), dp, dp, dp]
        _lib.ref_lanczos_heff.restype = ctypes.c_int
        _lib.ref_heff_apply_A_z.argtypes = [ctypes.POINTER(_Dims), dp, dp, dp, dp, dp, ctypes.c_int64,
                                            ctypes.c_int64, dp]
        _lib.ref_heff_apply_A_z.restype = ctypes.c_int
        _lib.ref_lanczos_heff_z.argtypes = [ctypes.POINTER(_Dims), dp, dp, dp, dp, dp, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_int, dp, dp, ctypes.POINTER(ctypes.c_int), dp, dp, dp]
        _lib.ref_lanczos_heff_z.restype = ctypes.c_int
        i64 = ctypes.c_int64
        for f in (_lib.ref_env_left, _lib.ref_env_right):
            f.argtypes = [i64, i64, i64, i64, i64, dp, dp, dp, dp]
            f.restype = ctypes.c_int
        _lib.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def dims_of(L, W1, W2, R) -> _Dims:
    mL, kL, mL2 = L.shape
    kL2, d1, d1b, kM = W1.shape
    kM2, d2, d2b, kR = W2.shape
    mR, kR2, mR2 = R.shape
    assert mL == mL2 and kL == kL2 and d1 == d1b and kM == kM2 and d2 == d2b and kR == kR2 and mR == mR2
    return _Dims(mL, d1, d2, mR, kL, kM, kR)


def heff_direct(L, W1, W2, R, psi) -> np.ndarray:
    """The definition (D) summed literally -- tiny sizes only."""
    L, W1, W2, R, psi = map(_c, (L, W1, W2, R, psi))
    D = dims_of(L, W1, W2, R)
    out = np.empty((D.mL, D.d1, D.d2, D.mR))
    lib().ref_heff_direct(ctypes.byref(D), _p(L), _p(W1), _p(W2), _p(R), _p(psi), _p(out))
    return out


def heff_apply(L, W1, W2, R, psi, rows: tuple[int, int] | None = None) -> np.ndarray:
    """Order A (L*psi -> *W1 -> *W2 -> *R); ``rows`` = (a_lo, a_hi) restricts the output rows a'."""
    L, W1, W2, R, psi = map(_c, (L, W1, W2, R, psi))
    D = dims_of(L, W1, W2, R)
    a_lo, a_hi = rows if rows is not None else (0, D.mL)
    out = np.empty((a_hi - a_lo, D.d1, D.d2, D.mR))
    rc = lib().ref_heff_apply_A(ctypes.byref(D), _p(L), _p(W1), _p(W2), _p(R), _p(psi), a_lo, a_hi, _p(out))
    if rc != 0:
        raise RuntimeError(f"ref_heff_apply_A failed: {rc}")
    return out


def heff_apply_B(L, W1, W2, R, psi, cols: tuple[int, int] | None = None) -> np.ndarray:
    """Order B (R*psi -> *W2 -> *W1 -> *L); ``cols`` = (b_lo, b_hi) gives the b'-shard [mL,d1,d2,nb]."""
    L, W1, W2, R, psi = map(_c, (L, W1, W2, R, psi))
    D = dims_of(L, W1, W2, R)
    b_lo, b_hi = cols if cols is not None else (0, D.mR)
    out = np.empty((D.mL, D.d1, D.d2, b_hi - b_lo))
    rc = lib().ref_heff_apply_B(ctypes.byref(D), _p(L), _p(W1), _p(W2), _p(R), _p(psi), b_lo, b_hi, _p(out))
    if rc != 0:
        raise RuntimeError(f"ref_heff_apply_B failed: {rc}")
    return out


def heff_apply_B_cols(L, W1, W2, R, psi, cols) -> np.ndarray:
    """Order B on an arbitrary list of output columns b' (sampled full-size parity): output
    column b' depends on R only through its row R[b', :, :], so the listed rows are moved to
    the front of an otherwise unread R' and ref_heff_apply_B runs on b' in [0, len(cols)).
    Returns [mL, d1, d2, len(cols)].  (Row selection only; the arithmetic is ref_heff_apply_B.)"""
    L, W1, W2, R, psi = map(_c, (L, W1, W2, R, psi))
    cols = [int(c) for c in cols]
    Rp = np.empty_like(R)                 # rows >= len(cols) are never read
    Rp[: len(cols)] = R[cols]
    return heff_apply_B(L, W1, W2, Rp, psi, cols=(0, len(cols)))


def _cz(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _pz(a: np.ndarray):
    assert a.dtype == np.complex128 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def heff_apply_z(L, W1, W2, R, psi, rows: tuple[int, int] | None = None) -> np.ndarray:
    """Complex order A (heff_oracle.c ref_heff_apply_A_z); no conjugation inside (D)."""
    L, W1, W2, R, psi = map(_cz, (L, W1, W2, R, psi))
    D = dims_of(L, W1, W2, R)
    a_lo, a_hi = rows if rows is not None else (0, D.mL)
    out = np.empty((a_hi - a_lo, D.d1, D.d2, D.mR), dtype=np.complex128)
    rc = lib().ref_heff_apply_A_z(ctypes.byref(D), _pz(L), _pz(W1), _pz(W2), _pz(R), _pz(psi), a_lo, a_hi, _pz(out))
    if rc != 0:
        raise RuntimeError(f"ref_heff_apply_A_z failed: {rc}")
    return out


def lanczos_heff_z(L, W1, W2, R, x0, max_iter: int, tol: float = 0.0, converge: bool = False) -> "LanczosResult":
    """Hermitian Lanczos (CGS2, <v,w> = sum conj(v) w) on the complex H_eff, all in C."""
    L, W1, W2, R = map(_cz, (L, W1, W2, R))
    D = dims_of(L, W1, W2, R)
    x0 = _cz(x0)
    e, it = ctypes.c_double(), ctypes.c_int()
    x = np.empty_like(x0)
    al, be, th = np.zeros(max_iter + 1), np.zeros(max_iter + 1), np.zeros(max_iter + 1)
    rc = lib().ref_lanczos_heff_z(ctypes.byref(D), _pz(L), _pz(W1), _pz(W2), _pz(R), _pz(x0), max_iter, tol,
                                  1 if converge else 0, ctypes.byref(e), _pz(x), ctypes.byref(it), _p(al), _p(be),
                                  _p(th))
    return _lanczos_out(rc, e, x, it, al, be, th)


def heff_apply_penalty(L, W1, W2, R, psi, phis, weight: float) -> np.ndarray:
    """H_eff psi + weight * sum_i phi_i <phi_i|psi> -- the excited-state energy penalty
    "projectors onto the previous states ... added to the Hamiltonian times an energy
    penalty" (Sec. 6.2).  phis: [nphi, *psi.shape]."""
    out = heff_apply(L, W1, W2, R, psi)
    for phi in np.asarray(phis, dtype=np.float64):
        out += weight * phi * float(np.sum(phi * psi))
    return out


def heff_apply_sum(terms, psi) -> np.ndarray:
    """sum_t H_eff^(t) psi over (L, W1, W2, R) terms -- an MPO sum "as if they were summed"
    (Sec. 6.2)."""
    out = None
    for (L, W1, W2, R) in terms:
        y = heff_apply(L, W1, W2, R, psi)
        out = y if out is None else out + y
    return out


def env_left(L, A, W) -> np.ndarray:
    """Lout[a',w',a] = sum A[x',s',a'] L[x',w,x] W[w,s',s,w'] A[x,s,a]  (heff_oracle.c ref_env_left)."""
    L, A, W = map(_c, (L, A, W))
    mi, kl, _ = L.shape
    _, d, mo = A.shape
    kr = W.shape[3]
    assert A.shape[0] == mi and W.shape[:3] == (kl, d, d)
    out = np.empty((mo, kr, mo))
    if lib().ref_env_left(mi, d, mo, kl, kr, _p(L), _p(A), _p(W), _p(out)) != 0:
        raise RuntimeError("ref_env_left failed")
    return out


def env_right(R, B, W) -> np.ndarray:
    """Rout[b',w,b] = sum B[b',s',y'] R[y',w',y] W[w,s',s,w'] B[b,s,y]  (heff_oracle.c ref_env_right)."""
    R, B, W = map(_c, (R, B, W))
    mi, kr, _ = R.shape
    mo, d, _ = B.shape
    kl = W.shape[0]
    assert B.shape[2] == mi and W.shape[1:] == (d, d, kr)
    out = np.empty((mo, kl, mo))
    if lib().ref_env_right(mi, d, mo, kl, kr, _p(R), _p(B), _p(W), _p(out)) != 0:
        raise RuntimeError("ref_env_right failed")
    return out


def env_left_rows(L, A, W, rows) -> np.ndarray:
    """Rows a' of env_left, one at a time (sampled checks at full size): the same sum as
    env_left, Lout[a',w',a] = sum A[x',s',a'] L[x',w,x] W[w,s',s,w'] A[x,s,a], contracted
    bra first for a fixed a' (numpy tensor contractions as library steps)."""
    L, A, W = map(_c, (L, A, W))
    out = []
    for ap in rows:
        Y = np.einsum("ys,ywx->swx", A[:, :, ap], L)      # sum_x' A[x',s',a'] L[x',w,x]
        Z = np.einsum("wstv,swx->tvx", W, Y)              # sum_{w,s'} W[w,s',s,w'] Y[s',w,x]
        out.append(np.einsum("tvx,xta->va", Z, A))        # sum_{x,s} Z[s,w',x] A[x,s,a]
    return np.stack(out)


def env_right_rows(R, B, W, rows) -> np.ndarray:
    """Rows b' of env_right, one at a time: Rout[b',w,b] = sum B[b',s',y'] R[y',w',y]
    W[w,s',s,w'] B[b,s,y], contracted bra first for a fixed b'."""
    R, B, W = map(_c, (R, B, W))
    out = []
    for bp in rows:
        Y = np.einsum("sy,yvz->svz", B[bp], R)            # sum_y' B[b',s',y'] R[y',w',y]
        Z = np.einsum("wstv,svz->wtz", W, Y)              # sum_{s',w'} W[w,s',s,w'] Y[s',w',y]
        out.append(np.einsum("wtz,btz->wb", Z, B))        # sum_{s,y} Z[w,s,y] B[b,s,y]
    return np.stack(out)


def tridiag_lowest(alpha, beta):
    alpha = _c(alpha)
    j = alpha.size
    beta = _c(np.append(np.asarray(beta, dtype=np.float64), np.zeros(max(0, j - len(beta)))))
    th = ctypes.c_double()
    y = np.empty(j)
    rc = lib().ref_tridiag_lowest(j, _p(alpha), _p(beta), ctypes.byref(th), _p(y))
    if rc != 0:
        raise RuntimeError("ref_tridiag_lowest failed")
    return th.value, y


class LanczosResult:
    def __init__(self, energy, x, iters, alpha, beta, thetas):
        self.energy, self.x, self.iters, self.alpha, self.beta, self.thetas = energy, x, iters, alpha, beta, thetas


def _lanczos_out(rc, e, x, it, al, be, th):
    if rc == -5:
        raise ValueError("zero initial vector")
    if rc != 0:
        raise RuntimeError(f"ref_lanczos failed: {rc}")
    j = it.value
    return LanczosResult(e.value, x, j, al[:j].copy(), be[:j].copy(), th[:j].copy())


def lanczos(matvec, x0, max_iter: int, tol: float = 0.0, converge: bool = False) -> LanczosResult:
    """Lanczos (CGS2) with a Python matvec callback ``matvec(x) -> H x`` (dense tests)."""
    x0 = _c(x0).ravel()
    n = x0.size

    def cb(_ctx, pin, pout):
        xin = np.ctypeslib.as_array(pin, shape=(n,))
        xout = np.ctypeslib.as_array(pout, shape=(n,))
        xout[:] = matvec(xin.copy())

    fn = MATVEC_FN(cb)
    e, it = ctypes.c_double(), ctypes.c_int()
    x = np.empty(n)
    al, be, th = np.zeros(max_iter + 1), np.zeros(max_iter + 1), np.zeros(max_iter + 1)
    rc = lib().ref_lanczos(fn, None, n, _p(x0), max_iter, tol, 1 if converge else 0, ctypes.byref(e), _p(x),
                           ctypes.byref(it), _p(al), _p(be), _p(th))
    return _lanczos_out(rc, e, x, it, al, be, th)


def lanczos_heff(L, W1, W2, R, x0, max_iter: int, tol: float = 0.0, converge: bool = False) -> LanczosResult:
    """Lanczos (CGS2) on H_eff with the order-A oracle matvec, all in C."""
    L, W1, W2, R = map(_c, (L, W1, W2, R))
    D = dims_of(L, W1, W2, R)
    x0 = _c(x0)
    e, it = ctypes.c_double(), ctypes.c_int()
    x = np.empty_like(x0)
    al, be, th = np.zeros(max_iter + 1), np.zeros(max_iter + 1), np.zeros(max_iter + 1)
    rc = lib().ref_lanczos_heff(ctypes.byref(D), _p(L), _p(W1), _p(W2), _p(R), _p(x0), max_iter, tol,
                                1 if converge else 0, ctypes.byref(e), _p(x), ctypes.byref(it), _p(al), _p(be), _p(th))
    return _lanczos_out(rc, e, x, it, al, be, th)


def heff_dense(L, W1, W2, R) -> np.ndarray:
    """H_eff as an explicit matrix, one oracle matvec per basis vector (tiny sizes only)."""
    D = dims_of(L, W1, W2, R)
    n = D.mL * D.d1 * D.d2 * D.mR
    H = np.empty((n, n))
    shape = (D.mL, D.d1, D.d2, D.mR)
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        H[:, i] = heff_apply(L, W1, W2, R, e.reshape(shape)).ravel()
    return H
