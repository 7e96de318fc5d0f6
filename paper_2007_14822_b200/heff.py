"""Thin ctypes binding of libheff (include/heff.h) -- argument marshalling only.

Every step of H_eff.psi and of the Lanczos solver runs in libheff's CUDA kernels; this
module passes torch device pointers, the current CUDA stream and plain sizes across the
C ABI.  There is no CPU fallback: if libheff.so is missing or the device is not a B200
(sm_100a) the calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libheff.so"

HEFF_OK, HEFF_EINVAL, HEFF_ENOMEM, HEFF_ECUDA, HEFF_ENCCL, HEFF_EZERO, HEFF_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
HEFF_ENOCONV = -7
OPT_GEMM_PATH, OPT_LAST_KERNEL_COUNT, OPT_MPO_NNZ, OPT_PROFILE, OPT_TOTAL_LAUNCHES, OPT_SPARSE_KBLOCKS = 1, 2, 3, 4, 5, 6
OPT_LANCZOS_RESERVE = 8
OPT_FUSED_GATHER = 7
OPT_FORCE_ALLGATHER, OPT_COMM_STATE = 9, 10


class HeffError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libheff error {code}: {msg}")
        self.code = code


class HeffZeroVector(HeffError, ValueError):
    pass


class _Dims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("mL", "d1", "d2", "mR", "kL", "kM", "kR")]


class _Dist(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("nccl_uid", ctypes.c_void_p),
                ("b_lo", ctypes.c_int64), ("b_hi", ctypes.c_int64)]


class _EnvDims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("mi", "d", "mo", "kl", "kr")]


class _EnvQN(ctypes.Structure):
    _fields_ = [(n, ctypes.POINTER(ctypes.c_int)) for n in ("q_in", "q_out", "qs", "cl", "cr")]


class _QN(ctypes.Structure):
    _fields_ = [(n, ctypes.POINTER(ctypes.c_int)) for n in ("qa", "qb", "qs1", "qs2", "cL", "cM", "cR")]


class _Trunc(ctypes.Structure):
    _fields_ = [("cutoff", ctypes.c_double), ("maxdim", ctypes.c_int64), ("mindim", ctypes.c_int64)]


class _LanczosOpts(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int), ("mode", ctypes.c_int), ("tol", ctypes.c_double),
                ("alpha_out", ctypes.c_void_p), ("beta_out", ctypes.c_void_p), ("theta_out", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libheff.so (built by __graft_entry__.build() / paper_2007_14822_b200/build.py)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, ip = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.heff_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(_Dims), vp, vp, vp, vp, ctypes.POINTER(_Dist), vp]
        L.heff_apply.argtypes = [vp, vp, vp, vp]
        L.heff_apply_host.argtypes = [vp, vp, vp, vp]
        L.heff_apply_blocked.argtypes = [vp, vp, vp, vp]
        L.lanczos_ground.argtypes = [vp, vp, ctypes.POINTER(_LanczosOpts), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ip), ctypes.POINTER(ctypes.c_double), vp]
        L.heff_destroy.argtypes = [vp]
        L.heff_last_error.restype = ctypes.c_char_p
        L.heff_workspace_bytes.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(_Dist)]
        L.heff_workspace_bytes.restype = ctypes.c_size_t
        L.heff_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.heff_set_option.argtypes = [vp, ip, i64]
        L.heff_get_option.argtypes = [vp, ip, ctypes.POINTER(i64)]
        L.heff_last_timings.argtypes = [vp] + [ctypes.POINTER(ctypes.c_float)] * 4
        L.heff_relayout_blocked.argtypes = [vp, vp, i64, i64, ip, vp]
        L.heff_create_sum.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp), ip]
        L.heff_create_z.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(_Dims), vp, vp, vp, vp, ctypes.POINTER(_Dist), vp]
        L.heff_set_penalty.argtypes = [vp, vp, ip, ctypes.c_double, vp]
        dp = ctypes.POINTER(ctypes.c_double)
        L.heff_tridiag_lowest.argtypes = [ip, dp, dp, dp, dp]
        L.heff_tridiag_lowest_check.argtypes = [ip, dp, dp, dp, dp]
        L.heff_set_qn.argtypes = [vp, ctypes.POINTER(_QN)]
        L.heff_gemm.argtypes = [i64, i64, i64, vp, i64, vp, i64, ip, vp, i64, ip, ip, vp]
        L.heff_env_update_left.argtypes = [ctypes.POINTER(_EnvDims), vp, vp, vp, vp, vp]
        L.heff_env_update_right.argtypes = [ctypes.POINTER(_EnvDims), vp, vp, vp, vp, vp]
        L.heff_env_update_left_qn.argtypes = [ctypes.POINTER(_EnvDims), vp, vp, vp, vp, ctypes.POINTER(_EnvQN), vp]
        L.heff_env_update_right_qn.argtypes = [ctypes.POINTER(_EnvDims), vp, vp, vp, vp, ctypes.POINTER(_EnvQN), vp]
        L.heff_svd_split.argtypes = [i64, i64, vp, ctypes.POINTER(_Trunc), ip, vp, vp, vp, ctypes.POINTER(i64),
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ip), vp]
        L.heff_truncate_spectrum.argtypes = [vp, i64, ctypes.POINTER(_Trunc), ctypes.POINTER(i64),
                                             ctypes.POINTER(ctypes.c_double)]
        L.heff_svd_split_qn.argtypes = [i64, i64, vp, vp, vp, ctypes.POINTER(_Trunc), ip, vp, vp, vp, vp, vp,
                                        ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ip), vp]
        L.heff_release_caches.argtypes = []
        L.heff_dot.argtypes = [i64, vp, vp, ctypes.POINTER(ctypes.c_double), vp]
        for f in ("heff_dot", "heff_env_update_left_qn", "heff_env_update_right_qn", "heff_release_caches", "heff_svd_split_qn", "heff_apply_blocked", "heff_truncate_spectrum", "heff_svd_split", "heff_create", "heff_apply", "heff_apply_host", "lanczos_ground", "heff_destroy",
                  "heff_nccl_unique_id", "heff_set_option", "heff_get_option", "heff_last_timings",
                  "heff_relayout_blocked", "heff_create_sum", "heff_set_penalty", "heff_env_update_left",
                  "heff_env_update_right", "heff_tridiag_lowest", "heff_gemm", "heff_set_qn", "heff_create_z",
                  "heff_tridiag_lowest_check"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTED = ("heff_create", "heff_apply", "heff_apply_host", "lanczos_ground", "heff_destroy", "heff_last_error",
            "heff_workspace_bytes", "heff_nccl_unique_id", "heff_set_option", "heff_get_option", "heff_last_timings",
            "heff_relayout_blocked", "heff_create_sum", "heff_set_penalty", "heff_env_update_left",
            "heff_env_update_right", "heff_tridiag_lowest", "heff_gemm", "heff_set_qn", "heff_create_z",
            "heff_svd_split", "heff_truncate_spectrum", "heff_apply_blocked", "heff_svd_split_qn",
            "heff_release_caches", "heff_env_update_left_qn", "heff_env_update_right_qn", "heff_dot",
            "heff_tridiag_lowest_check")


def _check(rc: int):
    if rc != HEFF_OK:
        msg = lib().heff_last_error().decode(errors="replace")
        if rc == HEFF_EZERO:
            raise HeffZeroVector(rc, msg)
        raise HeffError(rc, msg)


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dev(t: torch.Tensor, name: str, cplx: bool = False) -> torch.Tensor:
    dt = torch.complex128 if cplx else torch.float64
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dt and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous {dt} CUDA tensor")
    return t


def relayout_blocked(src: torch.Tensor, P: int, stream=None) -> torch.Tensor:
    """[P][rows][nb] -> [rows][P*nb] on the device (libheff's post-all-gather map)."""
    _dev(src, "src")
    _, rows, nb = src.shape
    dst = torch.empty((rows, P * nb), dtype=torch.float64, device=src.device)
    _check(lib().heff_relayout_blocked(src.data_ptr(), dst.data_ptr(), rows, nb, P, _stream(stream)))
    return dst


def gemm(A: torch.Tensor, B: torch.Tensor, b_kmajor: bool = False, C: torch.Tensor | None = None,
         accumulate: bool = False, path: int = 0, stream=None) -> torch.Tensor:
    """C (+)= A @ B (B [K,N]) or A @ B.T (b_kmajor, B [N,K]) on libheff's FP64 DMMA GEMM."""
    _dev(A, "A")
    _dev(B, "B")
    M, K = A.shape
    N = B.shape[0] if b_kmajor else B.shape[1]
    if (B.shape[1] if b_kmajor else B.shape[0]) != K:
        raise ValueError("inner dimensions differ")
    if C is None:
        C = torch.zeros((M, N), dtype=torch.float64, device=A.device)
    _dev(C, "C")
    _check(lib().heff_gemm(M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), int(b_kmajor),
                           C.data_ptr(), C.stride(0), int(accumulate), int(path), _stream(stream)))
    return C


def tridiag_lowest(alpha, beta):
    """libheff's host QL solve of the Lanczos tridiagonal (no GPU needed)."""
    import numpy as np
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    j = a.size
    b = np.ascontiguousarray(np.append(np.asarray(beta, dtype=np.float64)[: max(0, j - 1)], 0.0), dtype=np.float64)
    y = np.empty(j)
    th = ctypes.c_double()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(lib().heff_tridiag_lowest(j, a.ctypes.data_as(dp), b.ctypes.data_as(dp), ctypes.byref(th),
                                     y.ctypes.data_as(dp)))
    return th.value, y


def tridiag_lowest_check(alpha, beta):
    """libheff's per-step Lanczos check (Sturm bisection + inverse iteration; no GPU needed):
    (theta, |y_last|)."""
    import numpy as np
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    j = a.size
    b = np.ascontiguousarray(np.append(np.asarray(beta, dtype=np.float64)[: max(0, j - 1)], 0.0), dtype=np.float64)
    th, yl = ctypes.c_double(), ctypes.c_double()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(lib().heff_tridiag_lowest_check(j, a.ctypes.data_as(dp), b.ctypes.data_as(dp), ctypes.byref(th),
                                           ctypes.byref(yl)))
    return th.value, abs(yl.value)


def _env_qn(qn):
    import numpy as np
    arrs = [np.ascontiguousarray(qn[k], dtype=np.int32) for k in ("q_in", "q_out", "qs", "cl", "cr")]
    return arrs, _EnvQN(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for a in arrs])


def env_update_left(L: torch.Tensor, A: torch.Tensor, W: torch.Tensor, stream=None, qn: dict | None = None) -> torch.Tensor:
    """Lout[a',w',a] = sum A[x',s',a'] L[x',w,x] W[w,s',s,w'] A[x,s,a] (heff_env_update_left);
    qn = dict(q_in, q_out, qs, cl, cr) selects the U(1) schedule (heff_env_update_left_qn)."""
    for t, n in ((L, "L"), (A, "A"), (W, "W")):
        _dev(t, n)
    mi, kl, _ = L.shape
    _, d, mo = A.shape
    kr = W.shape[3]
    if tuple(L.shape) != (mi, kl, mi) or tuple(A.shape) != (mi, d, mo) or tuple(W.shape) != (kl, d, d, kr):
        raise ValueError("expected L[mi,kl,mi], A[mi,d,mo], W[kl,d,d,kr]")
    out = torch.empty((mo, kr, mo), dtype=torch.float64, device=L.device)
    if qn is not None:
        keep, q = _env_qn(qn)
        _check(lib().heff_env_update_left_qn(ctypes.byref(_EnvDims(mi, d, mo, kl, kr)), L.data_ptr(), A.data_ptr(),
                                             W.data_ptr(), out.data_ptr(), ctypes.byref(q), _stream(stream)))
        return out
    _check(lib().heff_env_update_left(ctypes.byref(_EnvDims(mi, d, mo, kl, kr)), L.data_ptr(), A.data_ptr(),
                                      W.data_ptr(), out.data_ptr(), _stream(stream)))
    return out


def env_update_right(R: torch.Tensor, B: torch.Tensor, W: torch.Tensor, stream=None, qn: dict | None = None) -> torch.Tensor:
    """Rout[b',w,b] = sum B[b',s',y'] R[y',w',y] W[w,s',s,w'] B[b,s,y] (heff_env_update_right);
    qn = dict(q_in, q_out, qs, cl, cr) selects the U(1) schedule (heff_env_update_right_qn)."""
    for t, n in ((R, "R"), (B, "B"), (W, "W")):
        _dev(t, n)
    mi, kr, _ = R.shape
    mo, d, _ = B.shape
    kl = W.shape[0]
    if tuple(R.shape) != (mi, kr, mi) or tuple(B.shape) != (mo, d, mi) or tuple(W.shape) != (kl, d, d, kr):
        raise ValueError("expected R[mi,kr,mi], B[mo,d,mi], W[kl,d,d,kr]")
    out = torch.empty((mo, kl, mo), dtype=torch.float64, device=R.device)
    if qn is not None:
        keep, q = _env_qn(qn)
        _check(lib().heff_env_update_right_qn(ctypes.byref(_EnvDims(mi, d, mo, kl, kr)), R.data_ptr(), B.data_ptr(),
                                              W.data_ptr(), out.data_ptr(), ctypes.byref(q), _stream(stream)))
        return out
    _check(lib().heff_env_update_right(ctypes.byref(_EnvDims(mi, d, mo, kl, kr)), R.data_ptr(), B.data_ptr(),
                                       W.data_ptr(), out.data_ptr(), _stream(stream)))
    return out


@dataclass
class SplitResult:
    Q: torch.Tensor       # dir 0: U [M, n]; dir 1: V^T [n, N]
    S: torch.Tensor       # all min(M, N) singular values, descending
    C: torch.Tensor       # dir 0: S V^T [n, N]; dir 1: U S [M, n]
    n: int
    trunc_err: float
    sweeps: int


def svd_split(psi: torch.Tensor, cutoff: float = 0.0, maxdim: int = 0, mindim: int = 1, direction: int = 0,
              stream=None) -> SplitResult:
    """Two-site split (heff_svd_split): psi [mL, d1, d2, mR] is viewed as Psi[(a s1), (s2 b)]
    (a 2-D tensor is taken as Psi itself) and factored by the truncated SVD."""
    _dev(psi, "psi")
    if psi.dim() == 4:
        mL, d1, d2, mR = psi.shape
        M, N = mL * d1, d2 * mR
    elif psi.dim() == 2:
        M, N = psi.shape
    else:
        raise ValueError("psi must be [mL, d1, d2, mR] or [M, N]")
    kmax = min(M, N) if maxdim <= 0 else min(M, N, maxdim)
    Q = torch.empty(max(1, M * kmax if direction == 0 else kmax * N), dtype=torch.float64, device=psi.device)
    C = torch.empty(max(1, kmax * N if direction == 0 else M * kmax), dtype=torch.float64, device=psi.device)
    S = torch.empty(min(M, N), dtype=torch.float64, device=psi.device)
    n = ctypes.c_int64(0)
    err = ctypes.c_double(0.0)
    sw = ctypes.c_int(0)
    tr = _Trunc(float(cutoff), int(maxdim), int(mindim))
    _check(lib().heff_svd_split(M, N, psi.data_ptr(), ctypes.byref(tr), int(direction), Q.data_ptr(), S.data_ptr(),
                                C.data_ptr(), ctypes.byref(n), ctypes.byref(err), ctypes.byref(sw), _stream(stream)))
    k = n.value
    if direction == 0:
        Qv, Cv = Q[: M * k].view(M, k), C[: k * N].view(k, N)
    else:
        Qv, Cv = Q[: k * N].view(k, N), C[: M * k].view(M, k)
    return SplitResult(Qv, S, Cv, k, err.value, sw.value)


@dataclass
class SplitQNResult(SplitResult):
    Sk: torch.Tensor = None   # kept values in new-bond order
    qk: list = None           # charges of the new bond (nondecreasing)


def psi_row_col_charges(qa, qs1, qs2, qb):
    """Charges of Psi's rows (a s1) and columns (s2 b) in the convention of DESIGN.md R18 (a
    bond carries the total charge to its left): q(a) + q(s1) and q(b) - q(s2)."""
    qrow = [int(x) + int(y) for x in qa for y in qs1]
    qcol = [int(b) - int(y) for y in qs2 for b in qb]
    return qrow, qcol


def svd_split_qn(psi: torch.Tensor, qrow, qcol, cutoff: float = 0.0, maxdim: int = 0, mindim: int = 1,
                 direction: int = 0, stream=None) -> SplitQNResult:
    """U(1) two-site split (heff_svd_split_qn): Psi's rows/columns carry charges qrow/qcol
    (host int sequences); one dense split per charge block, one global truncation."""
    _dev(psi, "psi")
    if psi.dim() == 4:
        mL, d1, d2, mR = psi.shape
        M, N = mL * d1, d2 * mR
    else:
        M, N = psi.shape
    qr = (ctypes.c_int * M)(*[int(v) for v in qrow])
    qc = (ctypes.c_int * N)(*[int(v) for v in qcol])
    if len(qrow) != M or len(qcol) != N:
        raise ValueError("charge arrays must match Psi's shape")
    kmax = min(M, N) if maxdim <= 0 else min(M, N, maxdim)
    Q = torch.empty(max(1, M * kmax if direction == 0 else kmax * N), dtype=torch.float64, device=psi.device)
    C = torch.empty(max(1, kmax * N if direction == 0 else M * kmax), dtype=torch.float64, device=psi.device)
    S = torch.empty(min(M, N), dtype=torch.float64, device=psi.device)
    Sk = torch.empty(max(1, kmax), dtype=torch.float64, device=psi.device)
    qk = (ctypes.c_int * max(1, kmax))()
    n = ctypes.c_int64(0)
    err = ctypes.c_double(0.0)
    sw = ctypes.c_int(0)
    tr = _Trunc(float(cutoff), int(maxdim), int(mindim))
    _check(lib().heff_svd_split_qn(M, N, psi.data_ptr(), qr, qc, ctypes.byref(tr), int(direction), Q.data_ptr(),
                                   S.data_ptr(), Sk.data_ptr(), qk, C.data_ptr(), ctypes.byref(n), ctypes.byref(err),
                                   ctypes.byref(sw), _stream(stream)))
    k = n.value
    if direction == 0:
        Qv, Cv = Q[: M * k].view(M, k), C[: k * N].view(k, N)
    else:
        Qv, Cv = Q[: k * N].view(k, N), C[: M * k].view(M, k)
    return SplitQNResult(Qv, S, Cv, k, err.value, sw.value, Sk[:k], list(qk)[:k])


def dot(x: torch.Tensor, y: torch.Tensor, stream=None) -> float:
    """x . y through libheff's Lanczos reduction kernels (heff_dot)."""
    _dev(x, "x")
    _dev(y, "y")
    if x.numel() != y.numel():
        raise ValueError("x and y must have the same length")
    r = ctypes.c_double(0.0)
    _check(lib().heff_dot(x.numel(), x.data_ptr(), y.data_ptr(), ctypes.byref(r), _stream(stream)))
    return r.value


def release_caches():
    """Free libheff's per-thread split / environment / GEMM workspaces (heff_release_caches)."""
    _check(lib().heff_release_caches())


def truncate_spectrum(s, cutoff: float = 0.0, maxdim: int = 0, mindim: int = 1) -> tuple[int, float]:
    """libheff's host-side truncation rule (heff_truncate_spectrum) on descending values."""
    import numpy as np
    a = np.ascontiguousarray(np.asarray(s, dtype=np.float64))
    n = ctypes.c_int64(0)
    err = ctypes.c_double(0.0)
    _check(lib().heff_truncate_spectrum(a.ctypes.data, a.size, ctypes.byref(_Trunc(float(cutoff), int(maxdim), int(mindim))),
                                        ctypes.byref(n), ctypes.byref(err)))
    return n.value, err.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().heff_nccl_unique_id(buf))
    return buf.raw


@dataclass
class LanczosResult:
    energy: float
    iters: int
    resid: float
    alpha: list
    beta: list
    thetas: list


class Heff:
    """A libheff plan: H_eff for fixed (L, W1, W2, R).

    dist = None: single GPU, order A.  dist = dict(nranks, rank, b_lo, b_hi, uid=None|bytes):
    this rank's b'-shard (order B); R must then hold only rows [b_lo, b_hi).
    The tensors are borrowed: keep them alive and unmodified while the plan lives.
    """

    def __init__(self, L, W1, W2, R, dist: dict | None = None, stream=None):
        self.cplx = isinstance(L, torch.Tensor) and L.is_complex()
        for t, n in ((L, "L"), (W1, "W1"), (W2, "W2"), (R, "R")):
            _dev(t, n, self.cplx)
        if L.dim() != 3 or W1.dim() != 4 or W2.dim() != 4 or R.dim() != 3:
            raise ValueError("expected L[mL,kL,mL], W1[kL,d1,d1,kM], W2[kM,d2,d2,kR], R[nb,kR,mR]")
        mL, kL, _ = L.shape
        _, d1, _, kM = W1.shape
        _, d2, _, kR = W2.shape
        mR = R.shape[2]
        nb = (dist["b_hi"] - dist["b_lo"]) if dist is not None else mR
        if (tuple(L.shape) != (mL, kL, mL) or tuple(W1.shape) != (kL, d1, d1, kM)
                or tuple(W2.shape) != (kM, d2, d2, kR) or tuple(R.shape) != (nb, kR, mR)):
            raise ValueError(f"inconsistent shapes L{tuple(L.shape)} W1{tuple(W1.shape)} W2{tuple(W2.shape)} "
                             f"R{tuple(R.shape)}")
        self.dims = dict(mL=mL, d1=d1, d2=d2, mR=mR, kL=kL, kM=kM, kR=kR)
        self._keep = (L, W1, W2, R)
        self._cdims = _Dims(mL, d1, d2, mR, kL, kM, kR)
        self.dist = dist
        pdist = None
        self._uid = None
        if dist is not None:
            uid = dist.get("uid")
            self._uid = ctypes.create_string_buffer(uid, 128) if uid is not None else None
            self._cdist = _Dist(dist["nranks"], dist["rank"],
                                ctypes.cast(self._uid, ctypes.c_void_p) if self._uid is not None else None,
                                dist["b_lo"], dist["b_hi"])
            pdist = ctypes.byref(self._cdist)
            self.nb = dist["b_hi"] - dist["b_lo"]
        else:
            self.nb = mR
        h = ctypes.c_void_p()
        create = lib().heff_create_z if self.cplx else lib().heff_create
        _check(create(ctypes.byref(h), ctypes.byref(self._cdims), L.data_ptr(), W1.data_ptr(), W2.data_ptr(),
                      R.data_ptr(), pdist, _stream(stream)))
        self._h = h

    def set_penalty(self, phis: torch.Tensor | None, weight: float = 0.0, stream=None):
        """Energy penalty: matvec becomes H psi + weight * sum_i phi_i <phi_i|psi>.
        phis: [nphi, *psi_shape] float64 CUDA tensor (copied), or None to remove."""
        if phis is None:
            _check(lib().heff_set_penalty(self._h, None, 0, 0.0, _stream(stream)))
            return
        _dev(phis, "phis")
        n = 1
        for x in self.psi_shape:
            n *= x
        if phis.numel() % n:
            raise ValueError("phis must hold whole psi-shaped vectors")
        _check(lib().heff_set_penalty(self._h, phis.data_ptr(), phis.numel() // n, float(weight), _stream(stream)))

    def set_qn(self, qn: dict | None):
        """Declare U(1) charges (keys qa, qb, qs1, qs2, cL, cM, cR; see heff.h) so the GEMMs
        skip k-blocks that vanish by symmetry; None returns to dense."""
        if qn is None:
            _check(lib().heff_set_qn(self._h, None))
            return
        import numpy as np
        arrs = {k: np.ascontiguousarray(qn[k], dtype=np.int32) for k in ("qa", "qb", "qs1", "qs2", "cL", "cM", "cR")}
        c = _QN(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for a in arrs.values()])
        _check(lib().heff_set_qn(self._h, ctypes.byref(c)))

    # -- shapes
    @property
    def psi_shape(self):
        d = self.dims
        return (d["mL"], d["d1"], d["d2"], d["mR"])

    @property
    def lanczos_len(self) -> int:
        """Entries of lanczos_ground's vector: the shard on communicating sharded plans, else
        the full psi (complex plans: complex entries)."""
        d = self.dims
        comm = self.dist is not None and self.dist.get("uid") is not None
        return d["mL"] * d["d1"] * d["d2"] * (self.nb if comm else d["mR"])

    @property
    def out_shape(self):
        d = self.dims
        return (d["mL"], d["d1"], d["d2"], self.nb)

    def apply(self, psi: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        cplx = getattr(self, "cplx", False)
        _dev(psi, "psi", cplx)
        if out is None:
            out = torch.empty(self.out_shape, dtype=psi.dtype, device=psi.device)
        _dev(out, "out", cplx)
        n_in = self.dims["mL"] * self.dims["d1"] * self.dims["d2"] * self.dims["mR"]
        if psi.numel() != n_in or out.numel() != n_in // self.dims["mR"] * self.nb:
            raise ValueError(f"psi must have {self.psi_shape} elements and out {self.out_shape}")
        _check(lib().heff_apply(self._h, psi.data_ptr(), out.data_ptr(), _stream(stream)))
        return out

    def apply_blocked(self, psi_blocked: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Gather-fused matvec of a b'-sharded plan (heff_apply_blocked): psi_blocked is the
        blocked all-gather layout [P, mL*d1*d2, nb]; returns this plan's out shard."""
        _dev(psi_blocked, "psi_blocked")
        d = self.dims
        if psi_blocked.numel() != d["mL"] * d["d1"] * d["d2"] * d["mR"]:
            raise ValueError(f"psi_blocked must hold P * mL*d1*d2 * nb = {d['mL'] * d['d1'] * d['d2'] * d['mR']} "
                             f"doubles, got {psi_blocked.numel()}")
        if out is None:
            out = torch.empty(self.out_shape, dtype=torch.float64, device=psi_blocked.device)
        _dev(out, "out")
        if out.numel() != d["mL"] * d["d1"] * d["d2"] * self.nb:
            raise ValueError(f"out must have {self.out_shape} elements")
        _check(lib().heff_apply_blocked(self._h, psi_blocked.data_ptr(), out.data_ptr(), _stream(stream)))
        return out

    def apply_host(self, psi_host: torch.Tensor, out_host: torch.Tensor, stream=None) -> torch.Tensor:
        """End-to-end entry: host buffers in and out (copies happen inside libheff)."""
        assert psi_host.device.type == "cpu" and out_host.device.type == "cpu"
        dt = torch.complex128 if getattr(self, "cplx", False) else torch.float64
        assert psi_host.dtype == dt and out_host.dtype == dt
        assert psi_host.is_contiguous() and out_host.is_contiguous()
        d = self.dims
        if psi_host.numel() != d["mL"] * d["d1"] * d["d2"] * d["mR"] or \
                out_host.numel() != d["mL"] * d["d1"] * d["d2"] * self.nb:
            raise ValueError(f"psi_host must have {self.psi_shape} elements and out_host {self.out_shape}")
        _check(lib().heff_apply_host(self._h, psi_host.data_ptr(), out_host.data_ptr(), _stream(stream)))
        return out_host

    def lanczos_ground(self, psi: torch.Tensor, max_iter: int, tol: float = 0.0, converge: bool = False,
                       stream=None, thetas: bool = False) -> LanczosResult:
        """psi: start vector (overwritten with the normalised Ritz vector): the full vector
        [mL, d1, d2, mR], or this rank's shard [mL, d1, d2, nb] on a communicating sharded plan.
        thetas: also return the lowest Ritz value of every step (theta_out; a fixed-step run
        without it solves only the last step's tridiagonal problem)."""
        _dev(psi, "psi", getattr(self, "cplx", False))
        if psi.numel() != self.lanczos_len:
            raise ValueError(f"psi must have {self.lanczos_len} entries for this plan, got {psi.numel()}")
        a = (ctypes.c_double * max_iter)()
        b = (ctypes.c_double * max_iter)()
        th = (ctypes.c_double * max_iter)()
        o = _LanczosOpts(max_iter, 1 if converge else 0, tol, ctypes.cast(a, ctypes.c_void_p),
                         ctypes.cast(b, ctypes.c_void_p), ctypes.cast(th, ctypes.c_void_p) if thetas else None)
        e, it, r = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
        _check(lib().lanczos_ground(self._h, psi.data_ptr(), ctypes.byref(o), ctypes.byref(e), ctypes.byref(it),
                                    ctypes.byref(r), _stream(stream)))
        j = it.value
        return LanczosResult(e.value, j, r.value, list(a[:j]), list(b[:j]), list(th[:j]) if thetas else [])

    def set_option(self, opt: int, value: int):
        _check(lib().heff_set_option(self._h, opt, int(value)))

    def get_option(self, opt: int) -> int:
        v = ctypes.c_int64()
        _check(lib().heff_get_option(self._h, opt, ctypes.byref(v)))
        return v.value

    def last_timings(self):
        f = [ctypes.c_float() for _ in range(4)]
        _check(lib().heff_last_timings(self._h, *[ctypes.byref(x) for x in f]))
        return tuple(x.value for x in f)

    def close(self):
        if getattr(self, "_h", None):
            lib().heff_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class HeffSum(Heff):
    """sum_t H_eff^(t) over term plans ("as if they were summed").  The terms
    must share mL, d1, d2, mR and stay alive while the sum is used."""

    def __init__(self, terms: list):
        if not terms:
            raise ValueError("need at least one term")
        self._terms = list(terms)
        self.dims = dict(terms[0].dims)
        self.cplx = False
        self.dist = None
        self.nb = self.dims["mR"]
        arr = (ctypes.c_void_p * len(terms))(*[t._h.value for t in terms])
        h = ctypes.c_void_p()
        _check(lib().heff_create_sum(ctypes.byref(h), arr, len(terms)))
        self._h = h


def workspace_bytes(dims: dict, dist: dict | None = None) -> int:
    cd = _Dims(*(dims[k] for k in ("mL", "d1", "d2", "mR", "kL", "kM", "kR")))
    pd = None
    if dist is not None:
        pd = ctypes.byref(_Dist(dist["nranks"], dist["rank"], None, dist["b_lo"], dist["b_hi"]))
    return int(lib().heff_workspace_bytes(ctypes.byref(cd), pd))
