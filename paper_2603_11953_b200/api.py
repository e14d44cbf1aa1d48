"""Python mirror of the reference's thin-SVD interface, executed by the B200
C-ABI library (include/mpsvd.h).

Names, argument meaning and error behaviour follow the reference
(proj/include/mpsvd/thinsvd.hpp:50-59, proj/include/mpsvd.h:116-134): the
same exception classes carrying the same 1-based payloads, the same result
fields (U, sigma, V, phase times that partition the total, sync events,
gram blocks). Matrices are numpy arrays in column-major (Fortran) order.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import ExecInfo, lib

# ---------------------------------------------------------------------------
# status codes / errors (proj/include/mpsvd.h:25-37, types.hpp:35-119)

OK = 0


class MpsvdError(RuntimeError):
    status = 10

    def __init__(self, message="", index=0, value=0.0):
        super().__init__(message)
        self.index = int(index)
        self.value = float(value)


class InvalidArgument(MpsvdError):
    status = 1


class NotPositiveDefiniteError(MpsvdError):
    status = 2

    @property
    def pivot(self):
        return self.index


class NoConvergenceError(MpsvdError):
    status = 3


class ZeroColumnError(MpsvdError):
    status = 4


class ZeroDivisorError(MpsvdError):
    status = 5


class CastOverflowError(MpsvdError):
    status = 6


class TinySingularValueError(MpsvdError):
    status = 7


class InfeasibleError(MpsvdError):
    status = 8


class IoError(MpsvdError):
    status = 9


class InternalError(MpsvdError):
    status = 10


_BY_STATUS = {c.status: c for c in (InvalidArgument, NotPositiveDefiniteError, NoConvergenceError, ZeroColumnError,
                                   ZeroDivisorError, CastOverflowError, TinySingularValueError, InfeasibleError,
                                   IoError, InternalError)}


def _check(st: int, value: float = 0.0):
    if st != OK:
        msg = lib.mpsvd_last_error_message().decode()
        idx = lib.mpsvd_last_error_index()
        raise _BY_STATUS.get(st, MpsvdError)(msg, idx, value)


class Precision(enum.IntEnum):
    WORKING = 0  # binary32
    HIGHER = 1   # binary64


class EigensolverChoice(enum.IntEnum):
    TWOSIDED_JACOBI = 0
    GRAM_CHOL_SVD = 1
    ONESIDED_JACOBI_GRAM = 2


def device_available() -> bool:
    return bool(lib.mpsvd_device_available())


def fp64_peak_tflops(device: int = 0) -> float:
    return float(lib.mpsvd_fp64_peak_tflops(device))


# ---------------------------------------------------------------------------
class Matrix:
    """Owning handle to an ``mpsvd_matrix`` (host, column-major, pinned when large)."""

    def __init__(self, rows: int, cols: int, prec: Precision):
        h = C.c_void_p()
        _check(lib.mpsvd_matrix_create(rows, cols, int(prec), C.byref(h)))
        self._h = h
        self._own = True

    @classmethod
    def _borrow(cls, handle):
        self = cls.__new__(cls)
        self._h = C.c_void_p(handle)
        self._own = False
        return self

    @classmethod
    def _adopt(cls, handle):
        """Take ownership of a matrix the library created (e.g. CholQR's Q, R)."""
        self = cls.__new__(cls)
        self._h = C.c_void_p(handle)
        self._own = True
        return self

    @classmethod
    def from_numpy(cls, a: np.ndarray) -> "Matrix":
        a = np.asarray(a)
        prec = Precision.WORKING if a.dtype == np.float32 else Precision.HIGHER
        m, n = a.shape
        self = cls(m, n, prec)
        self.numpy()[...] = a
        return self

    def __del__(self):
        if getattr(self, "_own", False) and self._h:
            lib.mpsvd_matrix_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def rows(self) -> int:
        return lib.mpsvd_matrix_rows(self._h)

    @property
    def cols(self) -> int:
        return lib.mpsvd_matrix_cols(self._h)

    @property
    def precision(self) -> Precision:
        return Precision(lib.mpsvd_matrix_precision(self._h))

    def get(self, i: int, j: int) -> float:
        v = C.c_double()
        _check(lib.mpsvd_matrix_get(self._h, i, j, C.byref(v)))
        return v.value

    def set(self, i: int, j: int, value: float) -> None:
        _check(lib.mpsvd_matrix_set(self._h, i, j, float(value)))

    def bitwise_equal(self, other: "Matrix") -> bool:
        return bool(lib.mpsvd_matrix_bitwise_equal(self._h, other._h))

    def write_file(self, path: str) -> None:
        """Text wire format (mpsvd_matrix_write_file; proj/src/io.cpp)."""
        _check(lib.mpsvd_matrix_write_file(str(path).encode(), self._h))

    @classmethod
    def read_file(cls, path: str) -> "Matrix":
        """Parse the text wire format (mpsvd_matrix_read_file); IoError-backed
        failures raise MpsvdError with status MPSVD_ERR_IO."""
        h = C.c_void_p()
        _check(lib.mpsvd_matrix_read_file(str(path).encode(), C.byref(h)))
        return cls._adopt(h.value)

    def numpy(self) -> np.ndarray:
        """Zero-copy column-major view of the storage (valid while self lives)."""
        m, n = self.rows, self.cols
        dt = np.float32 if self.precision == Precision.WORKING else np.float64
        if m * n == 0:
            return np.zeros((m, n), dt, order="F")
        ptr = lib.mpsvd_matrix_data(self._h)
        ct = C.c_float if dt == np.float32 else C.c_double
        buf = (ct * (m * n)).from_address(ptr)
        return np.ndarray((m, n), dtype=dt, buffer=buf, order="F")


@dataclass
class PhaseTimes:
    gram: float = 0.0
    eigen: float = 0.0
    compute_u: float = 0.0
    overlap: float = 0.0
    total: float = 0.0


@dataclass
class ThinSvdResult:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    times: PhaseTimes = field(default_factory=PhaseTimes)
    gram_sync_events: int = 0
    gram_blocks: int = 0
    qr_baseline: bool = False
    jacobi_sweeps: int = 0
    jacobi_rotations: int = 0
    eigensolver: int = 0  # EigensolverChoice of the call (thinsvd.hpp ThinSvdResult::eigensolver)


class _ResultOwner:
    """Keeps an mpsvd_svd_result alive while numpy views of its U / V exist."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        if self.handle:
            lib.mpsvd_svd_destroy(self.handle)
            self.handle = None


def _view(mat_handle, owner) -> np.ndarray:
    m, n = lib.mpsvd_matrix_rows(mat_handle), lib.mpsvd_matrix_cols(mat_handle)
    f32 = lib.mpsvd_matrix_precision(mat_handle) == Precision.WORKING
    dt, ct = (np.float32, C.c_float) if f32 else (np.float64, C.c_double)
    if m * n == 0:
        return np.zeros((m, n), dt, order="F")
    buf = (ct * (m * n)).from_address(lib.mpsvd_matrix_data(mat_handle))
    buf._owner = owner  # the array's base keeps the result alive
    return np.ndarray((m, n), dtype=dt, buffer=buf, order="F")


def _result(r) -> ThinSvdResult:
    """Zero-copy: U and V are views of the library's (page-locked) result buffers."""
    owner = _ResultOwner(r)
    u = _view(lib.mpsvd_svd_u(r), owner)
    v = _view(lib.mpsvd_svd_v(r), owner)
    cnt = C.c_int64()
    sp = lib.mpsvd_svd_sigma(r, C.byref(cnt))
    sigma = np.ctypeslib.as_array(sp, shape=(cnt.value,)).copy() if cnt.value else np.zeros(0)
    t = (C.c_double * 5)()
    lib.mpsvd_svd_times(r, t)
    sw = C.c_int()
    rot = C.c_int64()
    lib.mpsvd_svd_jacobi_stats(r, C.byref(sw), C.byref(rot))
    return ThinSvdResult(u, sigma, v, PhaseTimes(*list(t)), lib.mpsvd_svd_sync_events(r),
                         lib.mpsvd_svd_gram_blocks(r), bool(lib.mpsvd_svd_is_qr_baseline(r)), sw.value, rot.value)


def mp_thin_svd(a, choice: EigensolverChoice = EigensolverChoice.TWOSIDED_JACOBI, threads: int = 1) -> ThinSvdResult:
    """mp_thin_svd (proj/include/mpsvd/thinsvd.hpp:58-59) via mpsvd_thin_svd.

    ``a`` may be a ``Matrix`` or a 2-D numpy array; fp64 input is rejected
    with InvalidArgument exactly like the reference (thinsvd.cpp:52-53).
    """
    mat = a if isinstance(a, Matrix) else Matrix.from_numpy(np.asarray(a))
    r = C.c_void_p()
    _check(lib.mpsvd_thin_svd(mat.handle, int(choice), int(threads), C.byref(r)))
    out = _result(r)
    out.eigensolver = EigensolverChoice(int(choice))
    return out


# thinsvd.hpp kDdMaxSweeps: sweep cap of the double-double path
DD_MAX_SWEEPS = 100


def mp_thin_svd_f64(a, threads: int = 1) -> ThinSvdResult:
    """ADDITIVE: fp64 A, Gram + Jacobi in double-double, U in fp64."""
    mat = a if isinstance(a, Matrix) else Matrix.from_numpy(np.asarray(a, dtype=np.float64))
    r = C.c_void_p()
    _check(lib.mpsvd_thin_svd_f64(mat.handle, int(threads), C.byref(r)))
    return _result(r)


def mp_cholesky_qr(a):
    """mp_cholesky_qr (proj/include/mpsvd/thinsvd.hpp:67-75) via mpsvd_cholesky_qr:
    returns (Q float32 m x n, R float32 n x n)."""
    mat = a if isinstance(a, Matrix) else Matrix.from_numpy(np.asarray(a))
    q, r = C.c_void_p(), C.c_void_p()
    _check(lib.mpsvd_cholesky_qr(mat.handle, C.byref(q), C.byref(r)))
    qm, rm = Matrix._adopt(q.value), Matrix._adopt(r.value)
    return qm.numpy().copy(), rm.numpy().copy()


def orth_error(q) -> float:
    mat = q if isinstance(q, Matrix) else Matrix.from_numpy(np.asarray(q))
    out = C.c_double()
    _check(lib.mpsvd_orth_error(mat.handle, C.byref(out)))
    return out.value


@dataclass
class BackwardErrorReport:
    """proj/include/mpsvd/metrics.hpp:44-47"""
    max_rel: float = 0.0
    skipped_rows: int = 0


def _dptr(x: np.ndarray):
    return x.ctypes.data_as(C.POINTER(C.c_double))


def max_rel_sv_error(computed, reference) -> float:
    """max_i |computed_i - reference_i| / reference_i (proj/src/metrics.cpp:26-38);
    InvalidArgument on a length mismatch or a non-positive reference entry."""
    c = np.ascontiguousarray(computed, dtype=np.float64)
    r = np.ascontiguousarray(reference, dtype=np.float64)
    if c.size != r.size:
        raise InvalidArgument("singular value arrays differ in length")
    out = C.c_double()
    _check(lib.mpsvd_max_rel_sv_error(_dptr(c), _dptr(r), int(r.size), C.byref(out)))
    return out.value


def rowwise_backward_error(a, u, sigma, v) -> BackwardErrorReport:
    """max_i ||(U diag(sigma) V^T - A)(i,:)|| / ||A(i,:)|| in binary64 on the GPU,
    zero rows of A skipped and counted (proj/src/metrics.cpp:40-70)."""
    mats = [x if isinstance(x, Matrix) else Matrix.from_numpy(np.asarray(x)) for x in (a, u, v)]
    s = np.ascontiguousarray(sigma, dtype=np.float64)
    out, skipped = C.c_double(), C.c_int64()
    _check(lib.mpsvd_rowwise_backward_error(mats[0].handle, mats[1].handle, _dptr(s), int(s.size), mats[2].handle,
                                            C.byref(out), C.byref(skipped)))
    return BackwardErrorReport(out.value, skipped.value)


def backward_error_device(a, u, sigma, v, stream=None) -> BackwardErrorReport:
    """The same on device-resident column-major torch tensors (a, u: m x n,
    v: n x n, all float32 or all float64; sigma: n float64). Row-sharded
    factors give per-rank maxima; the caller takes the max over ranks."""
    import torch

    f64 = a.dtype == torch.float64
    for t in (a, u, v):
        if t.dtype != a.dtype or not t.is_cuda:
            raise InvalidArgument("backward_error_device: a, u, v must be CUDA tensors of one dtype")
        if t.stride(0) != 1:
            raise InvalidArgument("backward_error_device: tensors must be column-major")
    if sigma.dtype != torch.float64 or not sigma.is_cuda:
        raise InvalidArgument("backward_error_device: sigma must be a float64 CUDA tensor")
    m, n = a.shape
    ld = lambda t: max(int(t.stride(1)), int(t.shape[0]), 1)
    st = stream if stream is not None else torch.cuda.current_stream(a.device)
    out, skipped = C.c_double(), C.c_int64()
    _check(lib.mpsvd_backward_error_device(int(Precision.HIGHER if f64 else Precision.WORKING), a.data_ptr(), ld(a),
                                           u.data_ptr(), ld(u), sigma.data_ptr(), v.data_ptr(), ld(v), m, n,
                                           st.cuda_stream, C.byref(out), C.byref(skipped)))
    return BackwardErrorReport(out.value, skipped.value)


# ---------------------------------------------------------------------------
# stage entry points (parity tests)

def gram(a: np.ndarray):
    """Device Gram: f32 A -> fp64 M; f64 A -> double-double (hi, lo)."""
    a = np.asfortranarray(a)
    m, n = a.shape
    hi = np.zeros((n, n), order="F")
    lo = np.zeros((n, n), order="F")
    prec = Precision.WORKING if a.dtype == np.float32 else Precision.HIGHER
    if prec == Precision.HIGHER:
        a = np.asfortranarray(a, dtype=np.float64)
    _check(lib.mpsvd_stage_gram(int(prec), a.ctypes.data, m, n, hi.ctypes.data_as(C.POINTER(C.c_double)),
                                lo.ctypes.data_as(C.POINTER(C.c_double))))
    return hi if prec == Precision.WORKING else (hi, lo)


def gram_schedule(m: int, n: int):
    """The double-double Gram schedule of an m x n plan (parity tests):
    (ozaki, scb, bsb) - split s covers 32-row chunks [scb[s], scb[s+1]),
    logical block b holds splits [bsb[b], bsb[b+1])."""
    cap = m // 32 + 64
    P = C.POINTER(C.c_int)
    scb = np.zeros(cap, np.int32)
    bsb = np.zeros(cap, np.int32)
    ns, nb, oz = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib.mpsvd_stage_gram_schedule(m, n, cap, C.byref(ns), C.byref(nb), scb.ctypes.data_as(P),
                                         bsb.ctypes.data_as(P), C.byref(oz)))
    return bool(oz.value), scb[: ns.value + 1].copy(), bsb[: nb.value + 1].copy()


def gram32_schedule(m: int, n: int):
    """The binary32 Gram schedule of an m x n plan (parity tests):
    (ozaki, npairs, bounds) - K1z launches once per chunk range
    [bounds[b], bounds[b+1]) with npairs CTA pairs."""
    cap = 64
    bounds = np.zeros(cap, np.int64)
    oz, npairs, nb = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib.mpsvd_stage_gram32_schedule(m, n, cap, C.byref(oz), C.byref(npairs), C.byref(nb),
                                           bounds.ctypes.data_as(C.POINTER(C.c_int64))))
    return bool(oz.value), npairs.value, bounds[: nb.value].copy()


def rank_combine(parts_hi, parts_lo=None):
    """The multi-GPU exchange's combine kernel on host-supplied per-rank
    partial Grams (shape (nranks, n, n); column-major n x n each): binary64
    adds (parts_lo None) or dd_add along the reference's tree over ranks.
    Returns M (fp64) or (hi, lo)."""
    ph = np.ascontiguousarray(np.stack([np.asfortranarray(x, dtype=np.float64).ravel(order="F") for x in parts_hi]))
    p, nn = ph.shape
    n = int(round(nn ** 0.5))
    dd = parts_lo is not None
    pl = (np.ascontiguousarray(np.stack([np.asfortranarray(x, dtype=np.float64).ravel(order="F") for x in parts_lo]))
          if dd else None)
    hi = np.zeros((n, n), order="F")
    lo = np.zeros((n, n), order="F")
    _check(lib.mpsvd_stage_rank_combine(int(Precision.HIGHER if dd else Precision.WORKING), _dptr(ph),
                                        _dptr(pl) if dd else None, p, n, _dptr(hi), _dptr(lo)))
    return (hi, lo) if dd else hi


def format_shortest(value: float) -> str:
    """mpsvd_format_shortest (proj/include/mpsvd.h:166-171)."""
    buf = C.create_string_buffer(48)
    k = lib.mpsvd_format_shortest(float(value), buf, 48)
    return buf.value.decode()[:k]


def twosided_jacobi_eig(m_hi, m_lo=None, dd: bool = False, tol: float = 0.0, max_sweeps: int | None = None):
    """Device two-sided Jacobi (jacobi.hpp:45-46); returns (lambda, V, sweeps, rotations).

    With ``dd`` the matrix is double-double (``m_lo`` its low words) and
    lambda / V come back as (hi, lo) pairs.
    """
    if max_sweeps is None:
        max_sweeps = DD_MAX_SWEEPS if dd else 30
    m_hi = np.asfortranarray(m_hi, dtype=np.float64)
    n = m_hi.shape[0]
    lo_in = np.asfortranarray(m_lo, dtype=np.float64) if m_lo is not None else None
    lh, ll = np.zeros(n), np.zeros(n)
    vh = np.zeros((n, n), order="F")
    vl = np.zeros((n, n), order="F")
    sw = C.c_int()
    rot = C.c_int64()
    P = C.POINTER(C.c_double)
    _check(lib.mpsvd_stage_jacobi(1 if dd else 0, m_hi.ctypes.data_as(P),
                                  lo_in.ctypes.data_as(P) if lo_in is not None else None, n, float(tol),
                                  int(max_sweeps), lh.ctypes.data_as(P), ll.ctypes.data_as(P), vh.ctypes.data_as(P),
                                  vl.ctypes.data_as(P), C.byref(sw), C.byref(rot)))
    if dd:
        return (lh, ll), (vh, vl), sw.value, rot.value
    return lh, vh, sw.value, rot.value


def onesided_spectral(choice, m_hi, tol: float = 0.0, max_sweeps: int = 30):
    """Spectral phase of the GRAM_CHOL_SVD / ONESIDED_JACOBI_GRAM branches
    (thinsvd.cpp:37-47,90-104) on the device for a binary64 Gram: returns
    (sigma, V float32, sweeps, rotations), sorted and sign-fixed."""
    m_hi = np.asfortranarray(m_hi, dtype=np.float64)
    n = m_hi.shape[0]
    sig = np.zeros(n)
    v = np.zeros((n, n), np.float32, order="F")
    sw = C.c_int()
    rot = C.c_int64()
    _check(lib.mpsvd_stage_onesided(int(choice), _dptr(m_hi), n, float(tol), int(max_sweeps), _dptr(sig),
                                    v.ctypes.data_as(C.POINTER(C.c_float)), C.byref(sw), C.byref(rot)))
    return sig, v, sw.value, rot.value


# ---------------------------------------------------------------------------
# device-resident plans (bench, multi-GPU)

class Comm:
    """NCCL communicator owned by the library (one rank per process)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        h = C.c_void_p()
        _check(lib.mpsvd_comm_init(unique_id, nranks, rank, C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib.mpsvd_comm_unique_id(buf))
        return buf.raw

    def __del__(self):
        if getattr(self, "_h", None):
            lib.mpsvd_comm_destroy(self._h)
            self._h = None


class Plan:
    """All device workspaces of one (m_local, n, precision, rank) pipeline."""

    def __init__(self, m_local: int, n: int, working: Precision = Precision.WORKING, comm: Comm | None = None):
        h = C.c_void_p()
        _check(lib.mpsvd_plan_create(m_local, n, int(working), comm._h if comm else None, C.byref(h)))
        self._h = h
        self._comm = comm
        self.m, self.n, self.working = m_local, n, working

    def execute(self, d_a: int, lda: int, d_u: int, ldu: int, d_sigma: int, d_v: int, stream: int = 0) -> None:
        _check(lib.mpsvd_plan_execute(self._h, d_a, lda, d_u, ldu, d_sigma, d_v, stream or None))

    def cholesky_qr(self, d_a: int, lda: int, d_q: int, ldq: int, d_r: int = 0, stream: int = 0) -> None:
        """Device-resident mixed-precision Cholesky QR (binary32 plans); finish with wait()."""
        _check(lib.mpsvd_plan_cholesky_qr(self._h, d_a, lda, d_q, ldq, d_r or None, stream or None))

    def set_eigensolver(self, choice: EigensolverChoice) -> None:
        _check(lib.mpsvd_plan_set_eigensolver(self._h, int(choice)))

    def orth_error(self, d_q: int, ldq: int, stream: int = 0) -> float:
        """||Q^T Q - I||_F (binary64) of a device-resident m_local x n Q in
        the plan's precision, through the plan's Gram (global over ranks)."""
        out = C.c_double()
        _check(lib.mpsvd_plan_orth_error(self._h, d_q, ldq, stream or None, C.byref(out)))
        return out.value

    def wait(self) -> ExecInfo:
        info = ExecInfo()
        st = lib.mpsvd_plan_wait(self._h, C.byref(info))
        _check(st, info.error_value)
        return info

    def __del__(self):
        if getattr(self, "_h", None):
            lib.mpsvd_plan_destroy(self._h)
            self._h = None
