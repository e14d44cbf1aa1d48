"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the two CPU oracles.

* ``Ref``  : the UNMODIFIED reference (``/root/reference/proj``) compiled in
  place by ``oracle/Makefile`` into ``oracle/_ref/libmpsvd_ref.so`` (flat C
  surface: ``oracle/ref_shim.cpp``).
* ``Port`` : our C restatement ``oracle/mpsvd_port.c`` (``oracle/_port``),
  pinned bit-for-bit against ``Ref`` by ``tests/test_oracle_port.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs import this module, and only as
the checker / CPU baseline. The product package never does.

All matrices are numpy arrays in Fortran (column-major) order, matching the
reference's ``j*rows+i`` layout (proj/include/mpsvd/types.hpp:175-177).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmpsvd_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libmpsvd_port.so")
REF_IO = os.path.join(HERE, "_ref", "ref_io")

SEM_REFERENCE = 0
SEM_DEVICE = 1

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


def _d(a):
    return a.ctypes.data_as(_dp)


def _f(a):
    return a.ctypes.data_as(_fp)


def _fcol(a, dtype):
    return np.asfortranarray(np.asarray(a, dtype=dtype))


class OracleError(RuntimeError):
    def __init__(self, status, index=0, value=0.0, msg=""):
        super().__init__(f"status={status} index={index} value={value} {msg}")
        self.status, self.index, self.value = int(status), int(index), float(value)


@dataclass
class SvdOut:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    times: np.ndarray
    sync_events: int = 1
    gram_blocks: int = 0


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Ref:
    """The reference library itself (built from /root/reference in place)."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle`")
            lib = C.CDLL(REF_SO)
            lib.refx_last_error.restype = C.c_char_p
            lib.refx_last_error.argtypes = [C.POINTER(_i64), _dp]
            Ref._lib = lib
        self.lib = Ref._lib

    def _check(self, st):
        if st != 0:
            idx = _i64(0)
            val = C.c_double(0)
            msg = self.lib.refx_last_error(C.byref(idx), C.byref(val))
            raise OracleError(st, idx.value, val.value, msg.decode())

    def thin_svd(self, a, threads=1, choice=0) -> SvdOut:
        a = _fcol(a, np.float32)
        m, n = a.shape
        u = np.zeros((m, n), np.float32, order="F")
        v = np.zeros((n, n), np.float32, order="F")
        s = np.zeros(n, np.float64)
        t = np.zeros(5, np.float64)
        se = C.c_int(0)
        gb = _i64(0)
        st = self.lib.refx_thin_svd(_f(a), _i64(m), _i64(n), C.c_int(choice), C.c_int(threads),
                                    _f(u), _d(s), _f(v), _d(t), C.byref(se), C.byref(gb))
        self._check(st)
        return SvdOut(u, s, v, t, se.value, gb.value)

    def thin_svd_f64_input(self, a):
        a = _fcol(a, np.float64)
        m, n = a.shape
        self._check(self.lib.refx_thin_svd_f64_input(_d(a), _i64(m), _i64(n)))

    def partitioned_gram_f32(self, a, workers=1, blocks=0):
        a = _fcol(a, np.float32)
        m, n = a.shape
        g = np.zeros((n, n), np.float64, order="F")
        se = C.c_int(0)
        nb = _i64(0)
        self._check(self.lib.refx_partitioned_gram_f32(_f(a), _i64(m), _i64(n), C.c_int(workers),
                                                       _i64(blocks), _d(g), C.byref(se), C.byref(nb)))
        return g, se.value, nb.value

    def partitioned_gram_f64(self, a, workers=1, blocks=0):
        a = _fcol(a, np.float64)
        m, n = a.shape
        g = np.zeros((n, n), np.float64, order="F")
        self._check(self.lib.refx_partitioned_gram_f64(_d(a), _i64(m), _i64(n), C.c_int(workers),
                                                       _i64(blocks), _d(g)))
        return g

    def gram_f64(self, a):
        a = _fcol(a, np.float64)
        m, n = a.shape
        g = np.zeros((n, n), np.float64, order="F")
        self._check(self.lib.refx_gram_f64(_d(a), _i64(m), _i64(n), _d(g)))
        return g

    def twosided_jacobi(self, mtx, tol=0.0, max_sweeps=30):
        mtx = _fcol(mtx, np.float64)
        n = mtx.shape[0]
        lam = np.zeros(n)
        v = np.zeros((n, n), order="F")
        sw = C.c_int(0)
        rot = _i64(0)
        self._check(self.lib.refx_twosided_jacobi(_d(mtx), _i64(n), C.c_double(tol), C.c_int(max_sweeps),
                                                  _d(lam), _d(v), C.byref(sw), C.byref(rot)))
        return lam, v, sw.value, rot.value

    def reference_svd(self, a):
        a = np.asfortranarray(a)
        m, n = a.shape
        s = np.zeros(n)
        if a.dtype == np.float32:
            self._check(self.lib.refx_reference_svd_f32(_f(a), _i64(m), _i64(n), _d(s)))
        else:
            a = _fcol(a, np.float64)
            self._check(self.lib.refx_reference_svd_f64(_d(a), _i64(m), _i64(n), _d(s)))
        return s

    def orth_error(self, q):
        q = np.asfortranarray(q)
        m, n = q.shape
        out = C.c_double(0)
        if q.dtype == np.float32:
            self._check(self.lib.refx_orth_error_f32(_f(q), _i64(m), _i64(n), C.byref(out)))
        else:
            q = _fcol(q, np.float64)
            self._check(self.lib.refx_orth_error_f64(_d(q), _i64(m), _i64(n), C.byref(out)))
        return out.value

    def cholesky_qr(self, a):
        a = _fcol(a, np.float32)
        m, n = a.shape
        q = np.zeros((m, n), np.float32, order="F")
        r = np.zeros((n, n), np.float32, order="F")
        self._check(self.lib.refx_cholesky_qr(_f(a), _i64(m), _i64(n), _f(q), _f(r)))
        return q, r

    def rowwise_backward_error(self, a, u, sigma, v):
        """(max_rel, skipped_rows) of proj/src/metrics.cpp:40-70; f32 or f64 factors."""
        a = np.asfortranarray(a)
        m, n = a.shape
        mr = C.c_double(0)
        sk = _i64(0)
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        if a.dtype == np.float32:
            st = self.lib.refx_rowwise_backward_error_f32(_f(a), _f(_fcol(u, np.float32)), _d(s),
                                                          _f(_fcol(v, np.float32)), _i64(m), _i64(n),
                                                          C.byref(mr), C.byref(sk))
        else:
            st = self.lib.refx_rowwise_backward_error_f64(_d(_fcol(a, np.float64)), _d(_fcol(u, np.float64)), _d(s),
                                                          _d(_fcol(v, np.float64)), _i64(m), _i64(n),
                                                          C.byref(mr), C.byref(sk))
        self._check(st)
        return mr.value, sk.value

    def max_rel_sv_error(self, computed, reference):
        c = np.ascontiguousarray(computed, dtype=np.float64)
        r = np.ascontiguousarray(reference, dtype=np.float64)
        out = C.c_double(0)
        self._check(self.lib.refx_max_rel_sv_error(_d(c), _d(r), _i64(r.size), C.byref(out)))
        return out.value

    def build_problem(self, m, n, kappa_d, kappa_b, matrix_id, seed):
        a = np.zeros((m, n), np.float32, order="F")
        s = np.zeros(n)
        kb = C.c_double(0)
        self._check(self.lib.refx_build_problem(_i64(m), _i64(n), C.c_double(kappa_d), C.c_double(kappa_b),
                                                C.c_int(matrix_id), C.c_uint64(seed), _f(a), _d(s), C.byref(kb)))
        return a, s, kb.value

    def haar_orthonormal(self, m, n, seed):
        q = np.zeros((m, n), np.float64, order="F")
        self._check(self.lib.refx_haar_orthonormal(_i64(m), _i64(n), C.c_uint64(seed), _d(q)))
        return q

    @staticmethod
    def io_roundtrip(src, dst) -> int:
        """The reference's read_matrix_file(src) then write_matrix_file(dst)
        (proj/src/io.cpp) in a child process (oracle/_ref/ref_io: the
        reference's iostreams and this interpreter's libstdc++ do not mix);
        returns its status (0 ok, 9 IoError)."""
        import subprocess
        return subprocess.run([REF_IO, str(src), str(dst)], capture_output=True).returncode

    def dd_gram(self, a):
        a = _fcol(a, np.float64)
        m, n = a.shape
        hi = np.zeros((n, n), order="F")
        lo = np.zeros((n, n), order="F")
        self._check(self.lib.refx_dd_gram(_d(a), _i64(m), _i64(n), _d(hi), _d(lo)))
        return hi, lo

    def dd_oracle_eigenvalues(self, mtx):
        mtx = _fcol(mtx, np.float64)
        n = mtx.shape[0]
        out = np.zeros(n)
        self._check(self.lib.refx_dd_oracle_eigenvalues(_d(mtx), _i64(n), _d(out)))
        return out

    def dd_oracle_singular_values(self, a):
        a = np.asfortranarray(a)
        m, n = a.shape
        out = np.zeros(n)
        if a.dtype == np.float32:
            self._check(self.lib.refx_dd_oracle_singular_values_f32(_f(a), _i64(m), _i64(n), _d(out)))
        else:
            a = _fcol(a, np.float64)
            self._check(self.lib.refx_dd_oracle_singular_values_f64(_d(a), _i64(m), _i64(n), _d(out)))
        return out


class _PortErr(C.Structure):
    _fields_ = [("status", C.c_int), ("index", _i64), ("value", C.c_double)]


class _PortStats(C.Structure):
    _fields_ = [("sweeps", C.c_int), ("rotations", _i64), ("pairs_per_sweep", _i64)]


class Port:
    """Our C restatement (oracle/mpsvd_port.c)."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            if not os.path.exists(PORT_SO):
                raise FileNotFoundError(f"{PORT_SO} missing: run `make -C oracle port`")
            lib = C.CDLL(PORT_SO)
            lib.port_orth_error_f32.restype = C.c_double
            lib.port_orth_error_f64.restype = C.c_double
            Port._lib = lib
        self.lib = Port._lib

    @staticmethod
    def _raise(st, err):
        if st != 0:
            raise OracleError(st, err.index, err.value)

    def partition_plan(self, m, workers, blocks=0):
        nb = _i64(0)
        st = self.lib.port_partition_plan(_i64(m), C.c_int(workers), _i64(blocks), None, C.byref(nb))
        if st != 0:
            raise OracleError(st)
        r = np.zeros(2 * nb.value, np.int64)
        self.lib.port_partition_plan(_i64(m), C.c_int(workers), _i64(blocks),
                                     r.ctypes.data_as(C.POINTER(_i64)), C.byref(nb))
        return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(nb.value)]

    def rr_pair(self, n, rnd, k):
        p, q = _i64(0), _i64(0)
        self.lib.port_rr_pair(_i64(n), _i64(rnd), _i64(k), C.byref(p), C.byref(q))
        return p.value, q.value

    def partitioned_gram_f32(self, a, blocks=16):
        a = _fcol(a, np.float32)
        m, n = a.shape
        g = np.zeros((n, n), order="F")
        st = self.lib.port_partitioned_gram_f32(_f(a), _i64(m), _i64(n), _i64(blocks), _d(g))
        if st:
            raise OracleError(st)
        return g

    def partitioned_gram_f64(self, a, blocks=16):
        a = _fcol(a, np.float64)
        m, n = a.shape
        g = np.zeros((n, n), order="F")
        st = self.lib.port_partitioned_gram_f64(_d(a), _i64(m), _i64(n), _i64(blocks), _d(g))
        if st:
            raise OracleError(st)
        return g

    def twosided_jacobi(self, mtx, tol=0.0, max_sweeps=30, sem=SEM_REFERENCE):
        mtx = _fcol(mtx, np.float64)
        n = mtx.shape[0]
        lam = np.zeros(n)
        v = np.zeros((n, n), order="F")
        stt = _PortStats()
        err = _PortErr()
        st = self.lib.port_twosided_jacobi_f64(_d(mtx), _i64(n), C.c_double(tol), C.c_int(max_sweeps),
                                               C.c_int(sem), _d(lam), _d(v), C.byref(stt), C.byref(err))
        self._raise(st, err)
        return lam, v, stt.sweeps, stt.rotations

    def thin_svd(self, a, threads=1, sem=SEM_REFERENCE, choice=0) -> SvdOut:
        a = _fcol(a, np.float32)
        m, n = a.shape
        u = np.zeros((m, n), np.float32, order="F")
        v = np.zeros((n, n), np.float32, order="F")
        s = np.zeros(n)
        t = np.zeros(5)
        err = _PortErr()
        st = self.lib.port_thin_svd_f32_choice(_f(a), _i64(m), _i64(n), C.c_int(threads), C.c_int(sem),
                                               C.c_int(choice), _f(u), _d(s), _f(v), _d(t), C.byref(err))
        self._raise(st, err)
        return SvdOut(u, s, v, t, 1, min(16, m))

    def cholesky_qr(self, a):
        a = _fcol(a, np.float32)
        m, n = a.shape
        q = np.zeros((m, n), np.float32, order="F")
        r = np.zeros((n, n), np.float32, order="F")
        err = _PortErr()
        self._raise(self.lib.port_cholesky_qr_f32(_f(a), _i64(m), _i64(n), _f(q), _f(r), C.byref(err)), err)
        return q, r

    def cholqr_solve(self, a, r):
        a = _fcol(a, np.float32)
        r = _fcol(r, np.float32)
        m, n = a.shape
        q = np.zeros((m, n), np.float32, order="F")
        self.lib.port_cholqr_solve(_f(a), _i64(m), _i64(n), _f(r), _f(q))
        return q

    def cholesky(self, mtx):
        mtx = _fcol(mtx, np.float64)
        n = mtx.shape[0]
        r = np.zeros((n, n), order="F")
        err = _PortErr()
        self._raise(self.lib.port_cholesky_f64(_d(mtx), _i64(n), _d(r), C.byref(err)), err)
        return r

    def onesided_spectral(self, choice, mtx, tol=0.0, max_sweeps=30, sem=SEM_DEVICE):
        """(sigma, V float32, sweeps, rotations) of the GramCholSvd (1) or
        OneSidedJacobiOnGram (2) spectral phase on the Gram mtx."""
        mtx = _fcol(mtx, np.float64)
        n = mtx.shape[0]
        s = np.zeros(n)
        v = np.zeros((n, n), np.float32, order="F")
        stt = _PortStats()
        err = _PortErr()
        st = self.lib.port_onesided_spectral(C.c_int(choice), _d(mtx), _i64(n), C.c_double(tol), C.c_int(max_sweeps),
                                             C.c_int(sem), _d(s), _f(v), C.byref(stt), C.byref(err))
        self._raise(st, err)
        return s, v, stt.sweeps, stt.rotations

    def av_f32(self, a, w, threads=8):
        a = _fcol(a, np.float32)
        w = _fcol(w, np.float32)
        m, n = a.shape
        u = np.zeros((m, n), np.float32, order="F")
        self.lib.port_av_f32(_f(a), _i64(m), _i64(n), _f(w), _f(u), C.c_int(threads))
        return u

    def dd_op(self, op, a, b=(0.0, 0.0)):
        rh, rl = C.c_double(0), C.c_double(0)
        f = getattr(self.lib, "port_dd_" + op)
        if op == "sqrt":
            f(C.c_double(a[0]), C.c_double(a[1]), C.byref(rh), C.byref(rl))
        else:
            f(C.c_double(a[0]), C.c_double(a[1]), C.c_double(b[0]), C.c_double(b[1]), C.byref(rh), C.byref(rl))
        return rh.value, rl.value

    def dd_gram(self, a, threads=8):
        a = _fcol(a, np.float64)
        m, n = a.shape
        hi = np.zeros((n, n), order="F")
        lo = np.zeros((n, n), order="F")
        st = self.lib.port_dd_gram(_d(a), _i64(m), _i64(n), C.c_int(threads), _d(hi), _d(lo))
        if st:
            raise OracleError(st)
        return hi, lo

    def oz_sub_group(self, i):
        """K2z sub-group i: (w_hi, nw, pa, pb)."""
        v = [C.c_int(0) for _ in range(4)]
        self.lib.port_oz_sub_group(C.c_int(i), *[C.byref(x) for x in v])
        return tuple(x.value for x in v)

    def gram_dd_ozaki(self, a, scb, bsb, span_cap=1 << 20):
        """K2z's double-double Gram (csrc/gram_ozaki.cu) on the split schedule
        scb (chunks) / bsb (logical blocks), bit for bit."""
        a = _fcol(a, np.float64)
        m, n = a.shape
        scb = np.ascontiguousarray(scb, dtype=np.int32)
        bsb = np.ascontiguousarray(bsb, dtype=np.int32)
        hi = np.zeros((n, n), order="F")
        lo = np.zeros((n, n), order="F")
        P = C.POINTER(C.c_int)
        st = self.lib.port_gram_dd_ozaki(_d(a), _i64(m), _i64(n), C.c_int(len(scb) - 1), scb.ctypes.data_as(P),
                                         C.c_int(len(bsb) - 1), bsb.ctypes.data_as(P), C.c_int(span_cap), _d(hi),
                                         _d(lo))
        if st:
            raise OracleError(st)
        return hi, lo

    def gram_f32_ozaki(self, a, npairs, bounds, span_max=512, threads=8):
        """K1z's binary64 Gram of a binary32 A (csrc/gram_ozaki32.cu) on the
        plan's schedule (npairs, chunk-range bounds), bit for bit."""
        a = _fcol(a, np.float32)
        m, n = a.shape
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        out = np.zeros((n, n), order="F")
        st = self.lib.port_gram_f32_ozaki(_f(a), _i64(m), _i64(n), C.c_int(npairs), C.c_int(len(bounds) - 1),
                                          bounds.ctypes.data_as(C.POINTER(C.c_int64)), C.c_int(span_max),
                                          C.c_int(threads), _d(out))
        if st:
            raise OracleError(st)
        return out

    def twosided_jacobi_dd(self, mhi, mlo=None, tol=0.0, max_sweeps=30, sem=SEM_REFERENCE):
        mhi = _fcol(mhi, np.float64)
        n = mhi.shape[0]
        mlo = np.zeros_like(mhi) if mlo is None else _fcol(mlo, np.float64)
        lh, ll = np.zeros(n), np.zeros(n)
        vh = np.zeros((n, n), order="F")
        vl = np.zeros((n, n), order="F")
        stt = _PortStats()
        err = _PortErr()
        st = self.lib.port_twosided_jacobi_dd(_d(mhi), _d(mlo), _i64(n), C.c_double(tol), C.c_int(max_sweeps),
                                              C.c_int(sem), _d(lh), _d(ll), _d(vh), _d(vl), C.byref(stt),
                                              C.byref(err))
        self._raise(st, err)
        return (lh, ll), (vh, vl), stt.sweeps, stt.rotations

    def thin_svd_f64dd(self, a, threads=8, sem=SEM_REFERENCE) -> SvdOut:
        a = _fcol(a, np.float64)
        m, n = a.shape
        u = np.zeros((m, n), order="F")
        v = np.zeros((n, n), order="F")
        s = np.zeros(n)
        t = np.zeros(5)
        err = _PortErr()
        st = self.lib.port_thin_svd_f64dd(_d(a), _i64(m), _i64(n), C.c_int(threads), C.c_int(sem),
                                          _d(u), _d(s), _d(v), _d(t), C.byref(err))
        self._raise(st, err)
        return SvdOut(u, s, v, t, 1, 0)

    def orth_error(self, q, threads=8):
        q = np.asfortranarray(q)
        m, n = q.shape
        if q.dtype == np.float32:
            return self.lib.port_orth_error_f32(_f(q), _i64(m), _i64(n), C.c_int(threads))
        q = _fcol(q, np.float64)
        return self.lib.port_orth_error_f64(_d(q), _i64(m), _i64(n), C.c_int(threads))
