"""ctypes bindings to the two CPU checkers under oracle/ (TEST INFRASTRUCTURE).

* ``Ref``  — oracle/_ref/libtenkit_ref.so: the UNMODIFIED reference library
  (tenkit, /root/reference/proj/src) compiled by oracle/Makefile, behind our
  thin C wrapper oracle/ref_capi.cpp.
* ``Port`` — oracle/_ref/liboracle_port.so: our plain-C restatement
  oracle/tenkit_oracle.c, pinned bitwise against ``Ref`` by
  tests/test_oracle_pins.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
Arrays are numpy float64 in Fortran (column-major) order, matching
tensor.hpp:10-11 / matrix.hpp:8-9.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtenkit_ref.so")
PORT_SO = os.path.join(ROOT, "oracle", "_ref", "liboracle_port.so")

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _u64(seq):
    arr = (C.c_uint64 * len(seq))(*[int(x) for x in seq])
    return arr


def _ext(t, mode):
    """Extent of a 1-based mode, 1 when out of range (the library reports it)."""
    return t.shape[mode - 1] if 1 <= mode <= t.ndim else 1


def fortran(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def flat(a) -> np.ndarray:
    """Column-major flat copy of an array."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, order="F"))


class OracleError(RuntimeError):
    def __init__(self, code: int, subtype: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.subtype = subtype


SUBTYPES = {
    1: "InvalidModeError",
    2: "DimensionMismatchError",
    3: "ZeroReferenceError",
    4: "RankTooLargeError",
    5: "SingularGramError",
    6: "DegenerateInitError",
    7: "NoConvergenceError",
    10: "Error",
}


@dataclass
class ModeRecord:
    mode: int
    iterations: int
    status: int
    achieved_eta: float
    residual_history: list = field(default_factory=list)
    seconds: float = 0.0


@dataclass
class HosvdResult:
    core: np.ndarray
    factors: list
    per_mode: list
    relative_residual: float
    seconds: float = 0.0


def build_if_missing():
    if not (os.path.exists(REF_SO) and os.path.exists(PORT_SO)):
        if not os.path.isdir("/root/reference/proj/src") and not os.path.exists(PORT_SO):
            raise FileNotFoundError("oracle/_ref not built and /root/reference absent")
        import subprocess
        target = "all" if os.path.isdir("/root/reference/proj/src") else "port"
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), target])


class Ref:
    """The compiled reference (oracle/_ref/libtenkit_ref.so)."""

    def __init__(self, path: str = REF_SO):
        build_if_missing()
        self.lib = C.CDLL(path)
        self._msg = C.create_string_buffer(512)
        self._sub = C.c_int(0)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._sub.value, self._msg.value.decode())

    def _e(self):
        return (C.byref(self._sub), self._msg, C.c_int(512))

    def set_threads(self, n: int):
        self.lib.ref_set_threads(C.c_int(n))

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    def engine_raw(self, seed, stream, n):
        out = np.zeros(n, dtype=np.uint64)
        self.lib.ref_engine_raw(C.c_uint64(seed), C.c_uint32(stream), C.c_uint64(n),
                                out.ctypes.data_as(_u64p))
        return out

    def uniform01(self, seed, stream, n):
        out = np.zeros(n)
        self.lib.ref_uniform01(C.c_uint64(seed), C.c_uint32(stream), C.c_uint64(n), _d(out))
        return out

    def uniform_in(self, seed, lo, hi, n, stream=0):
        out = np.zeros(n)
        self.lib.ref_uniform_in(C.c_uint64(seed), C.c_uint32(stream), C.c_double(lo),
                                C.c_double(hi), C.c_uint64(n), _d(out))
        return out

    def gaussian(self, seed, n, stream=0):
        out = np.zeros(n)
        self.lib.ref_gaussian(C.c_uint64(seed), C.c_uint32(stream), C.c_uint64(n), _d(out))
        return out

    # -- tensor_ops ----------------------------------------------------------
    def unfold_times(self, t, mode, m):
        t = fortran(t)
        m = fortran(m)
        out = np.zeros((_ext(t, mode), m.shape[1]), order="F")
        self._check(self.lib.ref_unfold_times(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                              C.c_uint32(mode), _d(flat(m)),
                                              C.c_uint64(m.shape[1]), _d(out), *self._e()))
        return out

    def unfold_t_times(self, t, mode, m):
        t = fortran(t)
        m = fortran(m)
        fibers = t.size // _ext(t, mode)
        out = np.zeros((fibers, m.shape[1]), order="F")
        self._check(self.lib.ref_unfold_t_times(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                                C.c_uint32(mode), _d(flat(m)),
                                                C.c_uint64(m.shape[1]), _d(out), *self._e()))
        return out

    def mode_n_product(self, t, u, mode):
        t = fortran(t)
        u = fortran(u)
        dims = list(t.shape)
        dims[mode - 1] = u.shape[0]
        out = np.zeros(dims, order="F")
        self._check(self.lib.ref_mode_n_product(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                                _d(flat(u)), C.c_uint64(u.shape[0]),
                                                C.c_uint64(u.shape[1]), C.c_uint32(mode),
                                                _d(out), *self._e()))
        return out

    def frobenius_norm(self, t):
        t = fortran(t)
        out = C.c_double(0)
        self._check(self.lib.ref_frobenius_norm(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                                C.byref(out), *self._e()))
        return out.value

    def relative_error(self, a, b):
        a = fortran(a)
        b = fortran(b)
        out = C.c_double(0)
        self._check(self.lib.ref_relative_error(_d(flat(a)), _d(flat(b)), C.c_int(a.ndim),
                                                _u64(a.shape), C.byref(out), *self._e()))
        return out.value

    # -- small dense LA --------------------------------------------------------
    def reduced_qr(self, a):
        a = fortran(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        r = np.zeros((n, n), order="F")
        self._check(self.lib.ref_reduced_qr(_d(flat(a)), C.c_uint64(m), C.c_uint64(n), _d(q),
                                            _d(r), *self._e()))
        return q, r

    def spd_solve(self, g, b):
        g = fortran(g)
        b = fortran(b)
        x = np.zeros(b.shape, order="F")
        self._check(self.lib.ref_spd_solve(_d(flat(g)), C.c_uint64(g.shape[0]), _d(flat(b)),
                                           C.c_uint64(b.shape[1]), _d(x), *self._e()))
        return x

    def gram(self, a):
        a = fortran(a)
        g = np.zeros((a.shape[1], a.shape[1]), order="F")
        self._check(self.lib.ref_gram(_d(flat(a)), C.c_uint64(a.shape[0]),
                                      C.c_uint64(a.shape[1]), _d(g), *self._e()))
        return g

    def singular_values(self, a):
        a = fortran(a)
        k = min(a.shape)
        v = np.zeros(k)
        self._check(self.lib.ref_dense_svd_values(_d(flat(a)), C.c_uint64(a.shape[0]),
                                                  C.c_uint64(a.shape[1]), _d(v), *self._e()))
        return v

    # -- ALS / HOSVD -----------------------------------------------------------
    def recover_singular_vectors(self, t, mode, q):
        t = fortran(t)
        q = fortran(q)
        out = np.zeros(q.shape, order="F")
        self._check(self.lib.ref_recover_singular_vectors(
            _d(flat(t)), C.c_int(t.ndim), _u64(t.shape), C.c_uint32(mode), _d(flat(q)),
            C.c_uint64(q.shape[0]), C.c_uint64(q.shape[1]), _d(out), *self._e()))
        return out

    def als_init(self, t, mode, r, seed):
        t = fortran(t)
        l = np.zeros((_ext(t, mode), r), order="F")
        self._check(self.lib.ref_als_init(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                          C.c_uint32(mode), C.c_uint64(r), C.c_uint64(seed),
                                          _d(l), *self._e()))
        return l

    def als_sweep(self, t, mode, l):
        t = fortran(t)
        l = fortran(l)
        r = l.shape[1]
        fibers = t.size // _ext(t, mode)
        ln = np.zeros(l.shape, order="F")
        rr = np.zeros((fibers, r), order="F")
        res = C.c_double(0)
        self._check(self.lib.ref_als_sweep(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                           C.c_uint32(mode), _d(flat(l)), C.c_uint64(r),
                                           _d(ln), _d(rr), C.byref(res), *self._e()))
        return ln, rr, res.value

    def als_low_rank(self, t, mode, r, eta=1e-4, max_iters=50, seed=0, init=None):
        t = fortran(t)
        fibers = t.size // _ext(t, mode)
        l = np.zeros((_ext(t, mode), r), order="F")
        rr = np.zeros((fibers, r), order="F")
        it = C.c_int(0)
        st = C.c_int(0)
        ae = C.c_double(0)
        cap = max(64, int(max_iters))
        hist = np.zeros(cap)
        self._check(self.lib.ref_als_low_rank(
            _d(flat(t)), C.c_int(t.ndim), _u64(t.shape), C.c_uint32(mode), C.c_uint64(r),
            C.c_double(eta), C.c_int(max_iters), C.c_uint64(seed),
            _d(flat(init)) if init is not None else None, _d(l), _d(rr), C.byref(it),
            C.byref(st), C.byref(ae), _d(hist), C.c_int(cap), *self._e()))
        rec = ModeRecord(mode, it.value, st.value, ae.value, list(hist[: min(it.value, cap)]))
        return l, rr, rec

    def select_order(self, dims, ranks):
        out = (C.c_uint32 * len(dims))()
        self._check(self.lib.ref_select_order(C.c_int(len(dims)), _u64(dims), _u64(ranks), out,
                                              *self._e()))
        return list(out)

    def hosvd_als(self, t, ranks, sequential=False, order=None, eta=1e-4, max_iters=50,
                  seed=0, want_singular_vectors=False):
        t = fortran(t)
        n = t.ndim
        core = np.zeros(ranks, order="F")
        total = sum(int(t.shape[k]) * int(ranks[k]) for k in range(n))
        fac = np.zeros(total)
        rep = (C.c_char * self.lib.ref_report_size())()
        mo = (C.c_uint32 * n)(*order) if order is not None else None
        self._check(self.lib.ref_hosvd_als(
            C.c_int(1 if sequential else (2 if want_singular_vectors else 0)), _d(flat(t)), C.c_int(n), _u64(t.shape),
            _u64(ranks), mo, C.c_double(eta), C.c_int(max_iters), C.c_uint64(seed), _d(core),
            _d(fac), rep, *self._e()))
        raw = bytes(rep)
        i32 = np.frombuffer(raw, dtype=np.int32, count=192)
        f64 = np.frombuffer(raw, dtype=np.float64, offset=768)
        ach = f64[0:64]
        secs = f64[64:128]
        hist = f64[128:128 + 64 * 64].reshape(64, 64)
        seconds = f64[128 + 4096]
        relres = f64[128 + 4097]
        factors = []
        ofs = 0
        for k in range(n):
            sz = int(t.shape[k]) * int(ranks[k])
            factors.append(fac[ofs:ofs + sz].reshape((t.shape[k], ranks[k]), order="F"))
            ofs += sz
        per_mode = []
        for p in range(n):
            its = int(i32[64 + p])
            per_mode.append(ModeRecord(int(i32[p]), its, int(i32[128 + p]), float(ach[p]),
                                       list(hist[p, :min(its, 64)]), float(secs[p])))
        return HosvdResult(core, factors, per_mode, float(relres), float(seconds))

    def hosvd_als_tnsr(self, path, dims, ranks, sequential=False, order=None, eta=1e-4,
                       max_iters=50, seed=0):
        """ref_hosvd_als_tnsr: the reference reads the TNSR itself (read_tnsr)
        and decomposes it; returns (HosvdResult, call_seconds)."""
        n = len(dims)
        core = np.zeros(ranks, order="F")
        total = sum(int(dims[k]) * int(ranks[k]) for k in range(n))
        fac = np.zeros(total)
        rep = (C.c_char * self.lib.ref_report_size())()
        mo = (C.c_uint32 * n)(*order) if order is not None else None
        dims_out = (C.c_uint64 * 64)()
        secs = C.c_double(0.0)
        self._check(self.lib.ref_hosvd_als_tnsr(
            C.c_int(1 if sequential else 0), os.fsencode(path), _u64(ranks), mo, C.c_double(eta),
            C.c_int(max_iters), C.c_uint64(seed), _d(core), _d(fac), rep, dims_out, C.byref(secs),
            *self._e()))
        if list(dims_out[:n]) != [int(d) for d in dims]:
            raise ValueError(f"TNSR extents {list(dims_out[:n])} != {list(dims)}")
        return self._unpack_report(bytes(rep), core, fac, dims, ranks), float(secs.value)

    @staticmethod
    def _unpack_report(raw, core, fac, dims, ranks):
        n = len(dims)
        i32 = np.frombuffer(raw, dtype=np.int32, count=192)
        f64 = np.frombuffer(raw, dtype=np.float64, offset=768)
        ach, secs = f64[0:64], f64[64:128]
        hist = f64[128:128 + 64 * 64].reshape(64, 64)
        factors, ofs = [], 0
        for k in range(n):
            sz = int(dims[k]) * int(ranks[k])
            factors.append(fac[ofs:ofs + sz].reshape((int(dims[k]), int(ranks[k])), order="F"))
            ofs += sz
        per_mode = []
        for p in range(n):
            its = int(i32[64 + p])
            per_mode.append(ModeRecord(int(i32[p]), its, int(i32[128 + p]), float(ach[p]),
                                       list(hist[p, :min(its, 64)]), float(secs[p])))
        return HosvdResult(core, factors, per_mode, float(f64[128 + 4097]), float(f64[128 + 4096]))

    def hosvd_exact(self, t, ranks, kind, sequential=False, order=None):
        """t_hosvd / st_hosvd with FactorEngine::svd() (kind "svd") or ::eig() ("eig")."""
        t = fortran(t)
        n = t.ndim
        core = np.zeros(ranks, order="F")
        total = sum(int(t.shape[k]) * int(ranks[k]) for k in range(n))
        fac = np.zeros(total)
        rep = (C.c_char * self.lib.ref_report_size())()
        mo = (C.c_uint32 * n)(*order) if order is not None else None
        self._check(self.lib.ref_hosvd_exact(
            C.c_int(1 if sequential else 0), C.c_int(0 if kind == "svd" else 1), _d(flat(t)), C.c_int(n),
            _u64(t.shape), _u64(ranks), mo, _d(core), _d(fac), rep, *self._e()))
        raw = bytes(rep)
        f64 = np.frombuffer(raw, dtype=np.float64, offset=768)
        i32 = np.frombuffer(raw, dtype=np.int32, count=192)
        factors = []
        ofs = 0
        for k in range(n):
            sz = int(t.shape[k]) * int(ranks[k])
            factors.append(fac[ofs:ofs + sz].reshape((t.shape[k], ranks[k]), order="F"))
            ofs += sz
        per_mode = [ModeRecord(int(i32[p]), 0, -1, 0.0) for p in range(n)]
        return HosvdResult(core, factors, per_mode, float(f64[128 + 4097]), float(f64[128 + 4096]))

    def hooi(self, t, ranks, init_core, init_factors, tol=1e-12, max_iters=100):
        """hooi.cpp:53-110; returns (core, factors, iterations, converged, fit_history)."""
        t = fortran(t)
        n = t.ndim
        core = np.zeros(ranks, order="F")
        fac = np.zeros(sum(int(t.shape[k]) * int(ranks[k]) for k in range(n)))
        f_in = np.concatenate([flat(u) for u in init_factors])
        fits = np.zeros(max(1, max_iters) + 1)
        it, cv = C.c_int(0), C.c_int(0)
        self._check(self.lib.ref_hooi(_d(flat(t)), C.c_int(n), _u64(t.shape), _u64(ranks), _d(flat(init_core)),
                                      _d(f_in), C.c_double(tol), C.c_int(max_iters), _d(core), _d(fac),
                                      C.byref(it), C.byref(cv), _d(fits), *self._e()))
        factors = []
        ofs = 0
        for k in range(n):
            sz = int(t.shape[k]) * int(ranks[k])
            factors.append(fac[ofs:ofs + sz].reshape((t.shape[k], ranks[k]), order="F"))
            ofs += sz
        return core, factors, int(it.value), bool(cv.value), list(fits[: it.value + 1])

    def write_tnsr(self, path, t):
        t = fortran(t)
        self._check(self.lib.ref_write_tnsr(os.fsencode(path), _d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                            *self._e()))

    def read_tnsr(self, path):
        order, dims = C.c_int(0), (C.c_uint64 * 64)()
        self._check(self.lib.ref_read_tnsr(os.fsencode(path), C.byref(order), dims, None, C.c_uint64(0),
                                           *self._e()))
        shape = [int(dims[k]) for k in range(order.value)]
        out = np.zeros(int(np.prod(shape)))
        self._check(self.lib.ref_read_tnsr(os.fsencode(path), C.byref(order), dims, _d(out),
                                           C.c_uint64(out.size), *self._e()))
        return out.reshape(shape, order="F")

    def read_tukr(self, path):
        """(core, factors, origin dims) of a TUKR file read by the reference."""
        order, dims, ranks = C.c_int(0), (C.c_uint64 * 64)(), (C.c_uint64 * 64)()
        self._check(self.lib.ref_read_tukr(os.fsencode(path), C.byref(order), dims, ranks, None, None,
                                           C.c_uint64(0), *self._e()))
        n = order.value
        d = [int(dims[k]) for k in range(n)]
        r = [int(ranks[k]) for k in range(n)]
        core = np.zeros(int(np.prod(r)))
        fac = np.zeros(sum(d[k] * r[k] for k in range(n)))
        self._check(self.lib.ref_read_tukr(os.fsencode(path), C.byref(order), dims, ranks, _d(core), _d(fac),
                                           C.c_uint64(core.size + fac.size), *self._e()))
        factors, ofs = [], 0
        for k in range(n):
            factors.append(fac[ofs:ofs + d[k] * r[k]].reshape((d[k], r[k]), order="F"))
            ofs += d[k] * r[k]
        return core.reshape(r, order="F"), factors, d

    def mode_gram(self, t, mode):
        t = fortran(t)
        ext = _ext(t, mode)
        out = np.zeros((ext, ext), order="F")
        self._check(self.lib.ref_mode_gram(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape), C.c_uint32(mode),
                                           _d(out), *self._e()))
        return out

    def sym_eig(self, g, k):
        g = fortran(g)
        n = g.shape[0]
        vals = np.zeros(k)
        vecs = np.zeros((n, k), order="F")
        self._check(self.lib.ref_sym_eig(_d(flat(g)), C.c_uint64(n), C.c_uint64(k), _d(vals), _d(vecs),
                                         *self._e()))
        return vals, vecs

    def reconstruct(self, core, factors, dims):
        core = fortran(core)
        ranks = core.shape
        out = np.zeros(dims, order="F")
        fac = np.concatenate([flat(u) for u in factors])
        self._check(self.lib.ref_reconstruct(_d(flat(core)), C.c_int(core.ndim), _u64(ranks),
                                             _u64(dims), _d(fac), _d(out), *self._e()))
        return out


class _OrcError(C.Structure):
    _fields_ = [("subtype", C.c_int), ("msg", C.c_char * 256)]


class _OrcAls(C.Structure):
    _fields_ = [("iterations", C.c_int), ("status", C.c_int), ("achieved_eta", C.c_double),
                ("history", C.c_double * 64)]


class _OrcHosvd(C.Structure):
    _fields_ = [("modes", C.c_int * 64), ("als", _OrcAls * 64),
                ("relative_residual", C.c_double)]


class _OrcMt(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class Port:
    """The plain-C restatement (oracle/_ref/liboracle_port.so)."""

    def __init__(self, path: str = PORT_SO):
        build_if_missing()
        self.lib = C.CDLL(path)
        self.lib.orc_uniform01.restype = C.c_double
        self.lib.orc_sum_sq.restype = C.c_double
        self.lib.orc_frobenius_norm.restype = C.c_double
        self.lib.orc_mt64_next.restype = C.c_uint64
        self.err = _OrcError()

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.err.subtype, self.err.msg.decode())

    def engine_raw(self, seed, stream, n):
        eng = _OrcMt()
        self.lib.orc_mt64_seeded(C.byref(eng), C.c_uint64(seed), C.c_uint32(stream))
        return np.array([self.lib.orc_mt64_next(C.byref(eng)) for _ in range(n)], dtype=np.uint64)

    def uniform01(self, seed, stream, n):
        eng = _OrcMt()
        self.lib.orc_mt64_seeded(C.byref(eng), C.c_uint64(seed), C.c_uint32(stream))
        return np.array([self.lib.orc_uniform01(C.byref(eng)) for _ in range(n)])

    def gaussian(self, seed, n, stream=0):
        out = np.zeros(n)
        self.lib.orc_gaussian_fill(C.c_uint64(seed), C.c_uint32(stream), _d(out), C.c_size_t(n))
        return out

    def frobenius_norm(self, t):
        t = flat(t)
        return self.lib.orc_frobenius_norm(_d(t), C.c_size_t(t.size))

    def relative_error(self, a, b):
        out = C.c_double(0)
        a = flat(a)
        self._check(self.lib.orc_relative_error(_d(a), _d(flat(b)), C.c_size_t(a.size),
                                                C.byref(out), C.byref(self.err)))
        return out.value

    def unfold_times(self, t, mode, m):
        t = fortran(t)
        m = fortran(m)
        out = np.zeros((_ext(t, mode), m.shape[1]), order="F")
        self._check(self.lib.orc_unfold_times(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                              C.c_int(mode), _d(flat(m)),
                                              C.c_size_t(m.shape[1]), _d(out),
                                              C.byref(self.err)))
        return out

    def unfold_t_times(self, t, mode, m):
        t = fortran(t)
        m = fortran(m)
        fibers = t.size // _ext(t, mode)
        out = np.zeros((fibers, m.shape[1]), order="F")
        self._check(self.lib.orc_unfold_t_times(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                                C.c_int(mode), _d(flat(m)),
                                                C.c_size_t(m.shape[1]), _d(out),
                                                C.byref(self.err)))
        return out

    def mode_n_product(self, t, u, mode):
        t = fortran(t)
        u = fortran(u)
        dims = list(t.shape)
        dims[mode - 1] = u.shape[0]
        out = np.zeros(dims, order="F")
        self._check(self.lib.orc_mode_n_product(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                                _d(flat(u)), C.c_size_t(u.shape[0]),
                                                C.c_size_t(u.shape[1]), C.c_int(mode), _d(out),
                                                C.byref(self.err)))
        return out

    def gram(self, a):
        a = fortran(a)
        g = np.zeros((a.shape[1], a.shape[1]), order="F")
        self.lib.orc_gram(_d(flat(a)), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]), _d(g))
        return g

    def reduced_qr(self, a):
        a = fortran(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        r = np.zeros((n, n), order="F")
        self._check(self.lib.orc_reduced_qr(_d(flat(a)), C.c_size_t(m), C.c_size_t(n), _d(q),
                                            _d(r), C.byref(self.err)))
        return q, r

    def spd_solve(self, g, b):
        g = fortran(g)
        b = fortran(b)
        x = np.zeros(b.shape, order="F")
        self._check(self.lib.orc_spd_solve(_d(flat(g)), C.c_size_t(g.shape[0]), _d(flat(b)),
                                           C.c_size_t(b.shape[1]), _d(x), C.byref(self.err)))
        return x

    def recover_singular_vectors(self, t, mode, q):
        t = fortran(t)
        q = fortran(q)
        out = np.zeros(q.shape, order="F")
        self._check(self.lib.orc_recover_singular_vectors(
            _d(flat(t)), C.c_int(t.ndim), _u64(t.shape), C.c_int(mode), _d(flat(q)),
            C.c_size_t(q.shape[0]), C.c_size_t(q.shape[1]), _d(out), C.byref(self.err)))
        return out

    def als_init(self, t, mode, r, seed):
        t = fortran(t)
        l = np.zeros((_ext(t, mode), r), order="F")
        self._check(self.lib.orc_als_init(_d(flat(t)), C.c_int(t.ndim), _u64(t.shape),
                                          C.c_int(mode), C.c_size_t(r), C.c_uint64(seed), _d(l),
                                          C.byref(self.err)))
        return l

    def als_low_rank(self, t, mode, r, eta=1e-4, max_iters=50, seed=0, init=None):
        t = fortran(t)
        fibers = t.size // _ext(t, mode)
        l = np.zeros((_ext(t, mode), r), order="F")
        rr = np.zeros((fibers, r), order="F")
        rep = _OrcAls()
        self._check(self.lib.orc_als_low_rank(
            _d(flat(t)), C.c_int(t.ndim), _u64(t.shape), C.c_int(mode), C.c_size_t(r),
            C.c_double(eta), C.c_int(max_iters), C.c_uint64(seed),
            _d(flat(init)) if init is not None else None, _d(l), _d(rr), C.byref(rep),
            C.byref(self.err)))
        rec = ModeRecord(mode, rep.iterations, rep.status, rep.achieved_eta,
                         list(rep.history[: min(rep.iterations, 64)]))
        return l, rr, rec

    def select_order(self, ranks):
        out = (C.c_int * len(ranks))()
        self.lib.orc_select_order(C.c_int(len(ranks)), _u64(ranks), out)
        return list(out)

    def hosvd_als(self, t, ranks, sequential=False, order=None, eta=1e-4, max_iters=50,
                  seed=0, want_singular_vectors=False):
        t = fortran(t)
        n = t.ndim
        core = np.zeros(ranks, order="F")
        total = sum(int(t.shape[k]) * int(ranks[k]) for k in range(n))
        fac = np.zeros(total)
        rep = _OrcHosvd()
        mo = (C.c_int * n)(*order) if order is not None else None
        self._check(self.lib.orc_hosvd_als(
            C.c_int(1 if sequential else (2 if want_singular_vectors else 0)), _d(flat(t)), C.c_int(n), _u64(t.shape),
            _u64(ranks), mo, C.c_double(eta), C.c_int(max_iters), C.c_uint64(seed), _d(core),
            _d(fac), C.byref(rep), C.byref(self.err)))
        factors = []
        ofs = 0
        for k in range(n):
            sz = int(t.shape[k]) * int(ranks[k])
            factors.append(fac[ofs:ofs + sz].reshape((t.shape[k], ranks[k]), order="F"))
            ofs += sz
        per_mode = []
        for p in range(n):
            a = rep.als[p]
            per_mode.append(ModeRecord(rep.modes[p], a.iterations, a.status, a.achieved_eta,
                                       list(a.history[: min(a.iterations, 64)])))
        return HosvdResult(core, factors, per_mode, rep.relative_residual)


# -- seeded builders mirroring tests/helpers.hpp (via the reference RNG) -------
def random_tensor(ref: Ref, dims, seed):
    """helpers.hpp:34-41: uniform_in(-1, 1) in storage order."""
    n = int(np.prod(dims))
    return ref.uniform_in(seed, -1.0, 1.0, n).reshape(dims, order="F")


def random_matrix(ref: Ref, rows, cols, seed):
    """helpers.hpp:43-53."""
    return ref.uniform_in(seed, -1.0, 1.0, rows * cols).reshape((rows, cols), order="F")


def random_gaussian(ref: Ref, rows, cols, seed):
    """helpers.hpp:55-63."""
    return ref.gaussian(seed, rows * cols).reshape((rows, cols), order="F")


def random_orthonormal(ref: Ref, rows, cols, seed):
    """helpers.hpp:66-70."""
    return ref.reduced_qr(random_gaussian(ref, rows, cols, seed))[0]


def counting_tensor(dims):
    """helpers.hpp:24-31."""
    n = int(np.prod(dims))
    return np.arange(1, n + 1, dtype=np.float64).reshape(dims, order="F")
