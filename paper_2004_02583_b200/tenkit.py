"""Python mirror of the reference tenkit decomposition API on the B200 path.

Names, argument meaning and error behaviour follow the reference headers:
  t_hosvd / st_hosvd / select_order   include/tenkit/hosvd.hpp:55-76
  als_low_rank / als_init             include/tenkit/als.hpp:46-71
  unfold_times / unfold_t_times / mode_n_product / frobenius_norm /
  relative_error                      include/tenkit/tensor_ops.hpp:22-55
  reduced_qr / gram                   include/tenkit/kernels.hpp:23, matrix.hpp:49
  error classes                       include/tenkit/errors.hpp:10-77
Tensors are numpy arrays interpreted in column-major (Fortran) order, as
tenkit's DenseTensor (tensor.hpp:10-11), or `DeviceTensor` views of HBM
(e.g. a torch CUDA tensor holding the column-major data). Every call goes
through libtenkit_b200.so; there is no CPU implementation behind it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib

# ---- errors (errors.hpp:10-77) -------------------------------------------------
USAGE, IO, NUMERICAL = 0, 1, 2


class Error(RuntimeError):
    category = USAGE

    def __init__(self, message: str, code: int = 0, subtype: int = 0):
        super().__init__(message)
        self.code = code
        self.subtype = subtype


class InvalidModeError(Error):
    category = USAGE


class DimensionMismatchError(Error):
    category = USAGE


class ZeroReferenceError(Error):
    category = USAGE


class RankTooLargeError(Error):
    category = NUMERICAL


class SingularGramError(Error):
    category = NUMERICAL


class DegenerateInitError(Error):
    category = NUMERICAL


class NoConvergenceError(Error):
    category = NUMERICAL


class IoError(Error):
    category = IO


class FormatError(Error):
    category = IO


class DeviceError(Error):
    """CUDA runtime failure (no device, launch error). Category io."""
    category = IO


class UnsupportedError(Error):
    """Outside this build's limits (e.g. rank > 64). Category usage."""
    category = USAGE


_SUBTYPE = {1: InvalidModeError, 2: DimensionMismatchError, 3: ZeroReferenceError,
            4: RankTooLargeError, 5: SingularGramError, 6: DegenerateInitError,
            7: NoConvergenceError, 8: IoError, 9: FormatError, 11: DeviceError,
            12: UnsupportedError}


def _raise(rc: int, err: _lib.TkgError):
    if rc != 0:
        cls = _SUBTYPE.get(err.subtype, Error)
        raise cls(err.message.decode(errors="replace"), rc, err.subtype)


# ---- value types (als.hpp:17-38, hosvd.hpp:19-44, tensor_ops.hpp:59-67) -------
@dataclass
class AlsConfig:
    eta: float = 1e-4
    max_iters: int = 50
    seed: int = 0
    init: Optional[np.ndarray] = None


@dataclass
class FactorEngine:
    """FactorEngine (hosvd.hpp:19-27): kind "svd" (the reference's default),
    "eig" or "als"; `als` is used by the ALS engine only."""
    kind: str = "svd"
    als: AlsConfig = field(default_factory=AlsConfig)

    @staticmethod
    def with_als(cfg: AlsConfig) -> "FactorEngine":
        return FactorEngine("als", cfg)

    @staticmethod
    def svd() -> "FactorEngine":
        """hosvd.hpp:24: leading left singular vectors of the unfolding."""
        return FactorEngine("svd")

    @staticmethod
    def eig() -> "FactorEngine":
        """hosvd.hpp:25: leading eigenvectors of the mode Gram matrix."""
        return FactorEngine("eig")


@dataclass
class Truncation:
    ranks: List[int]


@dataclass
class ModeOrder:
    order: List[int]


@dataclass
class AlsReport:
    iterations: int = 0
    residual_history: List[float] = field(default_factory=list)
    status: str = "converged"  # or "max_iters_reached"
    achieved_eta: float = 0.0


@dataclass
class ModeReport:
    mode: int = 0
    seconds: float = 0.0
    als: Optional[AlsReport] = None


@dataclass
class DecompositionReport:
    per_mode: List[ModeReport] = field(default_factory=list)
    relative_residual: float = 0.0
    seconds: float = 0.0
    # device accounting (not in the reference struct)
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    residual_seconds: float = 0.0
    kernel_launches: int = 0
    tensor_passes: int = 0
    algorithmic_bytes: int = 0


@dataclass
class HooiConfig:
    """hooi.hpp:15-18."""
    tol: float = 1e-12
    max_iters: int = 100


@dataclass
class HooiResult:
    """hooi.hpp:20-31 (fit_history[0] = the warm start's fit)."""
    tucker: "TuckerTensor"
    iterations: int = 0
    fit_history: List[float] = field(default_factory=list)
    converged: bool = False
    relative_residual: float = 0.0


@dataclass
class TuckerTensor:
    core: np.ndarray
    factors: List[np.ndarray]
    origin_shape: tuple


class OwnedDeviceTensor:
    """A DeviceTensor whose HBM buffer belongs to the library (tkg_device_alloc);
    freed with the object."""

    def __init__(self, ptr: int, dims, ctx):
        self.ptr, self.dims, self._ctx = ptr, list(dims), ctx

    def __del__(self):
        try:
            if self.ptr and self._ctx._ctx:
                self._ctx._l.tkg_device_free(self._ctx._ctx, C.c_void_p(self.ptr))
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass
        self.ptr = 0


@dataclass
class DeviceTensor:
    """A column-major fp64 tensor already resident in HBM."""
    ptr: int
    dims: Sequence[int]

    @staticmethod
    def from_torch(t, dims: Sequence[int]) -> "DeviceTensor":
        """`t`: contiguous CUDA float64 tensor holding the column-major data."""
        assert t.is_cuda and t.dtype.itemsize == 8 and t.is_contiguous()
        assert t.numel() == int(np.prod(dims))
        return DeviceTensor(int(t.data_ptr()), tuple(int(d) for d in dims))


def _host(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _flat_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _full_history(m: _lib.TkgModeReport, ctx, position: int) -> List[float]:
    """One entry per sweep (als.cpp:137-138): the first TKG_MAX_HISTORY come
    inline in the report, the rest from tkg_residual_history."""
    hist = [m.residual_history[k] for k in range(m.history_len)]
    if ctx is not None and m.iterations > m.history_len:
        buf = np.zeros(int(m.iterations))
        n = C.c_uint64(0)
        err = _lib.TkgError()
        _raise(ctx._l.tkg_residual_history(ctx._ctx, int(position), _flat_ptr(buf), buf.size, C.byref(n),
                                           C.byref(err)), err)
        hist = list(buf[: int(n.value)])
    return hist


def _mode_report(m: _lib.TkgModeReport, ctx=None, position: int = 0) -> ModeReport:
    if m.status < 0:  # SVD / EIG engine: ModeReport::als is empty (hosvd.hpp:33-37)
        return ModeReport(m.mode, m.seconds, None)
    als = AlsReport(m.iterations, _full_history(m, ctx, position),
                    "converged" if m.status == 0 else "max_iters_reached", m.achieved_eta)
    return ModeReport(m.mode, m.seconds, als)


def _decomp_report(r: _lib.TkgReport, ctx=None) -> DecompositionReport:
    return DecompositionReport([_mode_report(r.per_mode[k], ctx, k) for k in range(r.n_modes)],
                               r.relative_residual, r.seconds, r.h2d_seconds, r.d2h_seconds,
                               r.residual_seconds, int(r.kernel_launches), int(r.tensor_passes),
                               int(r.algorithmic_bytes))


def _engine(e: "FactorEngine", keep):
    if e.kind not in _lib.ENGINE_KINDS:
        raise UnsupportedError(f"unknown factor engine kind {e.kind!r}")
    return _lib.TkgFactorEngine(_lib.ENGINE_KINDS[e.kind], _cfg(e.als, keep))


def _cfg(c: AlsConfig, keep):
    init, rows, cols = None, 0, 0
    if c.init is not None:
        arr = _host(c.init)
        keep.append(arr)
        init = _flat_ptr(arr)
        rows = arr.shape[0] if arr.ndim >= 1 else 1
        cols = (arr.shape[1] if arr.ndim >= 2 else 1) * int(np.prod(arr.shape[2:]) if arr.ndim > 2 else 1)
    return _lib.TkgAlsConfig(float(c.eta), int(c.max_iters), int(c.seed) & (2**64 - 1), init, rows, cols)


class Context:
    """One device + stream + workspaces (tkg_ctx). Not thread-safe."""

    def __init__(self, device: int = 0):
        self._l = _lib.lib()
        self._ctx = C.c_void_p()
        err = _lib.TkgError()
        _raise(self._l.tkg_create(C.byref(self._ctx), int(device), C.byref(err)), err)

    def close(self):
        if self._ctx:
            self._l.tkg_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- input marshalling --------------------------------------------------------
    @staticmethod
    def _tensor(t):
        if isinstance(t, (DeviceTensor, OwnedDeviceTensor)):
            return C.c_void_p(t.ptr), 1, tuple(t.dims), None
        a = _host(t)
        if a.ndim == 0:
            a = a.reshape(1)
        return C.c_void_p(a.ctypes.data), 0, a.shape, a

    # -- decomposition drivers ----------------------------------------------------
    def t_hosvd(self, t, trunc: Truncation, engine: FactorEngine,
                want_singular_vectors: bool = False):
        ptr, on_dev, dims, keep = self._tensor(t)
        ranks = list(trunc.ranks)
        n = len(dims)
        if len(ranks) != n:  # Truncation::validate (shape.cpp:57-60)
            raise DimensionMismatchError(f"truncation lists {len(ranks)} ranks for an order-{n} tensor")
        core = np.zeros(int(np.prod(ranks)))
        fac = np.zeros(sum(int(dims[k]) * int(ranks[k]) for k in range(n)))
        rep = _lib.TkgReport()
        err = _lib.TkgError()
        hold = []
        eng = _engine(engine, hold)
        rc = self._l.tkg_t_hosvd_engine(self._ctx, ptr, on_dev, n, _lib.u64(dims), _lib.u64(ranks),
                                        C.byref(eng), int(bool(want_singular_vectors)), _flat_ptr(core),
                                        _flat_ptr(fac), C.byref(rep), C.byref(err))
        _raise(rc, err)
        return self._tucker(core, fac, dims, ranks), _decomp_report(rep, self)

    def st_hosvd(self, t, trunc: Truncation, order: Optional[ModeOrder], engine: FactorEngine):
        ptr, on_dev, dims, keep = self._tensor(t)
        ranks = list(trunc.ranks)
        n = len(dims)
        if len(ranks) != n:
            raise DimensionMismatchError(f"truncation lists {len(ranks)} ranks for an order-{n} tensor")
        core = np.zeros(int(np.prod(ranks)))
        fac = np.zeros(sum(int(dims[k]) * int(ranks[k]) for k in range(n)))
        rep = _lib.TkgReport()
        err = _lib.TkgError()
        hold = []
        eng = _engine(engine, hold)
        mo = None
        if order is not None:
            if len(order.order) != n:
                raise InvalidModeError(f"st_hosvd: order has {len(order.order)} entries for an order-{n} tensor")
            mo = _lib.u32([max(0, int(m)) for m in order.order])
        rc = self._l.tkg_st_hosvd_engine(self._ctx, ptr, on_dev, n, _lib.u64(dims), _lib.u64(ranks), mo,
                                         C.byref(eng), _flat_ptr(core), _flat_ptr(fac), C.byref(rep),
                                         C.byref(err))
        _raise(rc, err)
        return self._tucker(core, fac, dims, ranks), _decomp_report(rep, self)

    @staticmethod
    def _tucker(core, fac, dims, ranks):
        factors = []
        ofs = 0
        for k in range(len(dims)):
            sz = int(dims[k]) * int(ranks[k])
            factors.append(fac[ofs:ofs + sz].reshape((dims[k], ranks[k]), order="F").copy())
            ofs += sz
        return TuckerTensor(core.reshape(tuple(ranks), order="F"), factors, tuple(dims))

    def als_low_rank(self, t, mode: int, r: int, cfg: AlsConfig):
        ptr, on_dev, dims, keep = self._tensor(t)
        n = len(dims)
        ext = dims[mode - 1] if 1 <= mode <= n else 1
        fibers = int(np.prod(dims)) // max(1, ext)
        l = np.zeros((ext, max(1, r)), order="F")
        rr = np.zeros((fibers, max(1, r)), order="F")
        rep = _lib.TkgModeReport()
        err = _lib.TkgError()
        hold = []
        c = _cfg(cfg, hold)  # init's shape travels with it; the library checks it (als.cpp:106-113)
        rc = self._l.tkg_als_low_rank(self._ctx, ptr, on_dev, n, _lib.u64(dims), int(mode), int(r),
                                      C.byref(c), _flat_ptr(l), _flat_ptr(rr), C.byref(rep),
                                      C.byref(err))
        _raise(rc, err)
        m = _mode_report(rep, self, 0)
        return (l, rr), m.als

    def als_init(self, t, mode: int, r: int, seed: int):
        ptr, on_dev, dims, keep = self._tensor(t)
        n = len(dims)
        ext = dims[mode - 1] if 1 <= mode <= n else 1
        l = np.zeros((ext, max(1, r)), order="F")
        err = _lib.TkgError()
        rc = self._l.tkg_als_init(self._ctx, ptr, on_dev, n, _lib.u64(dims), int(mode), int(r),
                                  int(seed) & (2**64 - 1), _flat_ptr(l), C.byref(err))
        _raise(rc, err)
        return l

    # -- primitives ---------------------------------------------------------------
    def unfold_times(self, t, mode: int, m):
        a = _host(t)
        m = _host(m)
        ext = a.shape[mode - 1] if 1 <= mode <= a.ndim else 1
        out = np.zeros((ext, m.shape[1]), order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_unfold_times(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape), int(mode),
                                        _flat_ptr(m), m.shape[1], _flat_ptr(out), C.byref(err)), err)
        return out

    def unfold_t_times(self, t, mode: int, m):
        a = _host(t)
        m = _host(m)
        ext = a.shape[mode - 1] if 1 <= mode <= a.ndim else 1
        out = np.zeros((a.size // max(1, ext), m.shape[1]), order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_unfold_t_times(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape),
                                          int(mode), _flat_ptr(m), m.shape[1], _flat_ptr(out),
                                          C.byref(err)), err)
        return out

    def mode_n_product(self, t, u, mode: int):
        a = _host(t)
        u = _host(u)
        dims = list(a.shape)
        if 1 <= mode <= a.ndim:
            dims[mode - 1] = u.shape[0]
        out = np.zeros(dims, order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_mode_n_product(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape),
                                          _flat_ptr(u), u.shape[0], u.shape[1], int(mode),
                                          _flat_ptr(out), C.byref(err)), err)
        return out

    def frobenius_norm(self, t) -> float:
        a = _host(t)
        out = C.c_double(0)
        err = _lib.TkgError()
        _raise(self._l.tkg_frobenius_norm(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape),
                                          C.byref(out), C.byref(err)), err)
        return out.value

    def relative_error(self, a, b) -> float:
        a = _host(a)
        b = _host(b)
        if a.shape != b.shape:
            raise DimensionMismatchError(f"relative_error: shapes {a.shape} vs {b.shape}")
        out = C.c_double(0)
        err = _lib.TkgError()
        _raise(self._l.tkg_relative_error(self._ctx, _flat_ptr(a), _flat_ptr(b), a.ndim,
                                          _lib.u64(a.shape), C.byref(out), C.byref(err)), err)
        return out.value

    def reduced_qr(self, a):
        a = _host(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        r = np.zeros((n, n), order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_reduced_qr(self._ctx, _flat_ptr(a), m, n, _flat_ptr(q), _flat_ptr(r),
                                      C.byref(err)), err)
        return q, r

    def gram(self, a):
        a = _host(a)
        g = np.zeros((a.shape[1], a.shape[1]), order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_gram(self._ctx, _flat_ptr(a), a.shape[0], a.shape[1], _flat_ptr(g),
                                C.byref(err)), err)
        return g

    def hooi(self, t, trunc: Truncation, init: "TuckerTensor", cfg: HooiConfig = None) -> HooiResult:
        """hooi.cpp:53-110: refine a conformal warm start (check_conformal :17-40)."""
        cfg = cfg or HooiConfig()
        ptr, on_dev, dims, keep = self._tensor(t)
        ranks = list(trunc.ranks)
        n = len(dims)
        if len(ranks) != n:
            raise DimensionMismatchError(f"truncation lists {len(ranks)} ranks for an order-{n} tensor")
        origin = tuple(int(x) for x in (init.origin_shape if init.origin_shape is not None else ()))
        if origin != tuple(dims):
            raise DimensionMismatchError(f"hooi: init origin shape {origin} does not match tensor {tuple(dims)}")
        core0 = np.asarray(init.core)
        if len(init.factors) != n or core0.ndim != n:
            raise DimensionMismatchError(f"hooi: init is not an order-{n} decomposition")
        for mode in range(1, n + 1):
            u = np.asarray(init.factors[mode - 1])
            if u.shape != (dims[mode - 1], ranks[mode - 1]) or core0.shape[mode - 1] != ranks[mode - 1]:
                raise DimensionMismatchError(f"hooi: init factor for mode {mode} does not match the truncation")
        c_in = np.ascontiguousarray(core0.reshape(-1, order="F"), dtype=np.float64)
        f_in = np.concatenate([np.asarray(u, dtype=np.float64).reshape(-1, order="F") for u in init.factors])
        core = np.zeros(int(np.prod(ranks)))
        fac = np.zeros(sum(int(dims[k]) * int(ranks[k]) for k in range(n)))
        fits = np.zeros(max(1, int(cfg.max_iters)) + 1)
        iters, conv, rr = C.c_int32(0), C.c_int32(0), C.c_double(0)
        err = _lib.TkgError()
        _raise(self._l.tkg_hooi(self._ctx, ptr, on_dev, n, _lib.u64(dims), _lib.u64(ranks), _flat_ptr(c_in),
                                _flat_ptr(f_in), float(cfg.tol), int(cfg.max_iters), _flat_ptr(core),
                                _flat_ptr(fac), C.byref(iters), C.byref(conv), _flat_ptr(fits), C.byref(rr),
                                C.byref(err)), err)
        return HooiResult(self._tucker(core, fac, dims, ranks), int(iters.value),
                          list(fits[: iters.value + 1]), bool(conv.value), relative_residual=rr.value)

    def read_tnsr(self, path: str, device: bool = True):
        """read_tnsr (io.cpp:150-161). device=True: the payload goes straight
        into HBM through pinned chunks and a DeviceTensor (owning its buffer)
        is returned; else a host numpy array."""
        order, dims = C.c_int32(0), (C.c_uint64 * _lib.MAX_ORDER)()
        err = _lib.TkgError()
        _raise(self._l.tkg_read_tnsr_shape(os.fsencode(path), C.byref(order), dims, C.byref(err)), err)
        shape = [int(dims[k]) for k in range(order.value)]
        n = int(np.prod(shape))
        if not device:
            out = np.zeros(shape, order="F")
            _raise(self._l.tkg_read_tnsr(self._ctx, os.fsencode(path), out.ctypes.data, 0, C.byref(err)), err)
            return out
        ptr = C.c_void_p()
        _raise(self._l.tkg_device_alloc(self._ctx, n * 8, C.byref(ptr), C.byref(err)), err)
        rc = self._l.tkg_read_tnsr(self._ctx, os.fsencode(path), ptr, 1, C.byref(err))
        if rc:
            self._l.tkg_device_free(self._ctx, ptr)
            _raise(rc, err)
        return OwnedDeviceTensor(int(ptr.value), shape, self)

    def write_tukr(self, path: str, tucker: "TuckerTensor"):
        """write_tukr (io.cpp:163-193)."""
        dims = [int(x) for x in tucker.origin_shape]
        ranks = list(np.asarray(tucker.core).shape)
        core = np.ascontiguousarray(np.asarray(tucker.core).reshape(-1, order="F"))
        fac = np.concatenate([np.asarray(u, dtype=np.float64).reshape(-1, order="F") for u in tucker.factors])
        err = _lib.TkgError()
        _raise(self._l.tkg_write_tukr(os.fsencode(path), len(dims), _lib.u64(dims), _lib.u64(ranks),
                                      _flat_ptr(core), _flat_ptr(fac), C.byref(err)), err)

    def multi_mode_product(self, t, factors):
        """tensor_ops.cpp:171-191: factors is a list of (matrix rows x I_mode, mode)."""
        a = _host(t)
        mats = [np.asfortranarray(np.asarray(u, dtype=np.float64)) for u, _ in factors]
        modes = [int(m) for _, m in factors]
        dims = list(a.shape)
        for u, m in zip(mats, modes):
            if 1 <= m <= a.ndim:
                dims[m - 1] = u.shape[0]
        out = np.zeros(dims, order="F")
        n = len(mats)
        ptrs = (_lib._dp * max(1, n))(*[_flat_ptr(u) for u in mats])
        err = _lib.TkgError()
        _raise(self._l.tkg_multi_mode_product(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape), n,
                                              _lib.u32(modes), ptrs, _lib.u64([u.shape[0] for u in mats]),
                                              _lib.u64([u.shape[1] for u in mats]), _flat_ptr(out),
                                              C.byref(err)), err)
        return out

    def reconstruct(self, tucker: "TuckerTensor"):
        """tensor_ops.cpp:420-440."""
        core = np.asfortranarray(np.asarray(tucker.core, dtype=np.float64))
        ranks = list(core.shape)
        dims = [int(x) for x in tucker.origin_shape]
        if len(tucker.factors) != core.ndim:
            raise DimensionMismatchError(f"reconstruct: {len(tucker.factors)} factors for an order-{core.ndim} core")
        for n, u in enumerate(tucker.factors):
            if np.asarray(u).shape != (dims[n], ranks[n]):
                raise DimensionMismatchError(f"reconstruct: factor {n + 1} is {np.asarray(u).shape}, "
                                             f"expected {(dims[n], ranks[n])}")
        fac = np.concatenate([np.asarray(u, dtype=np.float64).reshape(-1, order="F") for u in tucker.factors])
        out = np.zeros(dims, order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_reconstruct(self._ctx, _flat_ptr(core), core.ndim, _lib.u64(ranks), _lib.u64(dims),
                                       _flat_ptr(fac), _flat_ptr(out), C.byref(err)), err)
        return out

    def als_sweep(self, t, mode: int, l):
        """als.cpp:89-96: (FactorPair(l_next, r), residual after the right update)."""
        a = _host(t)
        l = _host(l)
        ext = a.shape[mode - 1] if 1 <= mode <= a.ndim else 1
        r = l.shape[1]
        ln = np.zeros(l.shape, order="F")
        rr = np.zeros((a.size // max(1, ext), r), order="F")
        res = C.c_double(0)
        err = _lib.TkgError()
        _raise(self._l.tkg_als_sweep(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape), int(mode), _flat_ptr(l),
                                     r, _flat_ptr(ln), _flat_ptr(rr), C.byref(res), C.byref(err)), err)
        return (ln, rr), res.value

    def mode_gram(self, t, mode: int):
        """tensor_ops.cpp:332-389: A_(mode) A_(mode)^T."""
        a = _host(t)
        ext = a.shape[mode - 1] if 1 <= mode <= a.ndim else 1
        out = np.zeros((ext, ext), order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_mode_gram(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape), int(mode),
                                     _flat_ptr(out), C.byref(err)), err)
        return out

    def sym_eig(self, g, k: int):
        """kernels.cpp:448-604: the k leading eigenpairs, descending (values, n x k vectors)."""
        g = _host(g)
        n = g.shape[0]
        if g.ndim != 2 or g.shape[1] != n:
            raise DimensionMismatchError(f"sym_eig: matrix is {g.shape[0]}x{g.shape[1] if g.ndim > 1 else 1}")
        vals = np.zeros(int(k))
        vecs = np.zeros((n, int(k)), order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_sym_eig(self._ctx, _flat_ptr(g), n, int(k), _flat_ptr(vals), _flat_ptr(vecs),
                                   C.byref(err)), err)
        return vals, vecs

    def recover_singular_vectors(self, t, mode: int, q):
        """hosvd.cpp:65-72: q (I_mode x r, orthonormal) -> q V, V the left
        singular vectors of q^T A_(mode) (descending, dense_svd's signs)."""
        a = _host(t)
        q = _host(q)
        out = np.zeros(q.shape, order="F")
        err = _lib.TkgError()
        _raise(self._l.tkg_recover_singular_vectors(self._ctx, _flat_ptr(a), a.ndim, _lib.u64(a.shape),
                                                    int(mode), _flat_ptr(q), q.shape[0], q.shape[1],
                                                    _flat_ptr(out), C.byref(err)), err)
        return out

    def uniform01(self, seed: int, stream: int, n: int):
        out = np.zeros(n)
        err = _lib.TkgError()
        _raise(self._l.tkg_uniform01(self._ctx, int(seed) & (2**64 - 1), int(stream), int(n),
                                     _flat_ptr(out), C.byref(err)), err)
        return out

    def timer_start(self):
        self._l.tkg_timer_start(self._ctx)

    def timer_stop(self) -> float:
        ms = C.c_double(0)
        self._l.tkg_timer_stop(self._ctx, C.byref(ms))
        return ms.value

    def flush_l2(self):
        self._l.tkg_flush_l2(self._ctx)

    def set_profiling(self, on: bool):
        self._l.tkg_set_profiling(self._ctx, int(bool(on)))

    def set_fused_sweep(self, on: bool):
        """The fused sweep pass for ranks up to 16 (csrc/sweep_fused.cu) on / off."""
        self._l.tkg_set_fused_sweep(self._ctx, int(bool(on)))

    def kernel_stats(self):
        st = _lib.TkgKernelStats()
        self._l.tkg_get_kernel_stats(self._ctx, C.byref(st))
        names = ["fc", "fr", "small", "rng", "ttm", "residual", "sweep"]
        return {names[k]: {"ms": st.ms[k], "launches": int(st.launches[k]), "bytes": st.bytes[k],
                           "flops": st.flops[k]} for k in range(len(names))}


def select_order(trunc: Truncation, shape: Sequence[int]) -> ModeOrder:
    """hosvd.cpp:54-63 — stable ascending-rank order."""
    l = _lib.lib()
    n = len(shape)
    out = (C.c_uint32 * max(1, n))()
    err = _lib.TkgError()
    ranks = list(trunc.ranks)
    if len(ranks) != n:
        raise DimensionMismatchError(f"truncation lists {len(ranks)} ranks for an order-{n} tensor")
    _raise(l.tkg_select_order(n, _lib.u64(shape), _lib.u64(ranks), out, C.byref(err)), err)
    return ModeOrder([int(out[k]) for k in range(n)])


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def t_hosvd(t, trunc, engine, want_singular_vectors=False):
    return default_context().t_hosvd(t, trunc, engine, want_singular_vectors)


def st_hosvd(t, trunc, order, engine):
    return default_context().st_hosvd(t, trunc, order, engine)


def als_low_rank(t, mode, r, cfg):
    return default_context().als_low_rank(t, mode, r, cfg)


def als_init(t, mode, r, seed):
    return default_context().als_init(t, mode, r, seed)


def unfold_times(t, mode, m):
    return default_context().unfold_times(t, mode, m)


def unfold_t_times(t, mode, m):
    return default_context().unfold_t_times(t, mode, m)


def mode_n_product(t, u, mode):
    return default_context().mode_n_product(t, u, mode)


def frobenius_norm(t):
    return default_context().frobenius_norm(t)


def relative_error(a, b):
    return default_context().relative_error(a, b)


def reduced_qr(a):
    return default_context().reduced_qr(a)


def gram(a):
    return default_context().gram(a)


def hooi(t, trunc, init, cfg=None):
    return default_context().hooi(t, trunc, init, cfg)


def multi_mode_product(t, factors):
    return default_context().multi_mode_product(t, factors)


def reconstruct(tucker):
    return default_context().reconstruct(tucker)


def als_sweep(t, mode, l):
    return default_context().als_sweep(t, mode, l)


def mode_gram(t, mode):
    return default_context().mode_gram(t, mode)


def sym_eig(g, k):
    return default_context().sym_eig(g, k)


def recover_singular_vectors(t, mode, q):
    return default_context().recover_singular_vectors(t, mode, q)


def synth_tucker(dims, ranks, alpha: float, nu: float, seed: int, out: Optional[np.ndarray] = None):
    """Seeded synthetic Tucker tensor — input synthesis for
    benches/tests, host C++/OpenMP (csrc/synth.cpp). Returns a flat
    column-major array (or fills `out`)."""
    n = int(np.prod(dims))
    if out is None:
        out = np.empty(n)
    assert out.size == n and out.dtype == np.float64
    rc = _lib.synth_lib().tkg_synth_tucker(len(dims), _lib.u64(dims), _lib.u64(ranks), float(alpha),
                                            float(nu), int(seed),
                                            out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        raise DimensionMismatchError("synth_tucker: invalid dims/ranks")
    return out


def synth_tucker_slab(dims, ranks, alpha: float, nu: float, seed: int, begin: int, length: int,
                      out: Optional[np.ndarray] = None, combine=None):
    """Slab [begin, begin+length) of the last mode of synth_tucker(dims, ...),
    bit-identical to the same slice of the whole tensor. The noise scale
    needs per-slice sums from every slab: `combine(sums)` receives this
    slab's (length, 2) array and returns the (I_N, 2) array of all slices
    (e.g. an all-gather across ranks); None = this slab is the whole tensor."""
    dims = [int(d) for d in dims]
    sl = list(dims[:-1]) + [int(length)]
    n = int(np.prod(sl))
    if out is None:
        out = np.empty(n)
    assert out.size == n and out.dtype == np.float64
    h = _lib.synth_lib()
    sq = np.zeros((int(length), 2))
    dp = C.POINTER(C.c_double)
    rc = h.tkg_synth_tucker_slab(len(dims), _lib.u64(dims), _lib.u64(ranks), float(alpha), int(seed),
                                 int(begin), int(length), out.ctypes.data_as(dp), sq.ctypes.data_as(dp))
    if rc != 0:
        raise DimensionMismatchError("synth_tucker_slab: invalid dims/ranks/slab")
    allsq = np.ascontiguousarray(combine(sq) if combine is not None else sq, dtype=np.float64)
    if allsq.shape != (dims[-1], 2):
        raise DimensionMismatchError("synth_tucker_slab: combine must return (I_N, 2) slice sums")
    scale = h.tkg_synth_noise_scale(dims[-1], allsq.ctypes.data_as(dp), float(nu))
    h.tkg_synth_add_noise(len(dims), _lib.u64(dims), int(seed), int(begin), int(length), scale,
                          out.ctypes.data_as(dp))
    return out
