"""Sharded t-HOSVD-ALS / st-HOSVD-ALS: one process (or thread) per GPU.

The global tensor is split along its LAST mode with the balanced
``shard_range``; every rank passes its slab and the GLOBAL dims and gets the
same TuckerTensor / DecompositionReport back as the single-GPU call on the
whole tensor would give (core and factors replicated). The reference
(hosvd.hpp:55-70) is single-process; this module keeps its argument and
result types and adds only the slab.

Communicators:
  * ``ShardedContext.nccl(device, rank, world, uid)``: NCCL over NVLink (the
    library dlopens libnccl.so.2); ``uid`` from ``nccl_unique_id()`` on one
    rank, broadcast with ``broadcast_unique_id`` (torch.distributed, any
    backend).
  * ``ShardedContext.local(device, group, rank)``: ranks that are threads of
    one process sharing a device (host-synchronous collectives), for tests.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .tenkit import (Context, DimensionMismatchError, FactorEngine, InvalidModeError, ModeOrder, Truncation,
                     _cfg, _decomp_report, _flat_ptr, _host, _raise)


def shard_range(extent: int, rank: int, world: int) -> Tuple[int, int]:
    """(begin, len) of rank's slab: floor(extent*rank/world) .. floor(extent*(rank+1)/world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    b = extent * rank // world
    return b, extent * (rank + 1) // world - b


def slab_of(a: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Rank's slab (last mode) of a full column-major tensor."""
    a = _host(a)
    b, n = shard_range(a.shape[-1], rank, world)
    return np.asfortranarray(a[..., b:b + n])


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    err = _lib.TkgError()
    _raise(_lib.lib().tkg_nccl_unique_id(buf, C.byref(err)), err)
    return bytes(buf)


def broadcast_unique_id(rank: int, src: int = 0, make=nccl_unique_id) -> bytes:
    """NCCL unique id created on `src` and broadcast over torch.distributed
    (any backend)."""
    import torch.distributed as dist
    obj = [make() if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def fiber_window(dims: Sequence[int], mode: int, sharded: int, begin: int, length: int):
    """Python mirror of the engine's fiber_window (engine_dist.cpp): global
    fiber index j of `mode` = jlo + Plo*(ism + Gsm*jhi) with ism the index
    along the sharded mode; the shard's local fiber order is
    jlo + Plo*((ism - begin) + length*jhi). Returns (Fg, Plo, Gsm)."""
    Fg = int(np.prod(dims)) // int(dims[mode - 1])
    Plo = int(np.prod([dims[k] for k in range(sharded - 1) if k != mode - 1]))
    return Fg, Plo, int(dims[sharded - 1])


def local_to_global_fibers(dims: Sequence[int], mode: int, sharded: int, begin: int, length: int) -> np.ndarray:
    """Global fiber indices of the shard's fibers, in the shard's local order."""
    Fg, Plo, Gsm = fiber_window(dims, mode, sharded, begin, length)
    Fl = Fg // Gsm * length
    loc = np.arange(Fl)
    jlo, t = loc % Plo, loc // Plo
    ism, jhi = t % length + begin, t // length
    return jlo + Plo * (ism + Gsm * jhi)


class LocalGroup:
    """In-process group of `world` ranks (threads), see ShardedContext.local."""

    def __init__(self, world: int):
        self._l = _lib.lib()
        self._g = C.c_void_p()
        err = _lib.TkgError()
        _raise(self._l.tkg_local_group_create(int(world), C.byref(self._g), C.byref(err)), err)
        self.world = int(world)

    def close(self):
        if self._g:
            self._l.tkg_local_group_destroy(self._g)
            self._g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedContext:
    """One rank: a Context with a communicator attached."""

    def __init__(self, ctx: Context, rank: int, world: int, keep=None):
        self.ctx, self.rank, self.world = ctx, int(rank), int(world)
        self._keep = keep

    @classmethod
    def nccl(cls, device: int, rank: int, world: int, uid: bytes) -> "ShardedContext":
        ctx = Context(device)
        err = _lib.TkgError()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        _raise(ctx._l.tkg_comm_init_nccl(ctx._ctx, int(rank), int(world), buf, C.byref(err)), err)
        return cls(ctx, rank, world)

    @classmethod
    def shm(cls, device: int, name: str, rank: int, world: int, slot_bytes: int = 0) -> "ShardedContext":
        """One process per rank, collectives staged through the POSIX shared
        memory segment `name` ("/..."; the same on every rank) behind a
        process-shared barrier (csrc/comm.cpp ShmComm): the real per-process
        sharded path where the ranks have no NVLink peers (one-GPU pools,
        tests). Every rank must call this (the constructor is a barrier)."""
        ctx = Context(device)
        err = _lib.TkgError()
        _raise(ctx._l.tkg_comm_init_shm(ctx._ctx, name.encode(), int(rank), int(world), int(slot_bytes),
                                        C.byref(err)), err)
        return cls(ctx, rank, world)

    @classmethod
    def local(cls, device: int, group: LocalGroup, rank: int) -> "ShardedContext":
        ctx = Context(device)
        err = _lib.TkgError()
        _raise(ctx._l.tkg_comm_init_local(ctx._ctx, group._g, int(rank), C.byref(err)), err)
        return cls(ctx, rank, group.world, keep=group)

    def _slab(self, slab, dims: Sequence[int]):
        dims = tuple(int(d) for d in dims)
        b, n = shard_range(dims[-1], self.rank, self.world)
        ptr, on_dev, sdims, keep = Context._tensor(slab)
        if tuple(sdims) != dims[:-1] + (n,):
            raise DimensionMismatchError(f"rank {self.rank}: slab dims {tuple(sdims)} != {dims[:-1] + (n,)}")
        return ptr, on_dev, dims, b, n, keep

    def _run(self, sequential: bool, slab, dims, trunc: Truncation, order: Optional[ModeOrder],
             engine: FactorEngine, want_singular_vectors: bool = False):
        ptr, on_dev, dims, b, n, keep = self._slab(slab, dims)
        ranks = list(trunc.ranks)
        N = len(dims)
        if len(ranks) != N:
            raise DimensionMismatchError(f"truncation lists {len(ranks)} ranks for an order-{N} tensor")
        core = np.zeros(int(np.prod(ranks)))
        fac = np.zeros(sum(int(dims[k]) * int(ranks[k]) for k in range(N)))
        rep = _lib.TkgReport()
        err = _lib.TkgError()
        hold = []
        cfg = _cfg(engine.als, hold)
        l = self.ctx._l
        if sequential:
            mo = None
            if order is not None:
                if len(order.order) != N:
                    raise InvalidModeError(f"st_hosvd: order has {len(order.order)} entries for an order-{N} tensor")
                mo = _lib.u32([max(0, int(m)) for m in order.order])
            rc = l.tkg_st_hosvd_sharded(self.ctx._ctx, ptr, on_dev, N, _lib.u64(dims), b, n, _lib.u64(ranks), mo,
                                        C.byref(cfg), _flat_ptr(core), _flat_ptr(fac), C.byref(rep), C.byref(err))
        else:
            rc = l.tkg_t_hosvd_sharded(self.ctx._ctx, ptr, on_dev, N, _lib.u64(dims), b, n, _lib.u64(ranks),
                                       C.byref(cfg), int(bool(want_singular_vectors)), _flat_ptr(core),
                                       _flat_ptr(fac), C.byref(rep), C.byref(err))
        _raise(rc, err)
        return Context._tucker(core, fac, dims, ranks), _decomp_report(rep, self.ctx)

    def t_hosvd(self, slab, dims: Sequence[int], trunc: Truncation, engine: FactorEngine,
                want_singular_vectors: bool = False):
        return self._run(False, slab, dims, trunc, None, engine, want_singular_vectors)

    def st_hosvd(self, slab, dims: Sequence[int], trunc: Truncation, order: Optional[ModeOrder],
                 engine: FactorEngine):
        return self._run(True, slab, dims, trunc, order, engine)

    def close(self):
        self.ctx.close()
