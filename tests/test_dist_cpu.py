"""Host-side logic of the sharded decomposition, on CPU with torch.distributed
(gloo, world_size 2; the GPU collectives are NCCL, tested in
test_gpu_dist.py): the balanced slab split, slab synthesis with the
cross-rank noise scale (bit-identical to the whole tensor), the unique-id
broadcast, the shard's fiber windows (which S draws a shard keeps), and the
algebra the engine distributes -- per-shard left-update partials and Gram
matrices summed over ranks equal the single-process ones."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2004_02583_b200 as tk
from paper_2004_02583_b200 import _lib
from paper_2004_02583_b200 import dist as tkd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _unfold(a, n):
    return np.reshape(np.moveaxis(a, n - 1, 0), (a.shape[n - 1], -1), order="F")


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # 1. unique-id broadcast (a fixed 128-byte token stands in for NCCL's)
        tok = tkd.broadcast_unique_id(rank, make=lambda: bytes(range(128)))
        out["uid_ok"] = tok == bytes(range(128))
        # 2. slab synthesis with the noise scale from every rank's slices
        dims, ranks = [14, 11, 9], [3, 4, 2]
        b, n = tkd.shard_range(dims[-1], rank, world)

        def combine(sq):
            full = torch.zeros((dims[-1], 2), dtype=torch.float64)
            full[b:b + n] = torch.from_numpy(sq)
            dist.all_reduce(full)
            return full.numpy()

        slab = tk.synth_tucker_slab(dims, ranks, 1.0, 1e-3, 77, b, n, combine=combine)
        full = tk.synth_tucker(dims, ranks, 1.0, 1e-3, 77).reshape(dims, order="F")
        out["slab_bitwise"] = bool(np.array_equal(slab.reshape(dims[:-1] + [n], order="F"), full[..., b:b + n]))
        # 3. distributed algebra of one ALS sweep of each mode != the sharded one
        rng = np.random.default_rng(5)
        ok = True
        for mode in (1, 2):
            A = _unfold(full, mode)                      # I x F (global fibers)
            loc = tkd.local_to_global_fibers(dims, mode, 3, b, n)
            Aloc = _unfold(full[..., b:b + n], mode)     # I x F_local, local fiber order
            ok &= bool(np.array_equal(Aloc, A[:, loc]))
            L = rng.standard_normal((dims[mode - 1], 2))
            R = A.T @ L                                  # right update, rows = fibers
            Rloc = Aloc.T @ L                            # local rows, no communication
            ok &= bool(np.allclose(Rloc, R[loc], rtol=1e-14, atol=1e-14))
            Y = torch.from_numpy(Aloc @ Rloc)            # left-update partial, summed
            G = torch.from_numpy(Rloc.T @ Rloc)          # Gram partial, summed
            dist.all_reduce(Y)
            dist.all_reduce(G)
            ok &= bool(np.allclose(Y.numpy(), A @ R, rtol=1e-12, atol=1e-12))
            ok &= bool(np.allclose(G.numpy(), R.T @ R, rtol=1e-12, atol=1e-12))
            # the initializer draws a shard keeps: S (F x r, column-major) rows loc
            Fg = A.shape[1]
            S = np.arange(Fg * 2, dtype=np.float64).reshape((Fg, 2), order="F")
            ok &= bool(np.array_equal(S[loc], np.stack([loc, loc + Fg], axis=1).astype(np.float64)))
        out["algebra"] = ok
        # 4. the moved mode: after re-sharding along mode 2, mode 3's fibers are local
        b2, n2 = tkd.shard_range(dims[1], rank, world)
        loc3 = tkd.local_to_global_fibers(dims, 3, 2, b2, n2)
        out["moved"] = bool(np.array_equal(_unfold(full[:, b2:b2 + n2, :], 3), _unfold(full, 3)[:, loc3]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    l = _lib.lib()
    for extent in (1, 7, 8, 1000, 1024):
        for world in (1, 2, 3, 8):
            if world > extent:
                continue
            cover = []
            for r in range(world):
                b, n = tkd.shard_range(extent, r, world)
                cb, cn = C.c_uint64(), C.c_uint64()
                assert l.tkg_shard_range(extent, r, world, C.byref(cb), C.byref(cn)) == 0
                assert (cb.value, cn.value) == (b, n)
                assert n in (extent // world, extent // world + 1)
                cover.extend(range(b, b + n))
            assert cover == list(range(extent))


def test_fiber_window_single_process():
    dims = [6, 5, 4, 3]
    a = np.arange(np.prod(dims), dtype=np.float64).reshape(dims, order="F")
    for sm in (2, 3, 4):
        for mode in range(1, 5):
            if mode == sm:
                continue
            for r in range(2):
                b, n = tkd.shard_range(dims[sm - 1], r, 2)
                sl = [slice(None)] * 4
                sl[sm - 1] = slice(b, b + n)
                loc = tkd.local_to_global_fibers(dims, mode, sm, b, n)
                assert np.array_equal(_unfold(a[tuple(sl)], mode), _unfold(a, mode)[:, loc])


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, out = q.get(timeout=180)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r] == {"uid_ok": True, "slab_bitwise": True, "algebra": True, "moved": True}, res[r]
