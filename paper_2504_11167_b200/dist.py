"""Multi-GPU plumbing: one process per GPU, partitions sharded across the ranks.

The CUDA library (``lrs_factorize_dist``) owns all the numerical work and calls back
into this module for its two exchange primitives (``include/lrspike_capi.h``
``lrs_comm``):

* ``allgather``: the per-partition dot-product partials (C4) and the small setup
  agreements, summed on every GPU in global partition order -- bit-identical iterates
  for any GPU count;
* ``sendrecv``: neighbour exchanges -- the rank-r interface messages of every apply
  (C1), the b-row SpMV halos (C3) and the cross-interface spike tips at setup (C5).

Backends: ``nccl`` uses the device buffers in place (NVLink / NVSwitch); any other
backend (``gloo``) stages through host memory, which lets several ranks share one GPU
in tests (no kernel of one rank ever waits on another rank's kernel: every cross-rank
dependency is a host-synchronous callback).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import api

_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_int64)
_SENDRECV = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                             ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32)


_NEIGHBORS = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class CommC(ctypes.Structure):
    """lrs_comm (include/lrspike_capi.h); host callbacks: neighbors NULL, stream_ordered 0."""

    _fields_ = [("rank", ctypes.c_int32), ("size", ctypes.c_int32), ("user", ctypes.c_void_p),
                ("allgather", _ALLGATHER), ("sendrecv", _SENDRECV), ("neighbors", _NEIGHBORS),
                ("stream_ordered", ctypes.c_int32)]


class _DevArray:
    """Zero-copy view of a raw device pointer for torch.as_tensor."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def shard_plan(n: int, p: int, size: int, rank: int):
    """(p_lo, p_hi, row_lo, row_hi) of ``rank`` -- contiguous balanced partition blocks."""
    L = api.lib()
    L.lrs_shard_plan.restype = ctypes.c_int32
    L.lrs_shard_plan.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32] + \
        [ctypes.POINTER(ctypes.c_int64)] * 4
    out = [ctypes.c_int64() for _ in range(4)]
    api._check(L.lrs_shard_plan(n, p, size, rank, *[ctypes.byref(o) for o in out]))
    return tuple(o.value for o in out)


class TorchComm:
    """``lrs_comm`` over a torch.distributed process group.

    ``device_buffers``: the library hands device pointers (True, the GPU library) or host
    pointers (False, CPU tests of the exchange semantics)."""

    def __init__(self, group=None, device_buffers: bool = True, stream_ordered: bool = False):
        """stream_ordered (NCCL on device buffers only): the library's context stream is
        torch's current stream, so a collective enqueued by torch is ordered with the
        library's kernels without a host synchronization on either side."""
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.device_buffers = device_buffers
        self.stream_ordered = bool(stream_ordered and self.nccl and device_buffers)
        self._ag = _ALLGATHER(self._allgather)
        self._sr = _SENDRECV(self._sendrecv)
        self.c = CommC(self.rank, self.size, None, self._ag, self._sr, _NEIGHBORS(),
                       1 if self.stream_ordered else 0)
        self.calls = {"allgather": 0, "sendrecv": 0, "bytes": 0}

    # -- buffer views ---------------------------------------------------------------------
    def _view(self, ptr, count):
        torch = self.torch
        if count == 0:
            return None
        if self.device_buffers:
            t = torch.as_tensor(_DevArray(ptr, count), device="cuda")
            return t if self.nccl else t.cpu()
        arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)),
                                    shape=(count,))
        return torch.from_numpy(arr)

    def _writeback(self, ptr, count, t):
        if count == 0 or (self.device_buffers and self.nccl) or not self.device_buffers:
            return  # written in place
        dst = self.torch.as_tensor(_DevArray(ptr, count), device="cuda")
        dst.copy_(t)
        self.torch.cuda.synchronize()

    # -- callbacks --------------------------------------------------------------------------
    def _allgather(self, user, send, recv, count):
        try:
            s = self._view(send, count)
            r = self._view(recv, count * self.size)
            if self.device_buffers and not self.nccl:
                r = self.torch.empty(count * self.size, dtype=self.torch.float64)
            self.dist.all_gather_into_tensor(r, s, group=self.group)
            if self.device_buffers and self.nccl and not self.stream_ordered:
                self.torch.cuda.synchronize()
            self._writeback(recv, count * self.size, r)
            self.calls["allgather"] += 1
            self.calls["bytes"] += 8 * count * self.size
            return 0
        except Exception as e:  # never let an exception cross the C boundary
            print(f"[lrs dist] allgather failed: {e}")
            return 1

    def _sendrecv(self, user, send, scount, dest, recv, rcount, source):
        try:
            ops = []
            s = r = None
            if dest >= 0 and scount > 0:
                s = self._view(send, scount)
                ops.append(self.dist.P2POp(self.dist.isend, s, dest, group=self.group))
            if source >= 0 and rcount > 0:
                r = self._view(recv, rcount)
                if self.device_buffers and not self.nccl:
                    r = self.torch.empty(rcount, dtype=self.torch.float64)
                ops.append(self.dist.P2POp(self.dist.irecv, r, source, group=self.group))
            if ops:
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()
                if self.device_buffers and self.nccl and not self.stream_ordered:
                    self.torch.cuda.synchronize()
            if r is not None:
                self._writeback(recv, rcount, r)
            self.calls["sendrecv"] += 1
            self.calls["bytes"] += 8 * (scount if dest >= 0 else 0)
            return 0
        except Exception as e:
            print(f"[lrs dist] sendrecv failed: {e}")
            return 1


class LibNcclComm:
    """The in-library NCCL data plane (lrs_comm_nccl_create, csrc/comm_nccl.cu): grouped
    ncclSend / ncclRecv and ncclAllGather enqueued on the context stream, no host callbacks.
    torch.distributed only carries the 128-byte ncclUniqueId from rank 0 to the others.
    Must outlive the factorizations built on it."""

    def __init__(self, ctx: api.Context, group=None):
        import torch.distributed as dist

        L = api.lib()
        L.lrs_comm_nccl_unique_id.restype = ctypes.c_int32
        L.lrs_comm_nccl_unique_id.argtypes = [ctypes.c_void_p]
        L.lrs_comm_nccl_create.restype = ctypes.c_int32
        L.lrs_comm_nccl_create.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.POINTER(ctypes.POINTER(CommC))]
        L.lrs_comm_nccl_destroy.restype = None
        L.lrs_comm_nccl_destroy.argtypes = [ctypes.POINTER(CommC)]
        import torch

        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.size = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            api._check(L.lrs_comm_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        ctypes.memmove(uid, obj[0], 128)
        self._p = ctypes.POINTER(CommC)()
        api._check(L.lrs_comm_nccl_create(ctx.h, uid, self.rank, self.size,
                                          ctypes.byref(self._p)), ctx.h)
        self.c = self._p.contents

    def close(self):
        if self._p:
            api.lib().lrs_comm_nccl_destroy(self._p)
            self._p = None


class DistFactorization(api.SpikeFactorization):
    """``lrs_factorize_dist`` on this rank's shard (collective over the group)."""

    def __init__(self, ctx: api.Context, A: api.CsrMatrix, cfg: api.SolverConfig, comm: TorchComm):
        L = api.lib()
        L.lrs_factorize_dist.restype = ctypes.c_int32
        L.lrs_factorize_dist.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.POINTER(api.SolverCfgC), ctypes.POINTER(CommC),
                                         ctypes.POINTER(ctypes.c_void_p)]
        self.ctx, self.A, self.cfg, self.comm = ctx, A, cfg, comm
        h = ctypes.c_void_p()
        c = cfg.c()
        api._check(L.lrs_factorize_dist(ctx.h, A.h, ctypes.byref(c), ctypes.byref(comm.c),
                                        ctypes.byref(h)), ctx.h)
        self.h = h
        inf = api.FactInfoC()
        api._check(L.lrs_fact_get_info(h, ctypes.byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in api.FactInfoC._fields_}
        P = self.info["p"]
        sz, of = (ctypes.c_int64 * P)(), (ctypes.c_int64 * P)()
        api._check(L.lrs_fact_get_layout(h, sz, of))
        self.sizes, self.offsets = list(sz), list(of)
        self.p_lo, self.p_hi, self.row_lo, self.row_hi = shard_plan(A.n, P, comm.size, comm.rank)


def gather_rows(x, row_lo: int, row_hi: int, n: int, comm: TorchComm):
    """Assemble the full solution from every rank's rows (host numpy, column-major)."""
    torch, dist = comm.torch, comm.dist
    x = np.asarray(x)
    local = np.ascontiguousarray(x[row_lo:row_hi])
    parts = [None] * comm.size
    dist.all_gather_object(parts, (row_lo, row_hi, local), group=comm.group)
    out = np.empty_like(x)
    for lo, hi, blk in parts:
        out[lo:hi] = blk
    del torch
    return out
