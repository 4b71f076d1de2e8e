"""Collectives of the SPD-KFAC step over NCCL (NVLink 5 / NVSwitch on B200).

`NcclComm` owns a communicator inside libspdkfac.so (include/spdkfac.h,
spdkfac_comm_*); the unique id is exchanged through the already-initialised
torch.distributed process group.  Every call is enqueued on the given CUDA
stream (the optimizer's communication side stream) and never blocks the host.
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from contextlib import contextmanager

import torch

from . import _lib as L


class NcclComm:
    def __init__(self, rank: int, world: int, uid: bytes | None = None):
        import torch.distributed as dist
        lib = L.load(require_device=True)
        if uid is None:
            buf = [None]
            if rank == 0:
                raw = (C.c_char * 128)()
                L.check(lib.spdkfac_comm_unique_id(raw), "nccl unique id")
                buf[0] = bytes(raw)
            dist.broadcast_object_list(buf, src=0)
            uid = buf[0]
        raw = (C.c_char * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        L.check(lib.spdkfac_comm_create(C.byref(h), raw, rank, world), "nccl comm create")
        self._h, self._lib, self.rank, self.world = h, lib, rank, world
        # program order of collective launches, one tag ("factor" / "inverse" / "grad") per
        # NCCL kernel (a group is one); read by the measured breakdown (breakdown.py)
        self.log = deque(maxlen=4096)
        self._group_tag, self._in_group = None, False

    def _note(self, tag: str) -> None:
        if self._in_group:
            self._group_tag = self._group_tag or tag
        else:
            self.log.append(tag)

    def allreduce_sum(self, buf: torch.Tensor, stream, tag: str = "factor") -> None:
        self._note(tag)
        L.check(self._lib.spdkfac_comm_allreduce_sum_f32(self._h, buf.data_ptr(), buf.numel(), stream.cuda_stream),
                "all-reduce")

    def bcast(self, buf: torch.Tensor, root: int, stream, tag: str = "inverse") -> None:
        self._note(tag)
        L.check(self._lib.spdkfac_comm_bcast_f32(self._h, buf.data_ptr(), buf.numel(), int(root), stream.cuda_stream),
                "broadcast")

    def reduce_sum(self, buf: torch.Tensor, root: int, stream, tag: str = "factor") -> None:
        self._note(tag)
        L.check(self._lib.spdkfac_comm_reduce_sum_f32(self._h, buf.data_ptr(), buf.numel(), int(root),
                                                     stream.cuda_stream), "reduce")

    @contextmanager
    def group(self):
        L.check(self._lib.spdkfac_comm_group_start(), "group start")
        self._in_group, self._group_tag = True, None
        try:
            yield
        finally:
            self._in_group = False
            if self._group_tag is not None:
                self.log.append(self._group_tag)
            L.check(self._lib.spdkfac_comm_group_end(), "group end")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.spdkfac_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
