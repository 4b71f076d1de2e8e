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


def peer_layout(world: int, sizes: dict, n_slots: int, extra: int = 0) -> tuple:
    """Byte layout of one rank's peer allocation (identical on every rank): (offsets, strides, total).
    offsets["A"/"G"]: inbox [world][stride] fp32 after the flags [n_slots][world] int32; offsets["X"]: the
    `extra` fp32 receive region.  Regions start 256-byte aligned and the inbox row stride is a multiple of
    64 elements, so element s of any row shares the address mod 16 of element s of a 256-aligned buffer."""
    up = lambda x: (x + 255) // 256 * 256  # noqa: E731
    stride = {k: (int(v) + 63) // 64 * 64 for k, v in sizes.items()}
    off, pos = {}, up(max(1, n_slots * world) * 4)
    for kind in ("A", "G"):
        off[kind] = pos
        pos = up(pos + world * stride[kind] * 4)
    off["X"] = pos
    pos = up(pos + max(1, int(extra)) * 4)
    return off, stride, pos


class _DeviceArray:
    """fp32 device memory not owned by torch (the peer allocation), seen through __cuda_array_interface__."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerExchange:
    """Factor aggregation over NVLink peer memory (factor_comm = "peer", csrc/peer.cu).

    Each rank owns one device allocation, mapped into every other rank through CUDA IPC:
      flags  [n_slots][world] int32  flags[slot][q]: the epoch at which rank q's group `slot` landed
      inbox  per kind ("A", "G"): [world][size] fp32, row q = rank q's 1/P-scaled packed factors
    The packed factors of a CT inverse another rank owns reach `remote_ptr(owner, kind, offset)`
    by a push right after the group's SYRK (`push`: the copy engine, or SM stores with SPDKFAC_PEER_ENGINE=sm) or straight from the SYRK
    epilogue (FactorGroup member target = the remote address; SPDKFAC_PEER_PUSH=epilogue: the
    epilogue's per-row stores cross NVLink as 4-byte writes, measured slower); `signal` then raises
    this rank's flag in every peer, and the owner's `wait_sum` polls the group's flags and adds the
    P - 1 inbox rows into its own packed factors (the same sum an NCCL reduce onto the owner forms).
    `extra` elements after the inboxes hold the owners' CT inverses: each owner packs its inverses into its
    own region and pushes them into every peer's region (`push_extra`), then signals a per-side slot.
    `epoch` advances once per step on every rank (inside CUDA graphs too)."""

    def __init__(self, rank: int, world: int, sizes: dict, n_slots: int, device, timeout_s: float | None = None,
                 extra: int = 0):
        import os
        import torch.distributed as dist
        lib = L.load(require_device=True)
        if world > 8:
            raise ValueError("peer-memory aggregation spans one NVSwitch node (world <= 8)")
        self.sizes, self.rank, self.world, self.n_slots = dict(sizes), rank, world, n_slots
        # inbox row stride: a multiple of 64 elements, so row q at offset s shares the fusion buffer's alignment;
        # `extra` fp32 elements after the inboxes: the inverse receive regions (same layout on every rank)
        self._off, self.stride, off = peer_layout(world, sizes, n_slots, extra)
        own = C.c_void_p()
        L.check(lib.spdkfac_peer_alloc(off, C.byref(own)), "peer alloc")
        h = (C.c_char * 64)()
        L.check(lib.spdkfac_peer_handle(own, h), "peer handle")
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h))
        self.bases = []
        for q in range(world):
            if q == rank:
                self.bases.append(own.value)
                continue
            p = C.c_void_p()
            L.check(lib.spdkfac_peer_open((C.c_char * 64).from_buffer_copy(handles[q]), C.byref(p)), "peer open")
            self.bases.append(p.value)
        self._own, self._lib = own.value, lib
        self._flag_ptrs = (C.c_void_p * world)(*self.bases)
        self.extra = torch.as_tensor(_DeviceArray(own.value + self._off["X"], max(1, int(extra))), device=device)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        # factor pushes: "ce" (copy engine, overlapping the backward pass without SM time; measured best) or "sm"
        self.engine = os.environ.get("SPDKFAC_PEER_ENGINE", "ce")
        self.timeout_s = float(timeout_s if timeout_s is not None else os.environ.get("SPDKFAC_PEER_TIMEOUT_S", "60"))

    def remote_ptr(self, owner: int, kind: str, offset: int) -> int:
        """Address (in this process) of this rank's inbox row at `offset` elements inside `owner`'s buffer."""
        return self.bases[owner] + self._off[kind] + (self.rank * self.stride[kind] + int(offset)) * 4

    def _send(self, dsts, src: torch.Tensor, stream, engine: str) -> None:
        if engine == "ce":  # copy engine: no SM time, one engine's bandwidth per copy
            for dst in dsts:
                L.check(self._lib.spdkfac_peer_copy(dst, src.data_ptr(), src.numel() * 4, stream.cuda_stream),
                        "peer copy")
        else:  # SM stores over NVLink, every destination in one launch
            L.check(self._lib.spdkfac_peer_scatter_f32(L.ptr_array(dsts), len(dsts), src.data_ptr(), src.numel(),
                                                       stream.cuda_stream), "peer scatter")

    def push_extra_all(self, offset: int, src: torch.Tensor, stream) -> None:
        """Push `src` (this rank's extra region at `offset` elements) into the same place of every peer."""
        # SM stores: the inverses are pushed at the end of the critical path, where one copy engine per
        # destination was measured ~5 ms slower per step (N = 2)
        self._send([self.bases[q] + self._off["X"] + int(offset) * 4 for q in range(self.world) if q != self.rank],
                   src, stream, "sm")

    def push(self, owner: int, kind: str, offset: int, src: torch.Tensor, stream) -> None:
        """Push this rank's packed range `src` (at `offset` of its fusion buffer) into its inbox row in
        `owner`'s buffer, ordered on `stream`."""
        self._send([self.remote_ptr(owner, kind, offset)], src, stream, self.engine)

    def advance(self, stream) -> None:
        L.check(self._lib.spdkfac_peer_epoch_advance(self.epoch.data_ptr(), stream.cuda_stream), "peer epoch")

    def signal(self, slot: int, stream) -> None:
        L.check(self._lib.spdkfac_peer_signal(self._flag_ptrs, self.world, self.rank, int(slot), self.epoch.data_ptr(),
                                              stream.cuda_stream), "peer signal")

    def wait_sum(self, slot: int, kind: str, packed: torch.Tensor, segs: torch.Tensor | None, max_count: int,
                 stream) -> None:
        """Wait for group `slot` from every peer, then packed[s:s+n] += the peers' inbox rows for each
        (s, n) row of `segs` (int64 [k, 2] on the device; None: wait only)."""
        n = 0 if segs is None else int(segs.shape[0])
        L.check(self._lib.spdkfac_peer_wait_sum(
            self._own, self.world, self.rank, int(slot), self.epoch.data_ptr(), self.err.data_ptr(), self.timeout_s,
            packed.data_ptr(), self._own + self._off[kind], self.stride[kind], n,
            segs.data_ptr() if n else None, int(max_count), stream.cuda_stream), "peer wait/sum")

    def wait(self, slot: int, stream) -> None:
        """Wait (on `stream`) until every peer raised its flag of `slot` for this step."""
        L.check(self._lib.spdkfac_peer_wait_sum(
            self._own, self.world, self.rank, int(slot), self.epoch.data_ptr(), self.err.data_ptr(), self.timeout_s,
            None, None, 1, 0, None, 0, stream.cuda_stream), "peer wait")

    def error(self) -> int:
        """0, or 1 + the slot whose peer signals timed out (synchronises)."""
        return int(self.err.item())

    def close(self) -> None:
        if getattr(self, "_lib", None) is None:
            return
        torch.cuda.synchronize()
        for q, b in enumerate(self.bases):
            if q != self.rank:
                self._lib.spdkfac_peer_close(b)
        self._lib.spdkfac_peer_free(self._own)
        self._lib = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

