"""CUDA-graph capture of a whole SPD-KFAC training step.

One replay = zero_grad + forward (A-factor hooks: staging on the compute stream,
tensor-core SYRK on the factor stream, fusion-group all-reduces on the comm stream)
+ loss + backward (G-factor hooks) + SPDKFAC.step() (gradient all-reduce, inverses,
owner broadcasts, preconditioning + update).  Every kernel of the step, ours, cuDNN's
and NCCL's, is launched by one cudaGraphLaunch, so the host's per-step cost no longer
bounds the iteration (the eager step spends ~20-30 ms of Python/launch time per
ResNet-50 iteration, comparable to the GPU time).

Update frequencies (the reference's `kfac_update_interval`, simulator.py:126,377, split into
factor_update_freq f and inv_update_freq v, v a multiple of f): a step is one of three types --
factors + inversion (step % v == 0), factors only (step % f == 0), or reuse (neither: the step
preconditions with the stored inverses) -- and the optimizer's Python control flow differs per
type, so one graph is captured per type that occurs and each replay picks the graph of the
optimizer's current step.  Each graph has its own memory pool (they never run concurrently and
nothing produced by one replay is read by another: factors, inverses and staging buffers live
outside the pools).  Inputs are copied into static buffers.  Gradients are reset with
zero_grad(set_to_none=True): backward then writes each weight gradient straight into a graph-pool
tensor (no zero-fill and no accumulate-add kernel per parameter), and the replays reuse those
same addresses.

Input prefetch: `prefetch(inputs, targets)` starts the host->device copy of the NEXT step's batch
on a copy stream into one of two device staging slots while the current replay runs; the next
call without inputs waits for that copy and moves the slot into the static buffers with a
device-to-device copy (microseconds) before replaying -- the double-buffered loader pattern, so
the PCIe transfer of batch i+1 overlaps the compute of step i.

The learning rate is read when a graph is captured: the captured kernels carry it as an argument.
A changed `param_groups[0]["lr"]` raises at the next call unless `recapture_on_lr_change=True`,
which captures the graphs again (a scheduler stepping every iteration would recapture every
iteration -- use a constant lr or a schedule of a few plateaus with graphs).
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch


class GraphedStep:
    def __init__(self, model: torch.nn.Module, loss_fn: Callable, optimizer, inputs: Sequence[torch.Tensor],
                 targets: Sequence[torch.Tensor], warmup: int = 3, before_capture: Callable | None = None,
                 priority: int = 0, recapture_on_lr_change: bool = False):
        self.model, self.loss_fn, self.opt = model, loss_fn, optimizer
        self.f = int(getattr(optimizer, "factor_update_freq", 1))
        self.v = int(getattr(optimizer, "inv_update_freq", 1))
        self.static_in = [t.detach().clone() for t in inputs]
        self.static_tg = [t.detach().clone() for t in targets]
        # prefetch: two device staging slots for the next batch, filled on a copy stream
        self._copy_stream = torch.cuda.Stream()
        self._slots = [[torch.empty_like(t) for t in self.static_in + self.static_tg] for _ in range(2)]
        self._slot_free = [torch.cuda.Event(), torch.cuda.Event()]
        self._next_slot = 0
        self._pending = None  # (slot, copy-done event)
        self.priority = priority
        self.recapture = recapture_on_lr_change
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream(priority=priority)
        self.stream = side
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                self._body()
        cur.wait_stream(side)
        torch.cuda.synchronize()
        if before_capture is not None:
            before_capture()
        self._capture_all()

    def prefetch(self, inputs: Sequence[torch.Tensor], targets: Sequence[torch.Tensor]) -> None:
        """Start copying the next step's batch (pinned host or device tensors) into a device staging
        slot on the copy stream; the next call without inputs consumes it.  One batch is pending at a
        time (a second prefetch before the call replaces the first); the source tensors must stay
        alive until that call."""
        slot = self._next_slot
        self._next_slot ^= 1
        cs = self._copy_stream
        cs.wait_event(self._slot_free[slot])  # the D2D copy that last read this slot has run
        with torch.cuda.stream(cs):
            for d, t in zip(self._slots[slot], list(inputs) + list(targets)):
                d.copy_(t, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._pending = (slot, ev)

    def _type(self, step: int) -> tuple:
        return (step % self.f == 0, step % self.v == 0)

    def _capture_all(self):
        opt = self.opt
        real = getattr(opt, "steps", 0)
        self.graphs, self.losses = {}, {}
        self.lr = opt.param_groups[0]["lr"]
        for off in range(self.v):  # one representative step of every type in a period
            t = self._type(off)
            if t in self.graphs:
                continue
            if hasattr(opt, "steps"):  # the optimizer's control flow follows its step counter
                opt.steps = (real // self.v + 1) * self.v + off
                opt._capture = t[0]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream if self.priority else None):
                self.losses[t] = self._body()
            torch.cuda.synchronize()
            self.graphs[t] = g
        if hasattr(opt, "steps"):
            opt.steps = real
            opt._capture = real % self.f == 0
        self.static_loss = self.losses[self._type(real)]

    def _body(self):
        self.opt.zero_grad(set_to_none=True)
        loss = self.loss_fn(self.model(*self.static_in), *self.static_tg)
        loss.backward()
        self.opt.step()
        return loss

    def __call__(self, inputs: Sequence[torch.Tensor] | None = None, targets: Sequence[torch.Tensor] | None = None):
        """Copy new data into the static buffers (non-blocking, stream-ordered) and replay the
        graph of the optimizer's current step type."""
        if self.opt.param_groups[0]["lr"] != self.lr:
            if not self.recapture:
                raise RuntimeError("GraphedStep: the learning rate changed after capture (it is baked into the "
                                   "captured kernels); pass recapture_on_lr_change=True to capture again")
            torch.cuda.synchronize()
            self._capture_all()
        if inputs is not None:
            for s, t in zip(self.static_in, inputs):
                s.copy_(t, non_blocking=True)
        if targets is not None:
            for s, t in zip(self.static_tg, targets):
                s.copy_(t, non_blocking=True)
        if inputs is None and targets is None and self._pending is not None:  # the prefetched batch
            slot, ev = self._pending
            cur = torch.cuda.current_stream()
            cur.wait_event(ev)
            for s, t in zip(self.static_in + self.static_tg, self._slots[slot]):
                s.copy_(t, non_blocking=True)
            self._slot_free[slot].record(cur)
            self._pending = None
        step = getattr(self.opt, "steps", 0)
        t = self._type(step)
        self.graphs[t].replay()
        self.static_loss = self.losses[t]
        if hasattr(self.opt, "_after_replay"):
            self.opt._after_replay(torch.cuda.current_stream(), inverted=t[1])
        return self.static_loss
