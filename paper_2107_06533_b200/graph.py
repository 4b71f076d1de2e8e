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
        step = getattr(self.opt, "steps", 0)
        t = self._type(step)
        self.graphs[t].replay()
        self.static_loss = self.losses[t]
        if hasattr(self.opt, "_after_replay"):
            self.opt._after_replay(torch.cuda.current_stream(), inverted=t[1])
        return self.static_loss
