"""CUDA-graph capture of a whole SPD-KFAC training step.

One replay = zero_grad + forward (A-factor hooks: staging on the compute stream,
tensor-core SYRK on the factor stream, fusion-group all-reduces on the comm stream)
+ loss + backward (G-factor hooks) + SPDKFAC.step() (gradient all-reduce, inverses,
owner broadcasts, preconditioning + update).  Every kernel of the step, ours, cuDNN's
and NCCL's, is launched by one cudaGraphLaunch, so the host's per-step cost no longer
bounds the iteration (the eager step spends ~20-30 ms of Python/launch time per
ResNet-50 iteration, comparable to the GPU time).

Constraints (checked): factor_update_freq == inv_update_freq == 1 (one graph per
step type), inputs copied into static buffers.  Gradients are reset with zero_grad(set_to_none=True):
backward then writes each weight gradient straight into a graph-pool tensor (no zero-fill and no
accumulate-add kernel per parameter), and the replays reuse those same addresses.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch


class GraphedStep:
    def __init__(self, model: torch.nn.Module, loss_fn: Callable, optimizer, inputs: Sequence[torch.Tensor],
                 targets: Sequence[torch.Tensor], warmup: int = 3, before_capture: Callable | None = None,
                 priority: int = 0):
        from .optimizer import SPDKFAC
        if isinstance(optimizer, SPDKFAC) and (optimizer.factor_update_freq != 1 or optimizer.inv_update_freq != 1):
            raise ValueError("GraphedStep captures one step type: factor_update_freq and inv_update_freq must be 1")
        self.model, self.loss_fn, self.opt = model, loss_fn, optimizer
        self.static_in = [t.detach().clone() for t in inputs]
        self.static_tg = [t.detach().clone() for t in targets]
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
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side if priority else None):
            self.static_loss = self._body()
        torch.cuda.synchronize()

    def _body(self):
        self.opt.zero_grad(set_to_none=True)
        loss = self.loss_fn(self.model(*self.static_in), *self.static_tg)
        loss.backward()
        self.opt.step()
        return loss

    def __call__(self, inputs: Sequence[torch.Tensor] | None = None, targets: Sequence[torch.Tensor] | None = None):
        """Copy new data into the static buffers (non-blocking, stream-ordered) and replay."""
        if inputs is not None:
            for s, t in zip(self.static_in, inputs):
                s.copy_(t, non_blocking=True)
        if targets is not None:
            for s, t in zip(self.static_tg, targets):
                s.copy_(t, non_blocking=True)
        self.graph.replay()
        if hasattr(self.opt, "_after_replay"):
            self.opt._after_replay(torch.cuda.current_stream())
        return self.static_loss
