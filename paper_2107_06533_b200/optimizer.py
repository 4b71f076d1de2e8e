"""SPDKFAC: the B200-native SPD-KFAC optimizer step behind a torch.optim API.

It executes the step the reference emulates in `dkfac_step`
(pkg/src/kfacsched/emulator.py:211-263) on real ranks and real devices:

  forward hooks   A_l = a^T a / M   per layer (im2col rows for convs), straight into
                  the packed forward fusion buffer, running average + 1/P fused
                  (factor kernels, factor side stream); each fusion group of the
                  init-time plan (`plan_fusion`, planner.py:249-298) is all-reduced on
                  the communication stream as soon as its last member is written
  backward hooks  G_l = (b g)^T (b g) / M likewise into the backward fusion buffer
                  the early G inversion groups are inverted mid-backward on their own
                  streams; P > 1: the first gradient bucket is all-reduced mid-backward
  step()          remaining gradient all-reduce; damped inverses of this rank's share of the
                  load-balanced placement (`lbp_place`, planner.py:301-356), NCT tensors
                  on every rank, CT inverses broadcast from their owners in packed form;
                  W_l -= lr * G_l^-1 grad_l A_l^-1 for every K-FAC layer (plain SGD for
                  the remaining parameters, as the reference has no bias: SPEC.md:418).

Knobs: lr (alpha, emulator.py:207), damping (gamma, linalg.py:130), factor_decay
(running-average rho; 0 reproduces the reference), factor_update_freq and
inv_update_freq (the reference's single `kfac_update_interval`, simulator.py:126,
split in two), fusion policy, placement mode ("lbp" | "seq" | "local") and LBP
balance ("dim_sq" | "dim" | "dim_cube"), early_g_fraction (inversion groups),
launch_groups, update_in_backward (P = 1: precondition + update early groups during
backward).  See DESIGN.md "Step schedule".
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Optional

import torch
import torch.nn as nn

from . import _lib as L
from . import schedule as S
from .linalg import FactorGroup, FactorPlan, InversePlan, NotPositiveDefiniteError, PrecondPlan
from .perfmodel import PerfParams, default_params
from .planner import (FactorKind, FusionPlan, FusionPolicy, inverse_tasks, factor_tasks, lbp_place, local_place,
                      plan_fusion, seq_place)


@dataclass
class LayerSpec:
    """One preconditioned layer: factor dims and (estimated) pass times, the
    shape of `kfacsched.profiles.LayerProfile` (profiles.py:53-86)."""

    name: str
    a_dim: int
    g_dim: int
    t_ff: float = 1e-5
    t_bp: float = 2e-5
    t_factorA: float = 1e-5
    t_factorG: float = 1e-5


@dataclass
class _Layer:
    index: int
    name: str
    module: nn.Module
    is_conv: bool
    spec: LayerSpec
    a_off: int = 0
    g_off: int = 0
    a_plan: Optional[FactorPlan] = None
    g_plan: Optional[FactorPlan] = None
    a_key: tuple = ()
    g_key: tuple = ()
    w_cl: bool = False  # conv weight stored channels-last: A rows ordered (kh, kw, c)
    handles: list = field(default_factory=list)
    events: dict = field(default_factory=dict)   # kind -> (compute done, staged)
    pending: dict = field(default_factory=lambda: {"A": False, "G": False})


def _conv_ok(m) -> bool:
    return isinstance(m, nn.Conv2d) and m.groups == 1 and m.padding_mode == "zeros" and isinstance(m.padding, tuple)


class SPDKFAC(torch.optim.Optimizer):
    def __init__(self, model: nn.Module, lr: float = 0.1, damping: float = 0.1, factor_decay: float = 0.0,
                 factor_update_freq: int = 1, inv_update_freq: int = 1, fusion: FusionPolicy = FusionPolicy.OPTIMAL,
                 placement: str = "lbp", balance: str = "dim_sq", perf: Optional[PerfParams] = None,
                 batch_averaged: bool = True, layer_times: Optional[dict] = None, comm=None,
                 early_g_fraction=(0.85, 0.983, 0.9985), factor_comm: str = "auto", launch_groups: str = "auto",
                 update_in_backward: bool = False):
        if damping < 0:
            raise ValueError(f"damping must be nonnegative, got {damping}")
        if not 0.0 <= factor_decay < 1.0:
            raise ValueError(f"factor_decay must be in [0, 1), got {factor_decay}")
        if factor_update_freq < 1 or inv_update_freq < 1 or inv_update_freq % factor_update_freq:
            raise ValueError("update frequencies must be >= 1 and inv_update_freq a multiple of factor_update_freq")
        if factor_comm == "auto":  # deployment override of the automatic choice
            factor_comm = os.environ.get("SPDKFAC_FACTOR_COMM", "auto")
        if factor_comm not in ("auto", "allreduce", "reduce", "peer"):
            raise ValueError(f"factor_comm must be 'auto', 'allreduce', 'reduce' or 'peer', got {factor_comm!r}")
        if factor_comm in ("reduce", "peer") and factor_decay != 0.0:
            raise ValueError(f"factor_comm={factor_comm!r} needs factor_decay == 0 (the running average needs the aggregate "
                             "on every rank)")
        if placement not in ("lbp", "seq", "local"):
            raise ValueError(f"placement must be 'lbp', 'seq' or 'local', got {placement!r}")
        L.load(require_device=True)
        self.model = model
        self.damping, self.factor_decay = float(damping), float(factor_decay)
        self.factor_update_freq, self.inv_update_freq = int(factor_update_freq), int(inv_update_freq)
        self.batch_averaged = batch_averaged
        self.perf = perf  # resolved below once the world size is known
        self.device = next(model.parameters()).device

        import torch.distributed as dist
        dist_on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank() if dist_on else 0
        self.world = dist.get_world_size() if dist_on else 1
        if self.world > 1 and comm is None:
            from .comm import NcclComm
            comm = NcclComm(self.rank, self.world)
        self.comm = comm
        self.perf = perf or default_params(self.world)
        # one communicator, one comm stream: every rank issues the same collective sequence
        # (factor all-reduces as fusion groups complete, then in step(): gradient all-reduce and
        # the owners' inverse broadcasts), so no all-reduce ever queues behind a broadcast that
        # waits for an inversion, and no two communicators' kernels can wait on each other
        self.comm_bc = comm

        # ---- preconditioned layers, forward order (model definition order)
        self.layers: list[_Layer] = []
        kfac_params = set()
        for name, m in model.named_modules():
            if _conv_ok(m) or isinstance(m, nn.Linear):
                conv = isinstance(m, nn.Conv2d)
                a_dim = m.in_channels * m.kernel_size[0] * m.kernel_size[1] if conv else m.in_features
                g_dim = m.out_channels if conv else m.out_features
                t = (layer_times or {}).get(name, {})
                spec = LayerSpec(name, a_dim, g_dim, **t) if t else self._estimate_times(name, a_dim, g_dim)
                self.layers.append(_Layer(len(self.layers), name, m, conv, spec))
                kfac_params.add(m.weight)
        if not self.layers:
            raise ValueError("model has no Conv2d/Linear layers to precondition")
        params = list(model.parameters())
        self.other_params = [p for p in params if p not in kfac_params and p.requires_grad]
        super().__init__([{"params": params}], dict(lr=lr))

        # ---- init-time plans (the paper's "executed during initialization")
        specs = [l.spec for l in self.layers]
        ff = [s.t_ff for s in specs]
        bp = [s.t_bp for s in reversed(specs)]
        self.fwd_plan = plan_fusion(factor_tasks(specs, FactorKind.A), ff, self.perf.allreduce, fusion)
        self.bwd_plan = plan_fusion(factor_tasks(specs, FactorKind.G), bp, self.perf.allreduce, fusion)
        if launch_groups not in ("auto", "fusion", "inversion"):
            raise ValueError(f"launch_groups must be 'auto', 'fusion' or 'inversion', got {launch_groups!r}")
        # auto: peer-memory aggregation inside one NVSwitch node (P <= 8), the NCCL reduce beyond
        auto = ("peer" if 1 < self.world <= 8 else "reduce") if factor_decay == 0.0 else "allreduce"
        self.factor_comm = auto if factor_comm == "auto" else factor_comm
        # auto launch groups (measured, DESIGN.md (e)): the inversion-group cuts at P = 1 and, with peer
        # aggregation and the optimal fusion policy, at P = 2 (16.4-16.5 vs 17.0-17.1 ms); the fusion plan beyond
        # (P = 4: 16.4-16.6 vs 17.8-18.1 ms with the inversion cuts)
        lg_auto = "inversion" if self.world == 1 or (self.world == 2 and self.factor_comm == "peer"
                                                     and fusion == FusionPolicy.OPTIMAL) else "fusion"
        self.launch_groups = lg_auto if launch_groups == "auto" else launch_groups
        if self.launch_groups == "inversion":
            # no factor communication (P = 1, or by request): a fusion group only batches SYRK
            # launches, so use few large ones: A in two halves of the forward pass, G cut at the
            # inversion-group boundaries (each early G inversion waits for exactly one launch)
            fa = factor_tasks(specs, FactorKind.A)
            fg = factor_tasks(specs, FactorKind.G)
            n_g = S.inversion_groups([s.a_dim for s in specs], [s.g_dim for s in specs],
                                     early_fraction=early_g_fraction)["n_g"]
            cuts = [sum(n_g[:i]) for i in range(len(n_g) + 1)]
            na = max(1, int(os.environ.get("SPDKFAC_A_GROUPS", "2")))  # A launch groups (diagnostics)
            cuts_a = [round(i * len(fa) / na) for i in range(na + 1)]
            self.fwd_plan = FusionPlan(tuple(tuple(fa[a:b]) for a, b in zip(cuts_a, cuts_a[1:]) if b > a), fusion)
            self.bwd_plan = FusionPlan(tuple(tuple(fg[a:b]) for a, b in zip(cuts, cuts[1:]) if b > a), fusion)
        tasks = inverse_tasks(specs)
        if placement == "lbp":
            self.placement = lbp_place(tasks, self.world, getattr(self.perf, "placement_inverse", self.perf.inverse),
                                       self.perf.bcast, balance=balance)
        elif placement == "seq":
            self.placement = seq_place(tasks, self.world)
        else:
            self.placement = local_place(tasks, self.world)

        # ---- packed fusion buffers: A in forward order, G in backward order (schedule.py)
        a_dims = [l.spec.a_dim for l in self.layers]
        g_dims = [l.spec.g_dim for l in self.layers]
        a_off, g_off, size_a, size_g = S.packed_layout(a_dims, g_dims)
        for l in self.layers:
            l.a_off, l.g_off = a_off[l.index], g_off[l.index]
        self.bufA = torch.zeros(size_a, dtype=torch.float32, device=self.device)
        self.bufG = torch.zeros(size_g, dtype=torch.float32, device=self.device)
        self._groups_fwd = S.fusion_slices(self.fwd_plan, a_off, a_dims)
        self._groups_bwd = S.fusion_slices(self.bwd_plan, g_off, g_dims)
        S.check_fusion_cover(self._groups_fwd, size_a)
        S.check_fusion_cover(self._groups_bwd, size_g)
        # group id per layer and member counts; slices keyed by group id
        self._gid = {"A": S.fusion_members(self.fwd_plan)[0], "G": S.fusion_members(self.bwd_plan)[0]}
        self._gsize = {"A": S.fusion_members(self.fwd_plan)[1], "G": S.fusion_members(self.bwd_plan)[1]}
        self._gslice = {"A": [self._groups_fwd[g[-1].layer_index - 1] for g in self.fwd_plan.groups],
                        "G": [self._groups_bwd[g[-1].layer_index - 1] for g in self.bwd_plan.groups]}
        self._gseen = {"A": [0] * len(self.fwd_plan.groups), "G": [0] * len(self.bwd_plan.groups)}
        # factor aggregation: all-reduce (every rank holds every aggregate, needed for a running
        # average) or, with factor_decay == 0, a sum onto the owner of each CT inverse only
        # (half the traffic; NCT factors are still all-reduced): over NVLink peer memory ("peer",
        # comm.PeerExchange) or an NCCL reduce ("reduce")
        self._gsegs = {"A": S.reduce_segments(self.fwd_plan, a_off, a_dims, self.placement, 0),
                       "G": S.reduce_segments(self.bwd_plan, g_off, g_dims, self.placement, 1)}
        self._fgroups = None  # per fusion group FactorGroup objects, built after the first iteration
        self._peer = None  # comm.PeerExchange (factor_comm "peer"), created below
        self._rec = {"A": [None] * len(self.layers), "G": [None] * len(self.layers)}

        # ---- inverses (every rank holds all of them for preconditioning)
        self.inv = []
        for l in self.layers:
            self.inv.append(torch.zeros(l.spec.a_dim, l.spec.a_dim, dtype=torch.float32, device=self.device))
            self.inv.append(torch.zeros(l.spec.g_dim, l.spec.g_dim, dtype=torch.float32, device=self.device))
        # this rank's inversions in groups, each launched as soon as its factors exist
        # (schedule.inversion_groups): A after the forward pass (own stream, overlaps the
        # backward pass), the early G groups G1..Gk (the layers backward reaches first, most of
        # the G work) mid-backward on their own streams, the tail G group in step()
        mine = list(self.placement.workers[self.rank])
        self._mine = mine
        grp = S.inversion_groups([l.spec.a_dim for l in self.layers], [l.spec.g_dim for l in self.layers],
                                 early_fraction=early_g_fraction)
        self._early, self._tail = list(grp["early"]), grp["tail"]
        self._sides = ["A"] + self._early + [self._tail]
        # an early G group may start once every backward fusion group holding one of its members
        # is computed; the factors its inverses read must be complete (members of a group run together)
        self._early_groups = {side: {self._gid["G"][t // 2] for t in grp[side]} for side in self._early}
        self._early_left = {side: len(g) for side, g in self._early_groups.items()}
        self._inv_plans, self._info_host, self._bcast, self._inv_ts = {}, {}, {}, {}
        for side in self._sides:
            ts = [t for t in mine if t in grp[side]]
            self._inv_ts[side] = ts
            self._inv_plans[side] = InversePlan([self._packed(t) for t in ts], [self.inv[t] for t in ts]) if ts else None
            # two pinned slots (eager steps alternate; a captured graph always writes slot 0): step N+1's
            # A inversion, launched from the forward hooks, cannot overwrite step N's info before
            # check_inverses reads it
            self._info_host[side] = ([torch.zeros(len(ts), dtype=torch.int32, pin_memory=True) for _ in range(2)]
                                     if ts else None)
            self._bcast[side] = self._bcast_layout(grp[side])
        # factor_comm = "peer": each fusion group's CT factors owned elsewhere are pushed into the owner's
        # inbox over NVLink (comm.PeerExchange) and the owner adds its inbox rows; the owners' CT inverses
        # can travel the same way (SPDKFAC_PEER_BCAST=1: pushed into every peer's receive region of the
        # allocation right after each inversion; default: the NCCL broadcasts)
        self._peer_bcast = False
        if self.world > 1 and self.factor_comm == "peer":
            from .comm import PeerExchange
            n_a = len(self.fwd_plan.groups)
            self._peer_base = {"A": 0, "G": n_a}
            n_groups = n_a + len(self.bwd_plan.groups)
            self._peer_bcast = os.environ.get("SPDKFAC_PEER_BCAST", "0") == "1"  # measured no gain: opt-in
            # receive regions: per inversion side and owner, that owner's packed CT inverses (same layout
            # on every rank); slot n_groups + k carries side k's "inverses pushed" flags
            self._bc_off, extra = {}, 0
            if self._peer_bcast:
                for side in self._sides:
                    self._bc_off[side] = []
                    for ct, dims, buf, views, n in self._bcast[side]:
                        self._bc_off[side].append(extra)
                        extra += max(n, 1)
                self._peer_slot_bc = {side: n_groups + k for k, side in enumerate(self._sides)}
            self._peer = PeerExchange(self.rank, self.world, {"A": size_a, "G": size_g},
                                      n_groups + len(self._sides), self.device, extra=extra)
            if self._peer_bcast:
                for side in self._sides:
                    lay = []
                    for (ct, dims, _, _, n), off in zip(self._bcast[side], self._bc_off[side]):
                        buf = self._peer.extra[off:off + max(n, 1)]
                        offs = [sum(S.packed_size(e) for e in dims[:k]) for k in range(len(dims))]
                        lay.append((ct, dims, buf, [buf[o:o + S.packed_size(d)] for o, d in zip(offs, dims)], n))
                    self._bcast[side] = lay
        if self._peer is not None:
            self._peer_epilogue = os.environ.get("SPDKFAC_PEER_PUSH", "copy") == "epilogue"
            self._peer_segs, self._peer_out = {}, {}
            for kind in ("A", "G"):
                self._peer_out[kind] = [[(s, e, root) for s, e, root in segs if root is not None and root != self.rank]
                                        for segs in self._gsegs[kind]]
                lst = []
                for segs in self._gsegs[kind]:
                    mine = [(s, e - s) for s, e, root in segs if root == self.rank]
                    t = torch.tensor(mine, dtype=torch.int64, device=self.device).reshape(-1, 2) if mine else None
                    lst.append((t, max((n for _, n in mine), default=0)))
                self._peer_segs[kind] = lst
        # preconditioning + update in groups that follow the G inversion groups (layer sets in
        # backward order): with update_in_backward, an early group's layers are preconditioned
        # and updated on that group's stream as soon as their gradients are accumulated and
        # their inverses exist, while the rest of the backward pass runs; step() handles the
        # tail group (and every group otherwise)
        if update_in_backward and self.world > 1:
            raise ValueError("update_in_backward needs P == 1 (the gradient mean is formed in step())")
        self.update_in_backward = bool(update_in_backward)
        # without it, one plan over every layer runs in step() (fewest launches)
        # P > 1 (SPDKFAC_EARLY_PRECOND): the early groups' layers are preconditioned in step() on their streams as
        # soon as the first gradient bucket, the A inverses and their G inverses are in, beside the tail inversion
        # (measured no gain at N = 2 / 4: opt-in)
        self._p_early = self.world > 1 and os.environ.get("SPDKFAC_EARLY_PRECOND", "0") == "1" and bool(self._early)
        per_side = self.update_in_backward or self._p_early
        self._pc_sides = self._early + [self._tail] if per_side else ["ALL"]
        if per_side:
            self._pc_side = {t // 2: side for side in self._pc_sides for t in grp[side]}
        else:
            self._pc_side = {li: "ALL" for li in range(len(self.layers))}
        self._pc_layers = {side: sorted(li for li, sd in self._pc_side.items() if sd == side) for side in self._pc_sides}
        self._pc_local = {li: k for side in self._pc_sides for k, li in enumerate(self._pc_layers[side])}
        self._precond = {side: PrecondPlan([(self.layers[li].spec.g_dim, self.layers[li].spec.a_dim)
                                            for li in self._pc_layers[side]], device=self.device)
                         for side in self._pc_sides if self._pc_layers[side]}
        self._precond_key = {side: None for side in self._precond}
        # gradient buckets (P > 1, see _bucket_hook)
        self._grad_order, self._order_seen, self._bucket1, self._bucket_params = [], set(), None, []
        self._b1_sent, self._b1_left, self._b1_count, self._b1_numel, self._b1_ids = False, 0, 0, 0, set()
        self._pc_done = {side: False for side in self._precond}
        self._grad_left = {side: len(self._pc_layers[side]) for side in self._precond}

        self.factor_stream = torch.cuda.Stream(self.device)
        # steady-state staging (im2col / precision split, HBM-bound) runs beside the
        # tensor-core convolutions instead of on the forward/backward stream
        self.stage_stream = torch.cuda.Stream(self.device)
        self._stage_refs = []  # inputs staged on stage_stream, kept alive until step() joins it
        # the inversion chains (latency-bound) may run at a higher stream priority than the throughput work
        # (SPDKFAC_INV_PRIORITY, e.g. -1; default 0); the inverse plan's look-ahead stream follows the env too
        inv_prio = int(os.environ.get("SPDKFAC_INV_PRIORITY", "0"))
        self.inv_stream = torch.cuda.Stream(self.device, priority=inv_prio)
        self._g_streams = {side: torch.cuda.Stream(self.device, priority=inv_prio) for side in self._early}
        # index of the early G group whose launch issues the A-inverse broadcast (default: the last)
        self._a_bcast_after = int(os.environ.get("SPDKFAC_A_BCAST_AFTER", len(self._early) - 1))
        self._g_count = 0
        self._g_inverted = {side: False for side in self._early}
        self._sent = {side: False for side in self._sides}
        self._recvd = set()  # sides whose received inverses are unpacked this step
        self._grad_src = {}
        self.comm_stream = torch.cuda.Stream(self.device) if self.world > 1 else None
        self._info_events = []
        self._a_count = 0
        self._a_inverted = False
        self.timeline = None  # set to {} to record per-phase CUDA events (eager diagnostics)
        # the preconditioner's split operands of the inverses are staged by the stream that
        # produced them (inversion or unpack); stale until the first inversion / after a load
        self._planes_stale = True
        self.steps = 0
        self._capture = True
        self._factor_updates = 0
        self._install_hooks()

    # ------------------------------------------------------------------ setup helpers
    @staticmethod
    def _estimate_times(name, a_dim, g_dim) -> LayerSpec:
        # rough shape-only estimates; only the relative readiness of factors matters to
        # the OPTIMAL fusion criterion (planner.py:280-290).  Pass `layer_times` to override.
        t_ff = 5e-6 + a_dim * g_dim * 2e-11
        return LayerSpec(name, a_dim, g_dim, t_ff, 2 * t_ff, 3e-6 + a_dim * a_dim * 5e-12, 3e-6 + g_dim * g_dim * 5e-12)

    def _packed(self, t: int) -> torch.Tensor:
        l = self.layers[t // 2]
        if t % 2 == 0:
            d = l.spec.a_dim
            return self.bufA[l.a_off:l.a_off + d * (d + 1) // 2]
        d = l.spec.g_dim
        return self.bufG[l.g_off:l.g_off + d * (d + 1) // 2]

    def _bcast_layout(self, members):
        """Per owner rank: its CT tensors of one group (placement order) and packed staging views."""
        if self.world == 1:
            return None
        lay = []
        for ct, dims, offs, n in S.bcast_layout(self.placement, [t.shape[0] for t in self.inv], members=members):
            buf = torch.empty(max(n, 1), dtype=torch.float32, device=self.device)
            views = [buf[o:o + S.packed_size(d)] for o, d in zip(offs, dims)]
            lay.append((ct, dims, buf, views, n))
        return lay

    def _weight_matrix(self, l: _Layer, t: torch.Tensor) -> torch.Tensor:
        """[d_out][d_in] view of a weight (or its gradient) in the A-factor column order."""
        if l.is_conv and l.w_cl:
            v = t.permute(0, 2, 3, 1).reshape(l.spec.g_dim, l.spec.a_dim)
        else:
            v = t.reshape(l.spec.g_dim, l.spec.a_dim)
        if v.data_ptr() != t.data_ptr() or not v.is_contiguous():
            raise RuntimeError(f"layer {l.name}: weight/gradient is not a dense [d_out, d_in] view")
        return v

    def _install_hooks(self):
        for l in self.layers:
            if l.is_conv:
                l.w_cl = self._weight_channels_last(l.module)
            l.events = {k: (torch.cuda.Event(), torch.cuda.Event()) for k in ("A", "G")}
            l.handles.append(l.module.register_forward_pre_hook(self._make_a_hook(l)))
            l.handles.append(l.module.register_forward_hook(self._make_out_hook(l)))
            l.handles.append(l.module.weight.register_post_accumulate_grad_hook(self._make_grad_hook(l)))
        # P > 1: gradient bucket all-reduced during backward (see _bucket_hook)
        self._param_handles = []
        if self.world > 1:
            for p in self.param_groups[0]["params"]:
                if p.requires_grad:
                    self._param_handles.append(p.register_post_accumulate_grad_hook(self._bucket_hook))

    def remove_hooks(self):
        for l in self.layers:
            for h in l.handles:
                h.remove()
            l.handles.clear()
        for h in getattr(self, "_param_handles", []):
            h.remove()
        self._param_handles = []

    # ------------------------------------------------------------------ gradient buckets (P > 1)
    # The gradient all-reduce is split into two buckets in the order gradients are accumulated
    # (recorded in the first backward): the first ~90 % of the elements (the layers backward
    # reaches first) is all-reduced on the comm stream as soon as its last gradient lands, under
    # the rest of the backward pass; step() all-reduces only the remainder.  Hooks fire in the same
    # order on every rank, so the collective sequence stays identical.  One backward per step()
    # is assumed (gradient accumulation over several backward passes falls back to step()).
    def _bucket_hook(self, param) -> None:
        if self._bucket1 is None:
            if id(param) not in self._order_seen:
                self._order_seen.add(id(param))
                self._grad_order.append(param)
            return
        if not self._b1_sent and id(param) in self._b1_ids:
            self._b1_left -= 1
            if self._b1_left == 0:
                main = torch.cuda.current_stream(self.device)
                cs = self.comm_stream
                cs.wait_stream(main)
                b1 = self._bucket_params[:self._b1_count]
                flat, views = self._flat_grad_buffer(self._bucket_params)
                with torch.cuda.stream(cs):
                    torch._foreach_copy_(views[:self._b1_count], [p.grad for p in b1])
                self.comm.allreduce_sum(flat[:self._b1_numel], cs, tag="grad")
                self._b1_sent = True

    def _build_buckets(self, params) -> None:
        order = [p for p in self._grad_order if p.grad is not None]
        if {id(p) for p in order} != {id(p) for p in params}:
            self._bucket1 = []  # accumulation order incomplete: no bucketing
            return
        total = sum(p.numel() for p in order)
        frac = float(os.environ.get("SPDKFAC_GRAD_BUCKET", "0.9"))  # share all-reduced during backward
        n1, acc = 0, 0
        while n1 < len(order) - 1 and acc + order[n1].numel() <= frac * total:
            acc += order[n1].numel()
            n1 += 1
        self._bucket_params = order
        self._bucket1, self._b1_count, self._b1_numel = order[:n1], n1, acc
        self._b1_ids = {id(p) for p in order[:n1]}
        self._b1_left = n1

    # ------------------------------------------------------------------ factor capture
    def _factor_args(self):
        decay = self.factor_decay if self._factor_updates > 0 else 0.0
        return decay, 1.0 / self.world

    @staticmethod
    def _weight_channels_last(m) -> bool:
        w = m.weight
        return w.dim() == 4 and not w.is_contiguous() and w.is_contiguous(memory_format=torch.channels_last)

    def _prepare(self, l: _Layer, x: torch.Tensor, kind: str):
        """Pick the staging layout that matches the tensor's memory format (no copy in the
        common cases).  A-factor rows follow the weight's column order: (c, kh, kw) for a
        contiguous conv weight, (kh, kw, c) for a channels-last one."""
        if x.dtype != torch.float32:
            x = x.to(torch.float32)
        if not l.is_conv:
            x = x.contiguous()
            return L.ROWS, x.reshape(-1, x.shape[-1])
        cl = torch.channels_last
        if kind == "A":
            pointwise = tuple(l.module.kernel_size) == (1, 1)
            if l.w_cl or (pointwise and not x.is_contiguous() and x.is_contiguous(memory_format=cl)):
                # 1x1 kernels: (kh, kw, c) and (c, kh, kw) are the same column order, so a
                # channels-last input is staged as rows whatever the weight's memory format
                return L.CONV_A_NHWC, x.contiguous(memory_format=cl)
            return L.CONV_A, x.contiguous()
        if x.is_contiguous():
            return L.SPATIAL, x
        return L.SPATIAL_NHWC, x.contiguous(memory_format=cl)

    def _plan_for(self, l: _Layer, layout: int, x: torch.Tensor, kind: str) -> FactorPlan:
        key = (layout,) + tuple(x.shape)
        m = l.module
        if kind == "A":
            if l.a_key != key:
                if l.is_conv:
                    l.a_plan = FactorPlan(layout, x.shape, m.kernel_size, m.stride, m.padding, m.dilation)
                else:
                    l.a_plan = FactorPlan(L.ROWS, x.shape)
                l.a_key = key
            return l.a_plan
        if l.g_key != key:
            l.g_plan = FactorPlan(layout, x.shape) if l.is_conv else FactorPlan(L.ROWS, x.shape)
            l.g_key = key
        return l.g_plan

    def _launch_factor(self, l: _Layer, x: torch.Tensor, kind: str):
        """Stage x on the stream that owns it (im2col/transpose + precision split into a
        staging buffer), then run the tensor-core SYRK on the factor stream.  The SYRK reads
        only staging memory, so x's lifetime is not extended across streams.

        Steady state: one FactorGroup per fusion group (planner.py:94-121); members are staged
        as their hooks fire and the group's single tensor-core launch (and, for P > 1, its
        all-reduce) follows its last member.  The first iteration (and any shape change) runs
        per-layer plans and records the shapes the groups are built from (in step())."""
        main = torch.cuda.current_stream(self.device)
        fs = self.factor_stream
        # samples of a batch-mean loss: the image batch for convs, the rows for linears
        nb = x.shape[0] if l.is_conv else x.numel() // x.shape[-1]
        if kind == "A" and self._a_count == 0:
            self._tl("fwd_start", main)
            if self._peer is not None:  # this step's signals carry the new epoch
                self._peer.advance(main)
        layout, x = self._prepare(l, x.detach(), kind)
        key = (layout,) + tuple(x.shape)
        capturing = torch.cuda.is_current_stream_capturing()
        decay = self.factor_decay if self._factor_updates > 0 else 0.0
        gid = self._gid[kind][l.index]
        if self._gseen[kind][gid] >= self._gsize[kind][gid]:
            # a second train-mode forward/backward before step(): the reference takes its factors from
            # one batch per step (emulator.py:234-241); a silent second capture would freeze the group's
            # SYRK (its staging counter never returns to 0) and, at P > 1, re-reduce stale buffers
            raise RuntimeError(f"SPDKFAC: layer {l.name!r} ({kind} factor) was captured twice before step(); "
                               "call step() after every backward, or run extra passes under torch.no_grad() "
                               "or with the module in eval mode")
        fg = self._fgroups[kind][gid] if self._fgroups is not None else None
        if fg is not None and fg["keys"][l.index] == key:
            ss = self.stage_stream
            ss.wait_stream(main)  # x is complete
            if fg["seen"] == 0 and not capturing and fg["pending"]:
                ss.wait_event(fg["done"])  # previous iteration's SYRK has consumed the staging buffers
            fg["obj"].stage(fg["member"][l.index], x, ss)
            # an output gradient may be freed once its layer's backward ran (and _prepare may
            # return a temporary): hold x until step() joins the stage and factor streams (row
            # layouts are read by the SYRK directly; A inputs are saved for backward anyway, so
            # they are never modified in place)
            self._stage_refs.append(x)
            fg["seen"] += 1
        else:
            if fg is not None:  # shape changed: per-layer plans this iteration, rebuild groups after
                self._fgroups = None
            plan = self._plan_for(l, layout, x, kind)
            ev_done, ev_staged = l.events[kind]
            if not capturing and l.pending[kind]:
                main.wait_event(ev_done)
            plan.stage(x, main)
            self._stage_refs.append(x)  # row layouts are read by the SYRK itself (factor stream)
            ev_staged.record(main)
            fs.wait_event(ev_staged)
            if kind == "A":
                buf, off, d, scale = self.bufA, l.a_off, l.spec.a_dim, 1.0 / plan.rows
            else:
                b = nb if self.batch_averaged else 1
                buf, off, d, scale = self.bufG, l.g_off, l.spec.g_dim, float(b * b) / plan.rows
            plan.compute(buf[off:off + d * (d + 1) // 2], scale, decay, 1.0 / self.world, fs)
            ev_done.record(fs)
            l.pending[kind] = not capturing
            m = l.module
            geo = (layout, tuple(x.shape), tuple(m.kernel_size), tuple(m.stride), tuple(m.padding),
                   tuple(m.dilation)) if (l.is_conv and kind == "A") else (layout, tuple(x.shape), (1, 1), (1, 1),
                                                                           (0, 0), (1, 1))
            self._rec[kind][l.index] = (key, geo, scale)
        self._gseen[kind][gid] += 1
        if self._gseen[kind][gid] == self._gsize[kind][gid]:  # every member of the fusion group staged
            self._group_complete(kind, gid, decay, capturing)
        if kind == "A":
            self._a_count += 1
            if self._a_count == len(self.layers):
                self._launch_inverse_A()

    def _group_complete(self, kind: str, gid: int, decay: float, capturing: bool) -> None:
        main = torch.cuda.current_stream(self.device)
        fs = self.factor_stream
        buf = self.bufA if kind == "A" else self.bufG
        fg = self._fgroups[kind][gid] if self._fgroups is not None else None
        grouped = fg is not None and fg["seen"] == self._gsize[kind][gid]
        peer = grouped and self._peer is not None
        if grouped:
            fg["staged"].record(self.stage_stream)
            fs.wait_event(fg["staged"])
            fg["obj"].compute(decay, 1.0 / self.world, fs)
            if peer:  # push this group's factors owned elsewhere into their owners' inboxes, raise the flags
                if not self._peer_epilogue:
                    for s, e, root in self._peer_out[kind][gid]:
                        self._peer.push(root, kind, s, buf[s:e], fs)
                self._peer.signal(self._peer_base[kind] + gid, fs)
            fg["done"].record(fs)
            fg["pending"] = not capturing
            fg["seen"] = 0
        if self.world > 1:
            cs = self.comm_stream
            cs.wait_stream(fs)
            if peer:
                nct = [(s, e) for s, e, root in self._gsegs[kind][gid] if root is None]
                if nct:  # replicated (NCT) inverses: every rank needs the aggregate
                    with self.comm.group():
                        for s, e in nct:
                            self.comm.allreduce_sum(buf[s:e], cs)
                segs, mx = self._peer_segs[kind][gid]
                if segs is not None:
                    self._peer.wait_sum(self._peer_base[kind] + gid, kind, buf, segs, mx, cs)
            elif self.factor_comm in ("reduce", "peer"):
                with self.comm.group():
                    for s, e, root in self._gsegs[kind][gid]:
                        if root is None:
                            self.comm.allreduce_sum(buf[s:e], cs)
                        else:
                            self.comm.reduce_sum(buf[s:e], root, cs)
            else:
                s, e = self._gslice[kind][gid]
                self.comm.allreduce_sum(buf[s:e], cs)
        if kind == "G":
            for side in self._early:
                if gid in self._early_groups[side]:
                    self._early_left[side] -= 1
                    if self._early_left[side] == 0:
                        self._launch_inverse_G(side)

    def _build_factor_groups(self) -> None:
        """One FactorGroup per fusion group from the shapes recorded by the per-layer path."""
        if any(r is None for k in ("A", "G") for r in self._rec[k]):
            return
        groups = {}
        for kind, plan in (("A", self.fwd_plan), ("G", self.bwd_plan)):
            buf = self.bufA if kind == "A" else self.bufG
            out = []
            for g in plan.groups:
                idx = [t.layer_index - 1 for t in g]
                members, packed, scales, keys, member = [], [], [], {}, {}
                for k, li in enumerate(idx):
                    key, geo, scale = self._rec[kind][li]
                    l = self.layers[li]
                    off, d = (l.a_off, l.spec.a_dim) if kind == "A" else (l.g_off, l.spec.g_dim)
                    members.append(geo)
                    tgt = buf[off:off + d * (d + 1) // 2]
                    if self._peer is not None and self._peer_epilogue:  # CT factor owned elsewhere: its inbox row there
                        t = 2 * li + (0 if kind == "A" else 1)
                        root = None if t in self.placement.nct else self.placement.owner(t)
                        if root is not None and root != self.rank:
                            tgt = self._peer.remote_ptr(root, kind, off)
                    packed.append(tgt)
                    scales.append(scale)
                    keys[li] = key
                    member[li] = k
                out.append({"obj": FactorGroup(members, packed, scales), "keys": keys, "member": member, "seen": 0,
                            "pending": False, "staged": torch.cuda.Event(), "done": torch.cuda.Event()})
            groups[kind] = out
        torch.cuda.current_stream(self.device).synchronize()
        self._fgroups = groups
        for l in self.layers:  # the per-layer staging buffers are no longer needed
            l.a_plan = l.g_plan = None
            l.a_key = l.g_key = ()

    def _tl(self, name: str, stream) -> None:
        if self.timeline is not None and not torch.cuda.is_current_stream_capturing():
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            self.timeline[name] = ev

    def timeline_ms(self) -> dict:
        """Milliseconds of each recorded phase event relative to 'fwd_start' (synchronises)."""
        tl = self.timeline or {}
        if "fwd_start" not in tl:
            return {}
        tl["fwd_start"].synchronize()
        for ev in tl.values():
            ev.synchronize()
        return {k: round(tl["fwd_start"].elapsed_time(v), 3) for k, v in tl.items()}

    def _inverting(self) -> bool:
        return self.steps % self.inv_update_freq == 0

    def _launch_inverse_A(self):
        """All A factors of this iteration are enqueued (and, for P > 1, their fusion-group
        all-reduces): invert this rank's A tensors on the inverse stream, overlapping the
        rest of the forward pass and the backward pass, and broadcast the CT ones."""
        if self._a_inverted or not self._inverting():
            return
        s = self.inv_stream
        s.wait_stream(self.factor_stream)
        if self.world > 1:
            s.wait_stream(self.comm_stream)
        self._tl("a_factors_done", s)
        self._run_inverse("A", s, exchange=False)  # NCCL: broadcast in step(), after the all-reduces
        if self._peer_bcast:  # peer pushes share no FIFO with the reductions: send right away
            self._exchange_send("A", s)
        self._tl("a_inverse_done", s)
        self._a_inverted = True

    def _launch_inverse_G(self, side: str):
        """The G factors of one early group (layers the backward reached first) are enqueued:
        invert them on the group's own stream while the rest of the backward pass runs."""
        if self._g_inverted[side] or not self._inverting():
            return
        for prev in self._early[:self._early.index(side)]:  # keep the program order of the sends
            self._launch_inverse_G(prev)
        s = self._g_streams[side]
        s.wait_stream(self.factor_stream)
        if self.world > 1:
            s.wait_stream(self.comm_stream)
            # A inverses are on their way: share them while backward runs.  The broadcast waits
            # for this rank's A inversions and every later collective on the single comm stream
            # queues behind it, so it is issued only after the last early G group's factor
            # reductions (earlier, it would hold those groups' inversions back until the A side
            # finished)
            if self._a_inverted and side == self._early[min(self._a_bcast_after, len(self._early) - 1)]:
                self._exchange_send("A", self.inv_stream)
        self._run_inverse(side, s, exchange=False)
        if self._peer_bcast:
            self._exchange_send(side, s)
        self._tl(f"{side.lower()}_inverse_done", s)
        self._g_inverted[side] = True

    def _run_inverse(self, side: str, stream, exchange: bool = True) -> None:
        plan = self._inv_plans[side]
        if plan is not None:
            plan.run(self.damping, stream)
            self._stage_planes(self._inv_ts[side], stream)
            capturing = torch.cuda.is_current_stream_capturing()
            slot = 0 if capturing else self.steps % 2
            self._info_host[side][slot].copy_(plan.info, non_blocking=True)
            if not capturing:
                ev = torch.cuda.Event()
                ev.record(stream)
                self._info_events.append((ev, side, self.steps, slot))
        if self.world > 1 and exchange:
            self._exchange_send(side, stream)
            stream.wait_stream(self.comm_stream)
            self._exchange_recv(side, stream)

    def _make_a_hook(self, l: _Layer):
        def hook(module, inputs):
            if self._capture and torch.is_grad_enabled() and module.training:
                self._launch_factor(l, inputs[0], "A")
        return hook

    def _make_out_hook(self, l: _Layer):
        def hook(module, inputs, output):
            if self._capture and torch.is_grad_enabled() and module.training and output.requires_grad:
                output.register_hook(lambda g: self._launch_factor(l, g, "G"))
        return hook

    # ------------------------------------------------------------------ step
    def check_inverses(self, previous_steps_only: bool = False) -> None:
        """Raise NotPositiveDefiniteError for completed inversions (linalg.py:141-145);
        synchronises only on those inversions' events.  step() checks the previous steps'
        inversions only, so it never waits for the current iteration's A inverses.  Unlike the
        reference, which raises before any update, the failing step's weight update has already
        been applied (with the failed matrix's inverse left unchanged); the error surfaces at the
        next step() or check_inverses()."""
        if previous_steps_only:
            events = [e for e in self._info_events if e[2] < self.steps]
            self._info_events = [e for e in self._info_events if e[2] >= self.steps]
        else:
            events, self._info_events = self._info_events, []
        if not previous_steps_only and self._peer is not None and self._peer.error():
            raise RuntimeError(f"SPDKFAC: peer factor signals of group slot {self._peer.error() - 1} timed out "
                               f"after {self._peer.timeout_s} s (SPDKFAC_PEER_TIMEOUT_S)")
        for ev, side, _, slot in events:
            ev.synchronize()
            info = self._info_host[side][slot]
            bad = torch.nonzero(info).flatten()
            if bad.numel():
                raise NotPositiveDefiniteError(int(info[bad[0]]) - 1)

    @torch.no_grad()
    def step(self, closure=None):
        loss = closure() if closure is not None else None
        capturing = torch.cuda.is_current_stream_capturing()
        if not capturing:
            self.check_inverses(previous_steps_only=True)
        main = torch.cuda.current_stream(self.device)
        lr = self.param_groups[0]["lr"]
        factors_now = self._capture
        invert_now = self.steps % self.inv_update_freq == 0
        self._tl("backward_done", main)
        if factors_now:  # every staged input / output gradient is consumed (a reuse step stages nothing:
            main.wait_stream(self.stage_stream)  # under graph capture the stage stream is then not part of it)
        if factors_now:
            main.wait_stream(self.factor_stream)
            self._factor_updates += 1
            self._tl("g_factors_done", main)
        # row-layout factor inputs are read by the SYRK on the factor stream: release them only now
        self._stage_refs.clear()
        factors_reduced = None
        if self.world > 1:
            cs = self.comm_stream
            if invert_now:
                if not self._a_inverted:  # hooks did not see a full forward (e.g. factors reused)
                    self._launch_inverse_A()
                for side in self._early:
                    self._launch_inverse_G(side)
            # every factor all-reduce of this iteration is enqueued: the tail G group's inversion waits for
            # exactly these, not for the broadcasts and the gradient all-reduce queued behind
            factors_reduced = torch.cuda.Event()
            factors_reduced.record(cs)
            if invert_now:
                self._exchange_send("A", self.inv_stream)
                for side in self._early:
                    self._exchange_send(side, self._g_streams[side])
            if self._p_early and self._b1_sent:
                self._early_precond(invert_now, lr)
            cs.wait_stream(main)
            params = [p for p in self.param_groups[0]["params"] if p.grad is not None]
            if self._bucket1 is None and not capturing:
                self._build_buckets(params)
            if self._b1_sent:  # the first bucket was all-reduced during backward: the rest
                params = self._bucket_params
                flat, views = self._flat_grad_buffer(params)
                with torch.cuda.stream(cs):
                    torch._foreach_copy_(views[self._b1_count:], [p.grad for p in params[self._b1_count:]])
                self.comm.allreduce_sum(flat[self._b1_numel:], cs, tag="grad")
            else:
                if self._bucket1:
                    params = self._bucket_params if len(params) == len(self._bucket_params) else params
                flat, views = self._flat_grad_buffer(params)
                with torch.cuda.stream(cs):  # one contiguous all-reduce instead of one per parameter
                    torch._foreach_copy_(views, [p.grad for p in params])
                self.comm.allreduce_sum(flat, cs, tag="grad")
            self._grad_src = {id(p): v for p, v in zip(params, views)}
            self._b1_sent = False
            if self._bucket1:
                self._b1_left = self._b1_count
            if not invert_now:
                main.wait_stream(cs)
        if invert_now:
            if not self._a_inverted:  # hooks did not see a full forward (e.g. factors reused)
                self._launch_inverse_A()
            for side in self._early:
                self._launch_inverse_G(side)
            if factors_reduced is not None:
                main.wait_event(factors_reduced)
            self._run_inverse(self._tail, main, exchange=False)
            self._tl("g_inverse_done", main)
            main.wait_stream(self.inv_stream)   # A inverses landed
            for side in self._early:  # early G groups likewise
                main.wait_stream(self._g_streams[side])
            if self.world > 1:
                self._exchange_send(self._tail, main)
                main.wait_stream(self.comm_stream)
                for side in self._sides:
                    if side not in self._recvd:
                        self._exchange_recv(side, main)
            self._tl("inverses_joined", main)
        # precondition + update for every K-FAC layer not yet done during backward (mean gradient
        # = sum / P); P > 1: the all-reduced gradient lives in the flat buffer (same shapes and strides)
        for side in self._precond:
            if self._pc_done[side]:
                main.wait_stream(self._g_streams[side])
            else:
                self._run_precond(side, main, lr)
        if invert_now:
            self._planes_stale = False
        self._tl("precond_done", main)
        others = [p for p in self.other_params if p.grad is not None]
        if others:
            src = self._grad_src if self.world > 1 else {}
            torch._foreach_add_([p.data for p in others], [src.get(id(p), p.grad) for p in others],
                                alpha=-lr / self.world)
        self._a_count = 0
        self._a_inverted = False
        self._g_count = 0
        self._g_inverted = {side: False for side in self._early}
        self._sent = {side: False for side in self._sides}
        self._recvd = set()
        self._early_left = {side: len(g) for side, g in self._early_groups.items()}
        self._pc_done = {side: False for side in self._precond}
        self._grad_left = {side: len(self._pc_layers[side]) for side in self._precond}
        for k in ("A", "G"):
            self._gseen[k] = [0] * len(self._gseen[k])
            for fg in (self._fgroups or {}).get(k, []):
                fg["seen"] = 0  # a group whose members were only partly captured this step starts afresh
        if self._fgroups is None and not capturing and factors_now:
            self._build_factor_groups()
        if not capturing:  # a captured step is counted per replay (_after_replay)
            self.steps += 1
            self._capture = self.steps % self.factor_update_freq == 0
        return loss

    def _early_precond(self, invert_now: bool, lr: float) -> None:
        """P > 1: precondition + update the early groups' layers while the tail G group is inverted.
        Their mean gradients are in the first bucket's all-reduce and their inverses are local (owned
        or NCT) or in the A / early-group broadcasts, all queued on the comm stream before this point:
        one stream unpacks the received inverses once, then each early group runs on its own stream."""
        b1 = self._b1_ids
        sides = [sd for sd in self._early if sd in self._precond and not self._pc_done[sd]
                 and all(id(self.layers[li].module.weight) in b1 for li in self._pc_layers[sd])]
        if not sides:
            return
        _, views = self._flat_grad_buffer(self._bucket_params)
        self._grad_src = {id(p): v for p, v in zip(self._bucket_params, views)}
        ev = torch.cuda.Event()
        ev.record(self.comm_stream)  # bucket-1 all-reduce and the A / early broadcasts
        u = self._g_streams[sides[0]]
        u.wait_event(ev)
        if invert_now:
            u.wait_stream(self.inv_stream)  # this rank's A inverses (and their staged planes)
            for sd in self._early:
                u.wait_stream(self._g_streams[sd])  # this rank's early G inverses
            for sd in ["A"] + self._early:
                self._exchange_recv(sd, u)
                self._recvd.add(sd)
        unpacked = torch.cuda.Event()
        unpacked.record(u)
        for sd in sides:
            s = self._g_streams[sd]
            s.wait_event(unpacked)
            self._run_precond(sd, s, lr)
            self._pc_done[sd] = True

    def _flat_grad_buffer(self, params):
        """One fp32 buffer holding every gradient (views with each parameter's shape and
        strides, which its gradient follows by autograd's layout contract, e.g. channels-last
        conv weights), allocated once per parameter layout.  Built from the parameters, so it
        also serves while later gradients of the step are still being accumulated."""
        layout = tuple((tuple(p.shape), tuple(p.stride()), p.dtype) for p in params)
        if getattr(self, "_flat_layout", None) != layout:
            dense = lambda g: g.is_contiguous() or (g.dim() == 4 and g.is_contiguous(memory_format=torch.channels_last))  # noqa: E731
            if any(not dense(p) or p.dtype != torch.float32 for p in params):
                raise RuntimeError("parameters must be dense float32 tensors")
            total = sum(p.numel() for p in params)
            flat = torch.empty(total, dtype=torch.float32, device=self.device)
            views, off = [], 0
            for p in params:
                n = p.numel()
                views.append(flat[off:off + n].as_strided(p.shape, p.stride()))
                off += n
            self._flat, self._flat_views, self._flat_layout = flat, views, layout
        return self._flat, self._flat_views

    def _after_replay(self, stream, inverted: bool = True) -> None:
        """Bookkeeping for one replay of a captured step (GraphedStep): the Python side
        effects of step() ran once at capture time."""
        self.steps += 1
        self._capture = self.steps % self.factor_update_freq == 0
        if not inverted:
            return
        for side in self._sides:
            if self._inv_plans[side] is not None:
                ev = torch.cuda.Event()
                ev.record(stream)
                self._info_events.append((ev, side, self.steps - 1, 0))

    def _exchange_send(self, side, src) -> None:
        """Owner ranks broadcast their CT inverses of one side (packed upper triangle,
        PAPER.md:281-283 / emulator.py:256-262), one NCCL broadcast per owner, on the comm
        stream once `src` (the stream that inverted them) has packed them.  Every rank issues
        the sends of an iteration in the same program order (single communicator)."""
        if self.world == 1 or self._sent[side]:
            return
        lib = L.load()
        lay = self._bcast[side]
        ct, dims, buf, views, n = lay[self.rank]
        if ct:
            L.check(lib.spdkfac_pack_upper_batched_f32(len(ct), L.i32_array(dims),
                                                       L.ptr_array([self.inv[t].data_ptr() for t in ct]),
                                                       L.ptr_array([v.data_ptr() for v in views]),
                                                       src.cuda_stream), "pack inverses")
        if self._peer_bcast:  # push into every peer's receive region, then raise this rank's flag
            if ct:
                self._peer.push_extra_all(self._bc_off[side][self.rank], buf[:n], src)
            self._peer.signal(self._peer_slot_bc[side], src)
            self._sent[side] = True
            return
        cs = self.comm_stream
        cs.wait_stream(src)
        with self.comm.group():
            for root, (ct_r, _, buf_r, _, n_r) in enumerate(lay):
                if n_r:
                    self.comm.bcast(buf_r[:n_r], root, cs)
        self._sent[side] = True

    def _exchange_recv(self, side, main) -> None:
        """Unpack the inverses received from the other owners (after main joined the comm stream):
        one pass per preconditioner group writes the full inverses and their operand planes."""
        if self._peer_bcast:  # every owner's pushes of this side have landed
            self._peer.wait(self._peer_slot_bc[side], main)
        for root, (ct_r, dims_r, _, views_r, n_r) in enumerate(self._bcast[side]):
            if root == self.rank or not ct_r:
                continue
            view = dict(zip(ct_r, views_r))
            for pside, plan in self._precond.items():
                for which, par in (("A", 0), ("G", 1)):
                    ts = [t for t in ct_r if t % 2 == par and self._pc_side[t // 2] == pside]
                    plan.stage_packed(which, [self._pc_local[t // 2] for t in ts], [view[t] for t in ts],
                                      [self.inv[t] for t in ts], main)

    def _stage_planes(self, tensors, stream) -> None:
        """Stage freshly produced inverses (tensor indices 2l / 2l+1) into the preconditioner
        group that owns their layer."""
        for side, plan in self._precond.items():
            for which, par in (("A", 0), ("G", 1)):
                ts = [t for t in tensors if t % 2 == par and self._pc_side[t // 2] == side]
                plan.stage_inverses(which, [self._pc_local[t // 2] for t in ts], [self.inv[t] for t in ts], stream)

    def _run_precond(self, side: str, stream, lr: float) -> None:
        """P = G^-1 grad A^-1 and W -= lr/P_world * P for the layers of one group, on `stream`;
        the pointer tables are rebuilt only when a gradient's storage changes."""
        layers = [self.layers[li] for li in self._pc_layers[side]]
        src = self._grad_src if self.world > 1 else {}
        grad_of = lambda p: src.get(id(p), p.grad)  # noqa: E731
        key = tuple(grad_of(l.module.weight).data_ptr() if l.module.weight.grad is not None else 0 for l in layers)
        plan = self._precond[side]
        if key != self._precond_key[side]:
            if 0 in key:
                missing = [l.name for l in layers if l.module.weight.grad is None]
                raise RuntimeError(f"layers {missing[:3]} have no gradient; call backward() before step()")
            for l in layers:  # memory format may change (model.to(channels_last) after construction)
                if l.is_conv:
                    l.w_cl = self._weight_channels_last(l.module)
            plan.bind([self.inv[2 * l.index + 1] for l in layers],
                      [self._weight_matrix(l, grad_of(l.module.weight)) for l in layers],
                      [self.inv[2 * l.index] for l in layers],
                      weights=[self._weight_matrix(l, l.module.weight.data) for l in layers])
            self._precond_key[side] = key
        # every inverse is staged by the stream that produced it once an inversion round has run
        plan.run_bound(lr / self.world, stream=stream, inverses_staged=not self._planes_stale)

    def _make_grad_hook(self, l: _Layer):
        def hook(param):
            if not self.update_in_backward or not l.module.training:
                return
            side = self._pc_side[l.index]
            self._grad_left[side] -= 1
            if self._grad_left[side] == 0 and side != self._tail:
                self._launch_precond(side)
        return hook

    def _launch_precond(self, side: str) -> None:
        """Every gradient of an early group's layers is accumulated (post-accumulate-grad hooks
        run after the layer's backward kernels were enqueued on the current stream): precondition
        and update those layers on the group's stream once its inverses exist."""
        if self._inverting() and not self._g_inverted[side]:
            return  # inverses not launched yet (factors reused / incomplete): step() handles it
        main = torch.cuda.current_stream(self.device)
        s = self._g_streams[side]
        s.wait_stream(main)
        if self._inverting():
            s.wait_stream(self.inv_stream)  # A inverses (the group's G inverses are on s already)
        self._run_precond(side, s, self.param_groups[0]["lr"])
        self._pc_done[side] = True

    # ------------------------------------------------------------------ introspection / checkpoint
    def factor(self, layer: int, kind: str) -> torch.Tensor:
        """Current aggregated (running-average) factor of a layer as a full matrix.  With
        factor_comm "reduce" / "peer" and P > 1 only the owner of the factor's inverse holds the
        aggregate (placement.owner(2 layer + side)); other ranks hold their own contribution
        ("reduce") or a stale buffer ("peer": their contribution went to the owner's inbox)."""
        from .linalg import unpack_upper
        t = 2 * layer + (0 if kind == "A" else 1)
        return unpack_upper(self._packed(t), self.inv[t].shape[0])

    def state_dict(self):
        sd = super().state_dict()
        sd["spdkfac"] = {"bufA": self.bufA.clone(), "bufG": self.bufG.clone(), "inv": [t.clone() for t in self.inv],
                         "steps": self.steps, "factor_updates": self._factor_updates}
        return sd

    def load_state_dict(self, sd):
        k = sd.pop("spdkfac", None)
        super().load_state_dict(sd)
        if k is not None:
            self.bufA.copy_(k["bufA"])
            self.bufG.copy_(k["bufG"])
            for t, s in zip(self.inv, k["inv"]):
                t.copy_(s)
            self._planes_stale = True
            self.steps = int(k["steps"])
            self._factor_updates = int(k["factor_updates"])
            self._capture = self.steps % self.factor_update_freq == 0
