"""The multi-rank step logic on CPU (torch.distributed gloo, world size 2 and 4).

Each rank runs the SPD-KFAC schedule of the B200 step -- the same schedule.py layout,
fusion groups and owner broadcasts SPDKFAC uses -- with the float64 oracle standing in
for the CUDA kernels, and the gloo collectives performing the real exchanges:

  factors packed into the fusion buffers pre-scaled by 1/P, one all_reduce per fusion group
  in plan order (forward: A, backward: G) -- or, factor_comm "reduce", each CT factor summed
  onto its inverse's owner only; gradient all_reduce; LBP placement; each rank
  inverts its own share; CT inverses broadcast in packed form from their owners; update.

The result must equal the reference's centralized step on the union batch (the frozen
fixture aggregated_step_w4.json) -- dkfac_step's worker-count invariance
(emulator.py:211-263, test_emulator.py:115-158) -- and be identical on every rank.
"""

import json
import os
import pathlib
import socket
from types import SimpleNamespace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle as O  # noqa: E402
from paper_2107_06533_b200 import planner as P  # noqa: E402
from paper_2107_06533_b200 import schedule as S  # noqa: E402
from paper_2107_06533_b200.perfmodel import AllReduceParams, BcastParams, InverseParams  # noqa: E402

GOLD = pathlib.Path(__file__).parent / "golden"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, placement_mode, out_dir, factor_comm="allreduce"):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    fx = json.loads((GOLD / "aggregated_step_w4.json").read_text())
    weights = [np.array(w) for w in fx["weights"]]
    acts = fx["activations"]
    per = 4 // world
    x = np.concatenate(fx["worker_inputs"][rank * per:(rank + 1) * per])
    t = np.concatenate(fx["worker_targets"][rank * per:(rank + 1) * per])
    _, ins, gs, dws = O.mlp_forward_backward(weights, acts, x, t)
    nl = len(weights)
    a_dims = [w.shape[1] for w in weights]
    g_dims = [w.shape[0] for w in weights]
    specs = [SimpleNamespace(a_dim=a, g_dim=g, t_factorA=1e-5 * (i + 1), t_factorG=2e-5, t_ff=1e-5, t_bp=2e-5)
             for i, (a, g) in enumerate(zip(a_dims, g_dims))]
    ar = AllReduceParams(1.5e-5, 1e-9)
    fwd = P.plan_fusion(P.factor_tasks(specs, P.FactorKind.A), [s.t_ff for s in specs], ar, P.FusionPolicy.OPTIMAL)
    bwd = P.plan_fusion(P.factor_tasks(specs, P.FactorKind.G), [s.t_bp for s in reversed(specs)], ar,
                        P.FusionPolicy.OPTIMAL)
    a_off, g_off, sa, sg = S.packed_layout(a_dims, g_dims)
    sl_a, sl_g = S.fusion_slices(fwd, a_off, a_dims), S.fusion_slices(bwd, g_off, g_dims)
    S.check_fusion_cover(sl_a, sa)
    S.check_fusion_cover(sl_g, sg)
    dims = [d for l in range(nl) for d in (a_dims[l], g_dims[l])]
    tasks = P.inverse_tasks(specs)
    if placement_mode == "lbp":  # all-CT calibration: every inverse travels from its owner
        plan = P.lbp_place(tasks, world, InverseParams(1.0, 1e-6), BcastParams(1e-9, 1e-12))
    elif placement_mode == "lbp_nct":  # everything cheaper to recompute than to send
        plan = P.lbp_place(tasks, world, InverseParams(1e-9, 1e-9), BcastParams(10.0, 1e-9))
    else:
        plan = P.seq_place(tasks, world)
    # factor_comm "reduce": each group's CT factors are summed onto their inverse's owner only
    # (schedule.reduce_segments), NCT ones all-reduced -- what SPDKFAC does for factor_decay == 0
    seg_a = dict(zip([g[-1].layer_index - 1 for g in fwd.groups], S.reduce_segments(fwd, a_off, a_dims, plan, 0)))
    seg_g = dict(zip([g[-1].layer_index - 1 for g in bwd.groups], S.reduce_segments(bwd, g_off, g_dims, plan, 1)))

    def aggregate(buf, sl, segs):
        if factor_comm == "allreduce":
            s, e = sl
            dist.all_reduce(buf[s:e])
            return
        for s, e, root in segs:
            if root is None:
                dist.all_reduce(buf[s:e])
            else:
                dist.reduce(buf[s:e], dst=root)

    buf_a, buf_g = torch.zeros(sa, dtype=torch.float64), torch.zeros(sg, dtype=torch.float64)
    for l in range(nl):  # forward pass order
        d = a_dims[l]
        buf_a[a_off[l]:a_off[l] + d * (d + 1) // 2] = torch.from_numpy(O.pack_upper(O.factor_A(ins[l])) / world)
        if l in sl_a:
            aggregate(buf_a, sl_a[l], seg_a[l])
    for l in reversed(range(nl)):  # backward pass order
        d = g_dims[l]
        buf_g[g_off[l]:g_off[l] + d * (d + 1) // 2] = torch.from_numpy(O.pack_upper(O.factor_G(gs[l])) / world)
        if l in sl_g:
            aggregate(buf_g, sl_g[l], seg_g[l])
    grads = [torch.from_numpy(np.ascontiguousarray(g)) for g in dws]
    for g in grads:
        dist.all_reduce(g)

    def packed(ti):
        l, side = ti // 2, ti % 2
        d = dims[ti]
        if side == 0:
            return buf_a[a_off[l]:a_off[l] + d * (d + 1) // 2].numpy()
        return buf_g[g_off[l]:g_off[l] + d * (d + 1) // 2].numpy()

    inv = {ti: O.damped_inverse(O.unpack_upper(packed(ti), dims[ti]), fx["gamma"]) for ti in plan.workers[rank]}
    for parity in (0, 1):
        for owner, (ct, dd, offs, n) in enumerate(S.bcast_layout(plan, dims, parity)):
            if not n:
                continue
            buf = torch.zeros(n, dtype=torch.float64)
            if owner == rank:
                for ti, d, o in zip(ct, dd, offs):
                    buf[o:o + d * (d + 1) // 2] = torch.from_numpy(O.pack_upper(inv[ti]))
            dist.broadcast(buf, src=owner)
            for ti, d, o in zip(ct, dd, offs):
                inv[ti] = O.unpack_upper(buf[o:o + d * (d + 1) // 2].numpy(), d)
    assert set(inv) == set(range(2 * nl)), "every inverse is on every rank after the exchange"
    new = [weights[l] - fx["alpha"] * O.precondition(grads[l].numpy() / world, inv[2 * l], inv[2 * l + 1])
           for l in range(nl)]
    err = max(float(np.abs(w - np.array(e)).max()) for w, e in zip(new, fx["expected_weights"]))
    flat = torch.from_numpy(np.concatenate([w.ravel() for w in new]))
    ref = flat.clone()
    dist.broadcast(ref, src=0)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([err, float(torch.equal(ref, flat))]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,placement,factor_comm", [(2, "lbp", "allreduce"), (2, "lbp_nct", "allreduce"),
                                                        (2, "seq", "allreduce"), (4, "lbp", "allreduce"),
                                                        (2, "seq", "reduce"), (4, "lbp", "reduce"),
                                                        (2, "lbp_nct", "reduce")])
def test_multirank_schedule_reproduces_centralized_step(tmp_path, world, placement, factor_comm):
    port = _free_port()
    mp.spawn(_rank_main, args=(world, port, placement, str(tmp_path), factor_comm), nprocs=world, join=True)
    for r in range(world):
        err, same = np.load(tmp_path / f"r{r}.npy")
        assert err < 1e-8, (r, err)
        assert same == 1.0


def test_bcast_layout_covers_ct_once():
    tasks = P.inverse_tasks([SimpleNamespace(a_dim=d, g_dim=d // 2 + 1) for d in (64, 147, 576, 2048, 4608)])
    dims = [t.dim for t in tasks]
    for world in (2, 4, 8):
        plan = P.lbp_place(tasks, world, InverseParams(1.0, 1e-6), BcastParams(1e-9, 1e-12))
        seen = []
        for parity in (0, 1):
            for owner, (ct, dd, offs, n) in enumerate(S.bcast_layout(plan, dims, parity)):
                assert all(plan.owner(t) == owner for t in ct)
                assert n == sum(d * (d + 1) // 2 for d in dd)
                seen += ct
        assert sorted(seen) == sorted(t for t in range(len(dims)) if t not in plan.nct)
