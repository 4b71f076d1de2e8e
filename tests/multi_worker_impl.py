"""Rank program for the multi-GPU parity test (launched by torchrun, one rank per GPU).

The reference's frozen fixture (aggregated_step_w4.json: 4 workers x 6 samples) is split
over the ranks (4 / P workers' samples per rank); the P-rank SPD-KFAC step (factor
all-reduce in fusion groups, LBP placement with owner broadcast of CT inverses, gradient
all-reduce) must reproduce the fixture's centralized-oracle weights, exactly as
dkfac_step does (emulator.py:211-263, worker-count invariance test_emulator.py:115-158).
Rank 0 prints one JSON line with the per-layer errors.
"""
import json
import os
import pathlib
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.nn as nn

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.perfmodel import PerfParams, AllReduceParams, BcastParams, InverseParams
    fx = json.loads((ROOT / "tests/golden/aggregated_step_w4.json").read_text())
    mods = []
    for w, act in zip(fx["weights"], fx["activations"]):
        w = np.array(w)
        lin = nn.Linear(w.shape[1], w.shape[0], bias=False)
        lin.weight.data = torch.tensor(w, dtype=torch.float32)
        mods.append(lin)
        if act == "relu":
            mods.append(nn.ReLU())
    model = nn.Sequential(*mods).to(dev)
    per = 4 // world
    xs = np.concatenate(fx["worker_inputs"][rank * per:(rank + 1) * per])
    ts = np.concatenate(fx["worker_targets"][rank * per:(rank + 1) * per])
    x = torch.tensor(xs, dtype=torch.float32, device=dev)
    t = torch.tensor(ts, dtype=torch.float32, device=dev)
    mode = os.environ.get("SPD_PLACEMENT", "lbp")
    # all-CT calibration: every inverse has one owner and is broadcast (exercises the bcast path);
    # lbp-nct: the B200 marginal batched-inverse model with a threshold inside the fixture's dims
    # (d <= 5 replicated on every rank, d = 6 owned + broadcast)
    perf = PerfParams(AllReduceParams(1e-5, 1e-9), BcastParams(1e-9, 1e-12), InverseParams(1.0, 1e-6), world)
    if mode == "lbp-nct":
        from paper_2107_06533_b200.perfmodel import MarginalInverseParams
        perf = PerfParams(perf.allreduce, perf.bcast, perf.inverse, world, MarginalInverseParams(1e-13))
        mode = "lbp"
        assert 5 < __import__("paper_2107_06533_b200.perfmodel", fromlist=["x"]).nct_threshold(perf.marginal, perf.bcast) <= 6
    opt = SPDKFAC(model, lr=fx["alpha"], damping=fx["gamma"], placement=mode, perf=perf)
    loss = ((model(x) - t) ** 2).mean()
    loss.backward()
    opt.step()
    torch.cuda.synchronize()
    errs = []
    for lin, w0, want in zip([m for m in model if isinstance(m, nn.Linear)], fx["weights"], fx["expected_weights"]):
        got = lin.weight.detach().double().cpu().numpy()
        d = np.array(want) - np.array(w0)
        errs.append(float(np.linalg.norm(got - np.array(w0) - d) / np.linalg.norm(d)))
    # weights must be identical on every rank
    w_all = torch.cat([p.detach().flatten() for p in model.parameters()])
    ref = w_all.clone()
    dist.broadcast(ref, 0)
    same = bool(torch.equal(ref, w_all))
    ok = torch.tensor([1 if same else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # several steps of a conv net: the gradient bucket all-reduced during backward (P > 1) gives the
    # same weights as one all-reduce in step()
    def convnet():
        torch.manual_seed(5)
        return nn.Sequential(nn.Conv2d(3, 8, 3, padding=1), nn.BatchNorm2d(8), nn.ReLU(), nn.Conv2d(8, 16, 3, padding=1),
                             nn.ReLU(), nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(16, 10)).to(dev)
    m_a, m_b = convnet(), convnet()
    o_a = SPDKFAC(m_a, lr=0.05, damping=0.1, placement=mode, perf=perf)
    o_b = SPDKFAC(m_b, lr=0.05, damping=0.1, placement=mode, perf=perf)
    o_b._bucket1 = []  # no bucketing: every gradient all-reduced in step()
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    crit = nn.CrossEntropyLoss()
    for _ in range(3):
        xb = torch.randn(6, 3, 8, 8, device=dev, generator=g)
        yb = torch.randint(0, 10, (6,), device=dev, generator=g)
        for m, o in ((m_a, o_a), (m_b, o_b)):
            o.zero_grad(set_to_none=True)
            crit(m(xb), yb).backward()
            o.step()
    torch.cuda.synchronize()
    bucket_err = max(float((pa - pb).abs().max() / (pb.abs().max() + 1e-30))
                     for pa, pb in zip(m_a.parameters(), m_b.parameters()))
    bucketed = bool(o_a._bucket1)
    for o in (o_a, o_b):
        o.comm.close()
    if rank == 0:
        print(json.dumps({"errors": errs, "identical_on_all_ranks": bool(ok.item()), "world": world,
                          "bucket_err": bucket_err, "bucketed": bucketed,
                          "placement": os.environ.get("SPD_PLACEMENT", "lbp"), "nct": sorted(opt.placement.nct),
                          "workers": [list(w) for w in opt.placement.workers]}), flush=True)
    opt.comm.close()
    if opt.comm_bc is not None and opt.comm_bc is not opt.comm:
        opt.comm_bc.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
