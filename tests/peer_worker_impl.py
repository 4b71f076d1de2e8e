"""Rank program for the peer-memory factor aggregation test (launched by torchrun, one rank per GPU).

factor_comm = "peer" (csrc/peer.cu, comm.PeerExchange) must give the same steps as the NCCL
reduce onto the owner ("reduce"), which tests/test_gpu_multi.py ties to the reference's
centralized step (emulator.py:211-263): several eager steps and several CUDA-graph replays of a
small conv net (grouped SYRK launches from the second step on, CT factors owned by both ranks,
NCT factors all-reduced), rank-specific data.  Rank 0 prints one JSON line.
"""
import json
import os
import pathlib
import sys

import torch
import torch.distributed as dist
import torch.nn as nn

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def convnet(dev):
    torch.manual_seed(7)
    m = nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.BatchNorm2d(16), nn.ReLU(), nn.Conv2d(16, 32, 3, padding=1),
                      nn.ReLU(), nn.Conv2d(32, 48, 1), nn.ReLU(), nn.Conv2d(48, 64, 3, padding=1, stride=2), nn.ReLU(),
                      nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(64, 10))
    return m.to(dev).to(memory_format=torch.channels_last)


def main():
    import faulthandler
    faulthandler.dump_traceback_later(150, exit=True)  # a stalled rank prints where it is and exits
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    # deterministic convolution backward: the two modes' runs may then differ only by the aggregation
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.perfmodel import AllReduceParams, BcastParams, InverseParams, PerfParams
    # every inverse owned by one rank and broadcast (CT), LBP spreading them over the ranks
    perf = PerfParams(AllReduceParams(1e-5, 1e-9), BcastParams(1e-9, 1e-12), InverseParams(1.0, 1e-6), world)
    crit = nn.CrossEntropyLoss()
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    data = [(torch.randn(8, 3, 16, 16, device=dev, generator=g).contiguous(memory_format=torch.channels_last),
             torch.randint(0, 10, (8,), device=dev, generator=g)) for _ in range(6)]
    out, keep = {}, []
    log = lambda *a: print(f"[rank {rank}]", *a, file=sys.stderr, flush=True)  # noqa: E731
    for mode in ("reduce", "peer"):
        # eager: the first step runs per-layer plans (NCCL), the grouped path (peer writes) from the second on
        m = convnet(dev)
        log(mode, "constructing")
        o = SPDKFAC(m, lr=0.05, damping=0.1, factor_comm=mode, perf=perf)
        log(mode, "constructed")
        for i, (x, y) in enumerate(data[:4]):
            o.zero_grad(set_to_none=True)
            crit(m(x), y).backward()
            o.step()
            torch.cuda.synchronize()
            log(mode, "eager step", i, "peer error", o._peer.error() if o._peer is not None else None)
        o.check_inverses()
        owned = [t for t in range(2 * len(o.layers)) if t not in o.placement.nct and o.placement.owner(t) == rank]
        out[mode] = {"eager": torch.cat([p.detach().flatten() for p in m.parameters()]),
                     "factors": {t: o.factor(t // 2, "AG"[t % 2]).clone() for t in owned},
                     "active": o._peer is not None and o._fgroups is not None, "nct": sorted(o.placement.nct)}
        o.remove_hooks()
        o.comm.close()
        # CUDA graph: warm-up steps, capture, replays
        m = convnet(dev)
        o = SPDKFAC(m, lr=0.05, damping=0.1, factor_comm=mode, perf=perf)
        gs = GraphedStep(m, crit, o, [data[0][0]], [data[0][1]], warmup=3)
        log(mode, "captured")
        for x, y in data[1:4]:
            gs([x], [y])
        torch.cuda.synchronize()
        log(mode, "replayed")
        o.check_inverses()
        out[mode]["graph"] = torch.cat([p.detach().flatten() for p in m.parameters()])
        o.remove_hooks()
        keep.append((gs, o))  # a communicator captured into a live CUDA graph is not destroyed (ncclCommDestroy stalls)
        # inverses every second step: two captured step types, aggregation on both, inversion on one
        m = convnet(dev)
        o = SPDKFAC(m, lr=0.05, damping=0.1, factor_comm=mode, perf=perf, inv_update_freq=2)
        gs = GraphedStep(m, crit, o, [data[0][0]], [data[0][1]], warmup=3)
        for x, y in data[1:6]:
            gs([x], [y])
        torch.cuda.synchronize()
        o.check_inverses()
        log(mode, "freq-2 replayed")
        out[mode]["freq2"] = torch.cat([p.detach().flatten() for p in m.parameters()])
        o.remove_hooks()
        keep.append((gs, o))

    def rel(a, b):
        return float((a - b).abs().max() / (b.abs().max() + 1e-30))

    r, p = out["reduce"], out["peer"]
    res = {"eager_err": rel(p["eager"], r["eager"]), "graph_err": rel(p["graph"], r["graph"]),
           "eager_exact": bool(torch.equal(p["eager"], r["eager"])),
           "graph_exact": bool(torch.equal(p["graph"], r["graph"])),
           "freq2_err": rel(p["freq2"], r["freq2"]), "freq2_exact": bool(torch.equal(p["freq2"], r["freq2"])),
           "factor_err": max([rel(p["factors"][t], r["factors"][t]) for t in r["factors"]] or [0.0]),
           "owned": len(r["factors"]), "active": p["active"] and not r["active"], "nct": p["nct"], "world": world}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps({"ranks": allres}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
