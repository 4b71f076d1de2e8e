"""Fit the three cost models of the planners on this machine (perfmodel.py:126-182).

  python -m torch.distributed.run --nproc-per-node P -m paper_2107_06533_b200.calibrate [--out PATH]

  all-reduce  alpha_ar + beta_ar * m        NCCL all-reduce(sum) of m fp32 elements on the
                                            optimizer's own communicator (fit_linear)
  broadcast   alpha_bcast + beta_bcast * d(d+1)/2   packed-triangle NCCL broadcast (fit_linear)
  inverse     alpha_inv * exp(beta_inv * d)  one damped inverse on one GPU (fit_exponential)
  marginal    c3 * d^3                        B200 extension: the ResNet-50 factor set inverted in ONE
                                              batched plan, c3 = time / sum d^3 (MarginalInverseParams)

Times are CUDA-event medians, max over ranks.  Rank 0 writes the reference's key-value
params format (write_params, perfmodel.py:221-235) with fitted_world_size = P; bench.py and
SPDKFAC load data/b200_p{P}.params for their world size (perfmodel.default_params(world)).
"""

from __future__ import annotations

import argparse
import os
import statistics

import torch
import torch.distributed as dist

from .perfmodel import (AllReduceParams, BcastParams, BenchSample, MarginalInverseParams, PerfParams,
                        fit_exponential, fit_linear, nct_threshold, write_params, DEFAULT_PARAMS_PATH)


def _time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def _max(v, dev):
    if not dist.is_initialized():
        return v
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None, help="default: data/b200_p{P}.params")
    ap.add_argument("--inverse-dims", default="64,128,256,512,1024,2048,3072,4608")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from .linalg import InversePlan
    # ---- inverse model (each rank measures; max over ranks)
    inv_samples = []
    for d in [int(x) for x in a.inverse_dims.split(",")]:
        g = torch.Generator(device=dev).manual_seed(d)
        b = torch.randn(d, d, device=dev, generator=g)
        m = b @ b.T / d + 0.1 * torch.eye(d, device=dev)
        r, c = torch.triu_indices(d, d, device=dev)
        packed = m[r, c].contiguous()
        out = torch.empty(d, d, device=dev)
        plan = InversePlan([packed], [out])
        t = _max(_time(lambda: plan.run(0.1), reps=5), dev)
        inv_samples.append(BenchSample(d, t))
    inv = fit_exponential(inv_samples)
    # ---- marginal batched model: every ResNet-50 factor in one plan (what a rank's placement share
    # runs as), c3 = time / sum d^3
    from .workloads import layer_shapes
    dims = [x for _, _, a_, g_ in layer_shapes("resnet50", 32) for x in (a_, g_)]
    packs, outs = [], []
    for i, d in enumerate(dims):
        g = torch.Generator(device=dev).manual_seed(i)
        b = torch.randn(d, d, device=dev, generator=g)
        m = b @ b.T / d + 0.1 * torch.eye(d, device=dev)
        r, c = torch.triu_indices(d, d, device=dev)
        packs.append(m[r, c].contiguous())
        outs.append(torch.empty(d, d, device=dev))
    bplan = InversePlan(packs, outs)
    t_batch = _max(_time(lambda: bplan.run(0.1), reps=3), dev)
    marginal = MarginalInverseParams(t_batch / float(sum(float(d) ** 3 for d in dims)))
    del packs, outs, bplan
    ar = bc = None
    ar_samples, bc_samples = [], []
    if world > 1:
        from .comm import NcclComm
        comm = NcclComm(rank, world)
        s = torch.cuda.current_stream()
        for e in [1 << k for k in range(10, 27, 2)]:
            buf = torch.ones(e, device=dev)
            t = _max(_time(lambda: comm.allreduce_sum(buf, s)), dev)
            ar_samples.append(BenchSample(e, t))
        for d in (64, 128, 256, 512, 1024, 2048, 4096):
            n = d * (d + 1) // 2
            buf = torch.ones(n, device=dev)
            t = _max(_time(lambda: comm.bcast(buf, 0, s)), dev)
            bc_samples.append(BenchSample(n, t))
        far, fbc = fit_linear(ar_samples), fit_linear(bc_samples)
        ar = AllReduceParams(max(far.alpha, 1e-7), far.beta)
        bc = BcastParams(max(fbc.alpha, 1e-7), fbc.beta)
        comm.close()
    else:  # single GPU: keep the collective models of the shipped file (fitted at P > 1)
        from .perfmodel import default_params
        p0 = default_params()
        ar, bc = p0.allreduce, p0.bcast
    if rank == 0:
        params = PerfParams(ar, bc, inv, world, marginal)
        out = a.out or str(DEFAULT_PARAMS_PATH.parent / f"b200_p{world}.params")
        write_params(out, params)
        print("batched inversion of the ResNet-50 factor set:", round(t_batch * 1e3, 3), "ms; c3 =", marginal.c3,
              "; marginal nct_threshold =", nct_threshold(marginal, bc), "; exponential nct_threshold =",
              nct_threshold(inv, bc))
        print("inverse samples (d, s):", [(s.size, round(s.time, 6)) for s in inv_samples])
        print("all-reduce samples (elems, s):", [(s.size, round(s.time, 6)) for s in ar_samples])
        print("bcast samples (elems, s):", [(s.size, round(s.time, 6)) for s in bc_samples])
        print("wrote", out, params)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
