"""Standalone kernel driver for ncu / timing: runs the batched inverse plan on the
ResNet-50 bs32 factor dims and factor plans for the heaviest conv shapes, with
CUDA-event timing and per-category kernel stats.  Usage:
  python scripts/prof_kernels.py [inverse|factor|all] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06533_b200 import _lib as L
from paper_2107_06533_b200.linalg import FactorPlan, InversePlan
from paper_2107_06533_b200.workloads import layer_shapes

what = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
shapes = layer_shapes("resnet50", 32)
dims = []
for _, m, a, g in shapes:
    dims += [a, g]


def timed(fn, label):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / reps:.3f} ms", flush=True)


def report(runs):
    st = L.stats()
    for k, v in st.items():
        if isinstance(v, dict) and v["launches"]:
            tf = v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["ms"] else 0
            print(f"   {k:20s} {v['ms'] / runs:8.3f} ms/run  {v['launches'] / runs:6.1f} launches/run  {tf:7.1f} TFLOP/s")


if what in ("inverse", "all"):
    g = torch.Generator(device=dev).manual_seed(0)
    packed, outs = [], []
    for d in dims:
        b = torch.randn(d, d, device=dev, generator=g)
        m = b @ b.T / d + 0.1 * torch.eye(d, device=dev)
        r, c = torch.triu_indices(d, d, device=dev)
        packed.append(m[r, c].contiguous())
        outs.append(torch.empty(d, d, device=dev))
    plan = InversePlan(packed, outs)
    L.stats_reset(timing=True)
    timed(lambda: plan.run(0.1), "inverse plan (108 ResNet-50 factors)")
    report(reps + 1)
    plan.check()

if what in ("factor", "all"):
    L.stats_reset(timing=True)
    for label, shp, layout, k in [("A layer4 conv2 (M=1568, d=4608)", (32, 512, 7, 7), L.CONV_A, 3),
                                  ("A layer1 conv2 (M=100352, d=576)", (32, 64, 56, 56), L.CONV_A, 3),
                                  ("A conv1 (M=401408, d=147)", (32, 3, 224, 224), L.CONV_A, 7),
                                  ("G layer1 conv3 (M=100352, d=256)", (32, 256, 56, 56), L.SPATIAL, 1)]:
        x = torch.randn(shp, device=dev)
        if layout == L.CONV_A:
            st, pd = (2, 3) if k == 7 else (1, 1)
            plan = FactorPlan(layout, shp, (k, k), (st, st), (pd, pd))
        else:
            plan = FactorPlan(layout, shp)
        packed = torch.empty(plan.packed_size, device=dev)
        timed(lambda: plan.run(x, packed), "factor " + label)
    report(4 * (reps + 1))
