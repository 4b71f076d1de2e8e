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

if what == "inverse_single":
    for d in (4608, 2304, 1024):
        g = torch.Generator(device=dev).manual_seed(d)
        b = torch.randn(d, d, device=dev, generator=g)
        m = b @ b.T / d + 0.1 * torch.eye(d, device=dev)
        r, c = torch.triu_indices(d, d, device=dev)
        plan = InversePlan([m[r, c].contiguous()], [torch.empty(d, d, device=dev)])
        L.stats_reset(timing=True)
        timed(lambda: plan.run(0.1), f"single inverse d={d}")
        report(reps + 1)

if what == "stage":  # every ResNet-50 bs32 layer side, channels-last, staging and SYRK timed apart
    from paper_2107_06533_b200.workloads import build_model
    model = build_model("resnet50").to(dev).to(memory_format=torch.channels_last)
    recs = []

    def hook(m, inp, out):
        recs.append((m, inp[0].detach(), out.detach()))

    hs = [m.register_forward_hook(hook) for m in model.modules() if isinstance(m, (torch.nn.Conv2d, torch.nn.Linear))]
    with torch.no_grad():
        model(torch.randn(32, 3, 224, 224, device=dev).contiguous(memory_format=torch.channels_last))
    for h in hs:
        h.remove()
    tot_stage = tot_syrk = tot_bytes = 0.0
    for m, x, y in recs:
        for side in ("A", "G"):
            if isinstance(m, torch.nn.Conv2d):
                if side == "A":
                    t = x.contiguous(memory_format=torch.channels_last)
                    plan = FactorPlan(L.CONV_A_NHWC, t.shape, m.kernel_size, m.stride, m.padding, m.dilation)
                else:
                    t = torch.randn_like(y).contiguous(memory_format=torch.channels_last)
                    plan = FactorPlan(L.SPATIAL_NHWC, t.shape)
            else:
                t = (x if side == "A" else torch.randn_like(y)).contiguous()
                plan = FactorPlan(L.ROWS, t.shape)
            packed = torch.zeros(plan.packed_size, device=dev)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            plan.stage(t)
            plan.compute(packed, 1.0)
            torch.cuda.synchronize()
            e[0].record()
            for _ in range(reps):
                plan.stage(t)
            e[1].record()
            for _ in range(reps):
                plan.compute(packed, 1.0)
            e[2].record()
            torch.cuda.synchronize()
            st, sy = e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps
            ld = (plan.dim + 7) // 8 * 8
            nbytes = plan.rows * ld * 4 + t.numel() * 4
            tot_stage += st
            tot_syrk += sy
            tot_bytes += nbytes
            print(f"{side} {tuple(t.shape)} k={getattr(m, 'kernel_size', '-')} M={plan.rows} d={plan.dim}: "
                  f"stage {st * 1e3:7.1f} us ({nbytes / st / 1e6:6.0f} GB/s)  syrk {sy * 1e3:7.1f} us "
                  f"({plan.rows * plan.dim * (plan.dim + 1) / sy / 1e9:6.1f} TF/s)", flush=True)
            del plan
    print(f"total stage {tot_stage:.3f} ms ({tot_bytes / tot_stage / 1e6:.0f} GB/s), syrk {tot_syrk:.3f} ms")

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

if what == "stage":
    # per-layer staging + SYRK time for every distinct ResNet-50 conv/fc shape (channels-last)
    import torch.nn as nn
    from paper_2107_06533_b200.workloads import build_model
    model = build_model("resnet50").to(dev).to(memory_format=torch.channels_last)
    geo = []

    def hook(m, inp, out):
        geo.append((m, tuple(inp[0].shape), tuple(out.shape)))
    hs = [m.register_forward_hook(hook) for m in model.modules() if isinstance(m, (nn.Conv2d, nn.Linear))]
    with torch.no_grad():
        model(torch.randn(32, 3, 224, 224, device=dev).contiguous(memory_format=torch.channels_last))
    for h in hs:
        h.remove()
    seen = {}
    tot = {"A_stage": 0.0, "A_syrk": 0.0, "G_stage": 0.0, "G_syrk": 0.0}
    for m, ishape, oshape in geo:
        for side in ("A", "G"):
            if isinstance(m, nn.Linear):
                key = (side, "fc")
                shp = ishape if side == "A" else oshape
                plan = FactorPlan(L.ROWS, shp)
                x = torch.randn(shp, device=dev)
            elif side == "A":
                key = ("A",) + ishape + tuple(m.kernel_size) + tuple(m.stride)
                plan = FactorPlan(L.CONV_A_NHWC, ishape, m.kernel_size, m.stride, m.padding, m.dilation)
                x = torch.randn(ishape, device=dev).contiguous(memory_format=torch.channels_last)
            else:
                key = ("G",) + oshape
                plan = FactorPlan(L.SPATIAL_NHWC, oshape)
                x = torch.randn(oshape, device=dev).contiguous(memory_format=torch.channels_last)
            if key not in seen:
                packed = torch.empty(plan.packed_size, device=dev)
                for _ in range(2):
                    plan.run(x, packed)
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record()
                for _ in range(5):
                    plan.stage(x)
                e[1].record()
                for _ in range(5):
                    plan.compute(packed, 1.0 / plan.rows)
                e[2].record()
                torch.cuda.synchronize()
                seen[key] = (e[0].elapsed_time(e[1]) / 5, e[1].elapsed_time(e[2]) / 5, plan.rows, plan.dim)
            st, sy, rows, dim = seen[key]
            tot[side + "_stage"] += st
            tot[side + "_syrk"] += sy
    for key, (st, sy, rows, dim) in seen.items():
        gbs = rows * dim * 4 / (st * 1e-3) / 1e9
        tf = rows * dim * (dim + 1) / (sy * 1e-3) / 1e12
        print(f"{str(key):60s} M={rows:7d} d={dim:5d} stage {st*1e3:8.1f} us ({gbs:6.0f} GB/s written)  syrk {sy*1e3:8.1f} us ({tf:6.1f} TF/s)")
    print({k: round(v, 3) for k, v in tot.items()}, "ms per step (sum over layers)")
