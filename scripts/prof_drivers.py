"""Small drivers for ncu captures (diagnostic): `inverse` runs the 108 ResNet-50 factors' batched
damped inverse twice; `stage` stages + computes the ResNet-50 bs32 factors of a few layer shapes
(rows, 3x3 im2col, spatial G) through FactorPlan twice."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2107_06533_b200 import _lib as L  # noqa: E402
from paper_2107_06533_b200.linalg import FactorPlan, InversePlan, pack_upper  # noqa: E402
from paper_2107_06533_b200.workloads import layer_shapes  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "inverse"
if what == "inverse":
    dims = []
    for _, m, a, g in layer_shapes("resnet50", 32):
        dims += [a, g]
    packed, outs = [], []
    for i, d in enumerate(dims):
        gen = torch.Generator(device="cuda").manual_seed(i)
        x = torch.randn(max(d // 2, 64), d, device="cuda", generator=gen)
        packed.append(pack_upper(x.T @ x / x.shape[0]))
        outs.append(torch.empty(d, d, device="cuda"))
    plan = InversePlan(packed, outs)
    for _ in range(2):
        plan.run(0.1)
    torch.cuda.synchronize()
    plan.check()
elif what == "stage":
    cl = torch.channels_last
    cases = [(L.CONV_A_NHWC, (32, 64, 56, 56), (3, 3), (1, 1), (1, 1)),      # layer1 conv2 A (im2col)
             (L.CONV_A_NHWC, (32, 256, 56, 56), (1, 1), (1, 1), (0, 0)),     # layer1 1x1 A (rows)
             (L.SPATIAL_NHWC, (32, 256, 56, 56), (1, 1), (1, 1), (0, 0))]    # layer1 G (rows)
    for layout, shape, k, st, pd in cases:
        x = torch.randn(shape, device="cuda").contiguous(memory_format=cl)
        plan = FactorPlan(layout, shape, k, st, pd) if layout == L.CONV_A_NHWC else FactorPlan(layout, shape)
        packed = torch.empty(plan.packed_size, device="cuda")
        for _ in range(2):
            plan.run(x, packed)
    torch.cuda.synchronize()
print("ok")
