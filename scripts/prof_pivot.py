"""Minimal driver for ncu captures of the inverse kernels: one d = 1024 damped inverse (8
pivot-block steps), run twice (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2107_06533_b200.linalg import InversePlan, pack_upper  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(d // 2, d, device="cuda", generator=g)
packed = [pack_upper(x.T @ x / x.shape[0])]
out = [torch.empty(d, d, device="cuda")]
plan = InversePlan(packed, out)
for _ in range(2):
    plan.run(0.1)
torch.cuda.synchronize()
plan.check()
print("ok", float(out[0].abs().sum()))
