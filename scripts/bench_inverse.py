"""Isolated timing of the batched damped inverse (diagnostic): one d = 4608 matrix (36 pivot
steps) and the 108 ResNet-50 factors in one plan, per-category kernel times from the library's
launch events.  Usage: python scripts/bench_inverse.py  (SPDKFAC_PIVOT=ffma: round-1 pivot)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2107_06533_b200 import _lib as L  # noqa: E402
from paper_2107_06533_b200.linalg import InversePlan, pack_upper  # noqa: E402
from paper_2107_06533_b200.workloads import layer_shapes  # noqa: E402


def spd(d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(max(d // 2, 64), d, device="cuda", generator=g)
    return x.T @ x / x.shape[0]


def run(dims, reps=5):
    packed = [pack_upper(spd(d, i)) for i, d in enumerate(dims)]
    outs = [torch.empty(d, d, device="cuda") for d in dims]
    plan = InversePlan(packed, outs)
    plan.run(0.1)
    torch.cuda.synchronize()
    plan.check()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.run(0.1)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / reps
    L.stats_reset(timing=True, reserve=4000)
    plan.run(0.1)
    torch.cuda.synchronize()
    st = L.stats()
    cats = {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                "us_per_launch": round(1e3 * v["ms"] / v["launches"], 2) if v["launches"] else None}
            for k, v in st.items() if isinstance(v, dict) and v["launches"]}
    return {"ms_total": round(total, 4), "cats": cats}


out = {"pivot": os.environ.get("SPDKFAC_PIVOT", "tc")}
out["d4608"] = run([4608])
out["d1024x8"] = run([1024] * 8)
dims = []
for _, m, a, g in layer_shapes("resnet50", 32):
    dims += [a, g]
out["resnet50_all108"] = run(dims, reps=3)
print(json.dumps(out, indent=1))
