"""Probe: accumulation error of the tcgen05 tile engine vs K (diagnostic, not a test).
Operands exactly representable (tf32 / bf16), so the only error is the MMA's internal
summation and the TMEM accumulation."""
import numpy as np
import torch
import paper_2107_06533_b200.linalg as K
from paper_2107_06533_b200 import _lib as L

torch.manual_seed(0)
def tf32(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)
def bf16(x):
    return x.to(torch.bfloat16).to(torch.float32)

for kdim in (128, 512, 2048, 4608):
    for kind in ("pos", "signed"):
        g = torch.rand(128, kdim, device="cuda") + 0.5 if kind == "pos" else torch.randn(128, kdim, device="cuda")
        a = torch.rand(kdim, kdim, device="cuda") + 0.5 if kind == "pos" else torch.randn(kdim, kdim, device="cuda")
        a = tf32((a + a.T) / 2)
        g = tf32(g)
        gi = torch.eye(128, device="cuda")
        out = K.precondition(g, a, gi)
        want = g.double() @ a.double()
        err = (out.double() - want)
        rel = (err.norm() / want.norm()).item()
        bias = (err.sum() / want.abs().sum()).item()
        # per-element error relative to sum |products|
        scale = g.double().abs() @ a.double().abs()
        print(f"precond tf32 K={kdim:5d} {kind:6s} relF={rel:.2e} mean_rel_bias={bias:+.2e} "
              f"max|err|/sum|prod|={(err.abs() / scale).max().item():.2e}", flush=True)

for m in (256, 1024, 4096, 16384):
    for kind in ("pos", "signed"):
        x = torch.rand(m, 128, device="cuda") + 0.5 if kind == "pos" else torch.randn(m, 128, device="cuda")
        x = bf16(x)
        plan = K.FactorPlan(L.ROWS, x.shape)
        packed = torch.empty(plan.packed_size, device="cuda")
        plan.run(x, packed, scale=1.0)
        got = K.unpack_upper(packed, 128).double()
        want = x.double().T @ x.double()
        err = got - want
        scale = x.double().abs().T @ x.double().abs()
        print(f"syrk bf16 M={m:6d} {kind:6s} relF={(err.norm() / want.norm()).item():.2e} "
              f"mean_rel_bias={(err.sum() / want.abs().sum()).item():+.2e} "
              f"max|err|/sum|prod|={(err.abs() / scale).max().item():.2e}", flush=True)
