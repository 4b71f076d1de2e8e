"""Precision probe (diagnostic): damped inverses of rank-deficient factors like ResNet-50's fc A
(rows = 32 pooled post-ReLU feature vectors, d = 2048) and small ones (d = 64, 128), tc vs ffma
pivot (run twice with SPDKFAC_PIVOT unset / =ffma); error vs float64 and vs cuSOLVER fp32."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2107_06533_b200.linalg import InversePlan, pack_upper  # noqa: E402

torch.manual_seed(0)
for d, m, scale in ((2048, 32, 1.0), (2048, 32, 10.0), (1024, 64, 1.0), (64, 32, 1.0), (128, 8, 1.0), (576, 100, 1.0)):
    a = torch.relu(torch.randn(m, d, device="cuda") + 0.3) * scale
    f = (a.T @ a / m)
    f = (f + f.T) / 2
    packed = [pack_upper(f)]
    out = [torch.empty(d, d, device="cuda")]
    plan = InversePlan(packed, out)
    plan.run(0.1)
    torch.cuda.synchronize()
    info = int(plan.info.item())
    f64 = f.double().cpu().numpy() + 0.1 * np.eye(d)
    want = np.linalg.inv(f64)
    want = (want + want.T) / 2
    err = np.linalg.norm(out[0].double().cpu().numpy() - want) / np.linalg.norm(want)
    t = torch.tensor(f64, dtype=torch.float32, device="cuda")
    ref = torch.cholesky_inverse(torch.linalg.cholesky(t)).double().cpu().numpy()
    eref = np.linalg.norm(ref - want) / np.linalg.norm(want)
    print(f"{os.environ.get('SPDKFAC_PIVOT', 'tc'):4s} d={d} m={m} scale={scale}: info={info} err={err:.3e} "
          f"cusolver={eref:.3e} kappa={np.linalg.cond(f64):.3e}", flush=True)
