"""Diagnostic: one channels-last conv factor through the TMA-im2col SYRK vs float64 (argv: n c h w kh kw ph pw)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle as O  # noqa: E402
from paper_2107_06533_b200 import _lib as L  # noqa: E402
from paper_2107_06533_b200.linalg import FactorGroup, unpack_upper  # noqa: E402

n, c, h, w, kh, kw, ph, pw = (int(v) for v in sys.argv[1:9])
x = torch.relu(torch.randn(n, c, h, w, device="cuda") + 0.2).contiguous(memory_format=torch.channels_last)
ho, wo = h + 2 * ph - kh + 1, w + 2 * pw - kw + 1
d, m = c * kh * kw, n * ho * wo
packed = [torch.zeros(d * (d + 1) // 2, device="cuda")]
grp = FactorGroup([(L.CONV_A_NHWC, (n, c, h, w), (kh, kw), (1, 1), (ph, pw), (1, 1))], packed, [1.0 / m])
grp.stage(0, x)
grp.compute()
torch.cuda.synchronize()
rows = O.im2col_rows(x.double().cpu().numpy(), kh, kw, 1, (ph, pw))
perm = [ci * kh * kw + ki * kw + kj for ki in range(kh) for kj in range(kw) for ci in range(c)]
want = (rows.T @ rows / m)[np.ix_(perm, perm)]
got = unpack_upper(packed[0], d).double().cpu().numpy()
print("rel err", np.linalg.norm(got - want) / np.linalg.norm(want))
