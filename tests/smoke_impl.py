"""One small SPD-KFAC step on cuda:0 checked against the CPU oracle.

Used by `__graft_entry__.smoke()` and by tests/test_gpu_optimizer.py.
  1. the reference's frozen golden fixture (pkg/tests/data/aggregated_step_w4.json:
     bias-free MLP [5,5,6,4], MSE loss, 4 workers x 6 samples) through the full
     optimizer path; the P-worker step equals the union-batch step
     (test_emulator.py:115-158), so one rank on the union batch must reproduce
     the fixture's expected weights;
  2. a small conv net (conv 3x3 s1 p1, conv 3x3 s2 p1, conv 1x1, linear) one step,
     every layer's new weight compared with the oracle's
     `layer_kfac_update` on the captured activations / output gradients.
"""

from __future__ import annotations

import json
import pathlib

import numpy as np
import torch
import torch.nn as nn

import oracle as O

GOLD = pathlib.Path(__file__).parent / "golden"
TOL = 1e-4  # relative Frobenius error of the weight update (north_star fp32 bound)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def fixture_step(device="cuda:0"):
    from paper_2107_06533_b200.optimizer import SPDKFAC
    fx = json.loads((GOLD / "aggregated_step_w4.json").read_text())
    mods = []
    for w, act in zip(fx["weights"], fx["activations"]):
        w = np.array(w)
        lin = nn.Linear(w.shape[1], w.shape[0], bias=False)
        lin.weight.data = torch.tensor(w, dtype=torch.float32)
        mods.append(lin)
        if act == "relu":
            mods.append(nn.ReLU())
    model = nn.Sequential(*mods).to(device)
    x = torch.tensor(np.concatenate(fx["worker_inputs"]), dtype=torch.float32, device=device)
    t = torch.tensor(np.concatenate(fx["worker_targets"]), dtype=torch.float32, device=device)
    opt = SPDKFAC(model, lr=fx["alpha"], damping=fx["gamma"])
    loss = ((model(x) - t) ** 2).mean()
    loss.backward()
    opt.step()
    torch.cuda.synchronize()
    errs = []
    for lin, w0, want in zip([m for m in model if isinstance(m, nn.Linear)], fx["weights"], fx["expected_weights"]):
        got = lin.weight.detach().double().cpu().numpy()
        errs.append(_rel(got - np.array(w0), np.array(want) - np.array(w0)))
    opt.remove_hooks()
    return errs


class SmallNet(nn.Module):
    def __init__(self):
        super().__init__()
        self.c1 = nn.Conv2d(3, 8, 3, 1, 1, bias=False)
        self.c2 = nn.Conv2d(8, 16, 3, 2, 1, bias=False)
        self.c3 = nn.Conv2d(16, 16, 1, bias=False)
        self.fc = nn.Linear(16 * 4 * 4, 10, bias=False)

    def forward(self, x):
        x = torch.relu(self.c1(x))
        x = torch.relu(self.c2(x))
        x = torch.relu(self.c3(x))
        return self.fc(x.flatten(1))


def conv_step(device="cuda:0", seed=0, gamma=0.1, lr=0.1, channels_last=False):
    from paper_2107_06533_b200.optimizer import SPDKFAC
    torch.manual_seed(seed)
    model = SmallNet().to(device)
    if channels_last:
        model = model.to(memory_format=torch.channels_last)
    w0 = {n: m.weight.detach().double().cpu().numpy().copy() for n, m in model.named_children()}
    cap = {}

    def pre(name):
        def h(m, inp):
            cap[name + ".in"] = inp[0].detach().double().cpu().numpy()
        return h

    def post(name):
        def h(m, inp, out):
            out.register_hook(lambda g: cap.__setitem__(name + ".g", g.detach().double().cpu().numpy()))
        return h

    for n, m in model.named_children():
        m.register_forward_pre_hook(pre(n))
        m.register_forward_hook(post(n))
    opt = SPDKFAC(model, lr=lr, damping=gamma)
    b = 16
    x = torch.randn(b, 3, 8, 8, device=device)
    if channels_last:
        x = x.contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 10, (b,), device=device)
    loss = nn.functional.cross_entropy(model(x), y)
    loss.backward()
    grads = {n: m.weight.grad.detach().double().cpu().numpy().reshape(m.weight.shape[0], -1)
             for n, m in model.named_children()}
    opt.step()
    torch.cuda.synchronize()
    errs = {}
    for n, m in model.named_children():
        if isinstance(m, nn.Conv2d):
            k, s, p = m.kernel_size[0], m.stride[0], m.padding[0]
            a_rows = O.im2col_rows(cap[n + ".in"], k, k, s, p)
            g_rows = O.conv_grad_rows(cap[n + ".g"], scale=b)
        else:
            a_rows = cap[n + ".in"].reshape(b, -1)
            g_rows = cap[n + ".g"] * b
        w_flat = w0[n].reshape(grads[n].shape)
        w_new, *_ = O.layer_kfac_update(w_flat, [a_rows], [g_rows], [grads[n]], gamma, lr)
        got = m.weight.detach().double().cpu().numpy().reshape(grads[n].shape)
        errs[n] = _rel(got - w_flat, w_new - w_flat)
    opt.remove_hooks()
    return errs


def token_linear_step(device="cuda:0", seed=0, gamma=0.1, lr=0.1, b=4, seq=24, h=48, f=96):
    """configs[4] path: linears on [batch, seq, features] token inputs (one small
    _LinearBlock); factor rows are the tokens (G rows scaled by the row count, the optimizer's
    linear-layer convention), each linear's update checked against the oracle."""
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.workloads import _LinearBlock
    torch.manual_seed(seed)
    model = _LinearBlock(h, f).to(device)
    lins = {n: m for n, m in model.named_modules() if isinstance(m, nn.Linear)}
    w0 = {n: m.weight.detach().double().cpu().numpy().copy() for n, m in lins.items()}
    cap = {}
    for n, m in lins.items():
        m.register_forward_pre_hook(lambda mod, inp, n=n: cap.__setitem__(n + ".in", inp[0].detach().double().cpu().numpy()))
        def post(mod, inp, out, n=n):  # returns None: the output is not replaced
            out.register_hook(lambda g: cap.__setitem__(n + ".g", g.detach().double().cpu().numpy()))
        m.register_forward_hook(post)
    opt = SPDKFAC(model, lr=lr, damping=gamma)
    x = torch.randn(b, seq, h, device=device)
    y = torch.randn(b, seq, h, device=device)
    nn.functional.mse_loss(model(x), y).backward()
    grads = {n: m.weight.grad.detach().double().cpu().numpy() for n, m in lins.items()}
    opt.step()
    torch.cuda.synchronize()
    errs = {}
    for n, m in lins.items():
        a_rows = cap[n + ".in"].reshape(-1, m.in_features)
        g_rows = cap[n + ".g"].reshape(-1, m.out_features) * a_rows.shape[0]
        w_new, *_ = O.layer_kfac_update(w0[n], [a_rows], [g_rows], [grads[n]], gamma, lr)
        got = m.weight.detach().double().cpu().numpy()
        errs[n] = _rel(got - w0[n], w_new - w0[n])
    opt.remove_hooks()
    return errs


def run_smoke():
    import faulthandler
    import os
    if os.environ.get("SPD_WATCHDOG"):
        faulthandler.dump_traceback_later(int(os.environ["SPD_WATCHDOG"]), exit=True)
    assert torch.cuda.is_available(), "smoke needs a CUDA device"
    from paper_2107_06533_b200 import _lib
    _lib.load(require_device=True)
    errs = fixture_step()
    print("golden fixture: per-layer relative update error", ["%.2e" % e for e in errs])
    assert max(errs) <= TOL, errs
    cerrs = conv_step()
    print("conv net: per-layer relative update error", {k: "%.2e" % v for k, v in cerrs.items()})
    assert max(cerrs.values()) <= TOL, cerrs
    cerrs = conv_step(channels_last=True)
    print("conv net (channels-last): per-layer relative update error", {k: "%.2e" % v for k, v in cerrs.items()})
    assert max(cerrs.values()) <= TOL, cerrs
    print("smoke OK")


if __name__ == "__main__":
    run_smoke()
