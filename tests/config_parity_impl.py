"""Config-level parity: one step of a BASELINE.json config, run exactly as bench.py times it
(bench.make_optimizer + GraphedStep: one CUDA graph per iteration, update_in_backward, SYRK
launch groups, early G inversion groups, d^3 LBP), checked layer by layer against the float64
oracle restating `dkfac_step` (/root/reference/pkg/src/kfacsched/emulator.py:234-263) on the
tensors the step itself consumed.

The tensors are captured INSIDE the graph (copy kernels recorded by forward / tensor hooks), so
the replayed step's own activations, output gradients and weight gradients are checked.  Per
layer l (conv layers restated as FC over im2col rows):

  stage 1  factor   A_l, G_l (the optimizer's packed buffers) vs factor_A/G(rows)      linalg.py:106-127
  stage 2  inverse  the optimizer's A_l^-1, G_l^-1 vs damped_inverse(GPU factor, gamma)  linalg.py:130-149
  stage 3  update   W1 - W0 vs -lr * precondition(grad, GPU A^-1, GPU G^-1)              linalg.py:152-167,
                                                                                         emulator.py:203-208
  end-to-end        W1 - W0 vs -lr * precondition(grad, damped_inverse(oracle factors))  emulator.py:234-263

Stage tolerances (north_star): 1e-4 relative Frobenius for factors and the update; the
kappa-scaled bound for inverses.  The end-to-end error compounds the factor error through the
inverse (a 1e-5 factor error becomes ~kappa * 1e-5 in A^-1), so it is reported per layer with
kappa and checked against that propagated bound.

TEST INFRASTRUCTURE ONLY (uses the oracle).
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch
import torch.nn as nn

import oracle as O

TOL = 1e-4


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _norm2(a, iters=50):
    v = np.random.default_rng(0).standard_normal(a.shape[0])
    for _ in range(iters):
        v = a @ v
        n = np.linalg.norm(v)
        if n == 0:
            return 0.0
        v /= n
    return float(v @ (a @ v))


class _Capture:
    """Copies each K-FAC layer's input and output gradient into persistent buffers.  The
    buffers are allocated during the eager warm-up steps; the copies are recorded into the
    CUDA graph and run on every replay."""

    def __init__(self, layers):
        self.a, self.g, self.handles = {}, {}, []
        for name, m in layers:
            self.handles.append(m.register_forward_pre_hook(self._pre(name)))
            self.handles.append(m.register_forward_hook(self._post(name)))

    @staticmethod
    def _into(store, name, t):
        t = t.detach()
        buf = store.get(name)
        if buf is None or buf.shape != t.shape:
            assert not torch.cuda.is_current_stream_capturing(), "capture buffers must exist before graph capture"
            buf = store[name] = torch.empty_like(t)
        buf.copy_(t)  # (autograd may hand over a gradient with other strides under capture: copy_ handles it)

    def _pre(self, name):
        def h(m, inp):
            if torch.is_grad_enabled() and m.training:
                self._into(self.a, name, inp[0])
        return h

    def _post(self, name):
        def h(m, inp, out):
            if torch.is_grad_enabled() and m.training and out.requires_grad:
                out.register_hook(lambda g: self._into(self.g, name, g))
        return h

    def remove(self):
        for h in self.handles:
            h.remove()


def _order_perm(m: nn.Module, w_cl: bool):
    """q[j_oracle] = j_gpu: the optimizer orders a channels-last conv's A rows (kh, kw, c); the
    oracle (and the logical weight reshape [cout, cin*kh*kw]) orders them (c, kh, kw)."""
    if not isinstance(m, nn.Conv2d) or not w_cl:
        return None
    c, (kh, kw) = m.in_channels, m.kernel_size
    return np.array([(ki * kw + kj) * c + ci for ci in range(c) for ki in range(kh) for kj in range(kw)])


def run_config(model_name: str, batch: int, device="cuda:0", seed: int = 0, warmup: int = 2, verbose=True):
    import bench
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.workloads import build_model, input_shape, num_classes

    a = bench.parse(["--model", model_name, "--batch", str(batch)])
    torch.manual_seed(seed)
    model = build_model(model_name).to(device).to(memory_format=torch.channels_last)
    opt = bench.make_optimizer(a, model, world=1)
    cap = _Capture([(l.name, l.module) for l in opt.layers])
    crit = nn.CrossEntropyLoss()
    g = torch.Generator(device=device).manual_seed(1000)
    shp = input_shape(model_name, batch)
    xs = [torch.randn(shp, device=device, generator=g).contiguous(memory_format=torch.channels_last) for _ in range(2)]
    ys = [torch.randint(0, num_classes(model_name), (batch,), device=device, generator=g) for _ in range(2)]
    gs = GraphedStep(model, crit, opt, [xs[0]], [ys[0]], warmup=warmup)
    gs([xs[1]], [ys[1]])  # one replay so the graph's pool holds settled buffers
    torch.cuda.synchronize()
    w0 = {l.name: l.module.weight.detach().clone() for l in opt.layers}
    gs([xs[0]], [ys[0]])  # the checked replay
    torch.cuda.synchronize()
    opt.check_inverses()
    gamma, lr = opt.damping, opt.param_groups[0]["lr"]

    report, t0 = [], time.perf_counter()
    for l in opt.layers:
        m = l.module
        q = _order_perm(m, l.w_cl)
        reorder = (lambda x: x[np.ix_(q, q)]) if q is not None else (lambda x: x)
        xin = cap.a[l.name].double().cpu().numpy()
        gout = cap.g[l.name].double().cpu().numpy()
        if isinstance(m, nn.Conv2d):
            kh, kw = m.kernel_size
            a_rows = O.im2col_rows(xin, kh, kw, tuple(m.stride), tuple(m.padding), tuple(m.dilation))
            g_rows = O.conv_grad_rows(gout, scale=batch)
        else:
            a_rows = xin.reshape(-1, m.in_features)
            g_rows = gout.reshape(-1, m.out_features) * a_rows.shape[0]
        fa_want = a_rows.T @ a_rows / a_rows.shape[0]
        fg_want = g_rows.T @ g_rows / g_rows.shape[0]
        del a_rows, g_rows
        fa_gpu = reorder(opt.factor(l.index, "A").double().cpu().numpy())
        fg_gpu = opt.factor(l.index, "G").double().cpu().numpy()
        ai_gpu = reorder(opt.inv[2 * l.index].double().cpu().numpy())
        gi_gpu = opt.inv[2 * l.index + 1].double().cpu().numpy()
        grad = m.weight.grad.detach().double().cpu().numpy().reshape(m.weight.shape[0], -1)
        delta = (m.weight.detach().double() - w0[l.name].double()).cpu().numpy().reshape(grad.shape)

        e_fa, e_fg = _rel(fa_gpu, fa_want), _rel(fg_gpu, fg_want)
        ai_want = O.damped_inverse(fa_gpu, gamma)   # stage 2 on the GPU's own factor
        gi_want = O.damped_inverse(fg_gpu, gamma)
        e_ai, e_gi = _rel(ai_gpu, ai_want), _rel(gi_gpu, gi_want)
        k_a = _norm2(fa_gpu + gamma * np.eye(fa_gpu.shape[0])) * _norm2(ai_want)
        k_g = _norm2(fg_gpu + gamma * np.eye(fg_gpu.shape[0])) * _norm2(gi_want)
        b_a = 16 * math.sqrt(fa_gpu.shape[0]) * k_a * 2.0 ** -24
        b_g = 16 * math.sqrt(fg_gpu.shape[0]) * k_g * 2.0 ** -24
        upd_want = -lr * O.precondition(grad, ai_gpu, gi_gpu)  # stage 3 on the GPU's own inverses
        e_up = _rel(delta, upd_want)
        e2e_want = -lr * O.precondition(grad, O.damped_inverse(fa_want, gamma), O.damped_inverse(fg_want, gamma))
        e_e2e = _rel(delta, e2e_want)
        # factor error propagated through the inverse (first order: kappa * relative perturbation)
        e2e_bound = max(TOL, 4.0 * (k_a * e_fa + k_g * e_fg + e_ai + e_gi) + e_up)
        report.append(dict(layer=l.name, a=fa_gpu.shape[0], g=fg_gpu.shape[0], factor_A=e_fa, factor_G=e_fg,
                           inv_A=e_ai, inv_G=e_gi, kappa_A=k_a, kappa_G=k_g, inv_bound_A=b_a, inv_bound_G=b_g,
                           update=e_up, e2e=e_e2e, e2e_bound=e2e_bound))
        if verbose:
            r = report[-1]
            print(f"{l.name:28s} a={r['a']:5d} g={r['g']:5d} fA={e_fa:.1e} fG={e_fg:.1e} iA={e_ai:.1e}"
                  f"(k={k_a:.1e}) iG={e_gi:.1e}(k={k_g:.1e}) upd={e_up:.1e} e2e={e_e2e:.1e}", flush=True)
    if verbose:
        print(f"oracle checks: {time.perf_counter() - t0:.1f} s for {len(report)} layers")
    cap.remove()
    opt.remove_hooks()
    return report


def check(report):
    bad = []
    for r in report:
        if r["factor_A"] > TOL or r["factor_G"] > TOL:
            bad.append((r["layer"], "factor", r["factor_A"], r["factor_G"]))
        if r["inv_A"] > r["inv_bound_A"] or r["inv_G"] > r["inv_bound_G"]:
            bad.append((r["layer"], "inverse", r["inv_A"], r["inv_bound_A"], r["inv_G"], r["inv_bound_G"]))
        if r["update"] > TOL:
            bad.append((r["layer"], "update", r["update"]))
        if r["e2e"] > r["e2e_bound"]:
            bad.append((r["layer"], "e2e", r["e2e"], r["e2e_bound"]))
    return bad


if __name__ == "__main__":
    import json
    import sys
    name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
    rep = run_config(name, 32)
    out = sys.argv[2] if len(sys.argv) > 2 else None
    if out:
        json.dump(rep, open(out, "w"), indent=1)
    print("violations:", check(rep))
