"""float64 restatement of the step in `kfacsched.emulator` (TEST INFRASTRUCTURE ONLY).

Weights are lists of [d_out, d_in] arrays, activations a list of
"relu"/"identity" (the reference's bias-free `TinyMLP`, emulator.py:46-89);
a worker batch is an (inputs [b, d0], targets [b, dL]) pair
(`WorkerBatch`, emulator.py:92-119).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .linalg import damped_inverse, factor_A, factor_G, precondition


def _act(z, kind):
    return z if kind == "identity" else np.maximum(z, 0.0)


def _dact(z, kind):
    return np.ones_like(z) if kind == "identity" else (z > 0.0).astype(np.float64)


def mlp_forward_backward(weights, acts, inputs, targets):
    """`forward_backward` (emulator.py:157-196).

    Returns (loss, layer_inputs, output_grads, weight_grads): output_grads are
    per-sample dLoss/dz without 1/b (MSE averaged over output dims, so the
    output gradient is 2(y-t)/d_out, emulator.py:177-179); weight grads are
    the batch-mean gradient g^T a / b (emulator.py:187).
    """
    x = np.asarray(inputs, dtype=np.float64)
    t = np.asarray(targets, dtype=np.float64)
    b = x.shape[0]
    ins, pre = [], []
    a = x
    for w, k in zip(weights, acts):
        ins.append(a)
        z = a @ np.asarray(w).T
        pre.append(z)
        a = _act(z, k)
    diff = a - t
    loss = float(np.mean(diff * diff))
    up = 2.0 * diff / a.shape[1]
    n = len(weights)
    gs, dws = [None] * n, [None] * n
    for l in reversed(range(n)):
        g = up * _dact(pre[l], acts[l])
        gs[l] = g
        dws[l] = (g.T @ ins[l]) / b
        if l:
            up = g @ np.asarray(weights[l])
    return loss, ins, gs, dws


def dkfac_step(weights, acts, worker_batches, gamma, alpha, owner_walk=None):
    """`dkfac_step` (emulator.py:211-263): per-worker factors, mean over
    workers (`_mean_sym`, emulator.py:199-200), one damped inverse per
    tensor, preconditioned update (`_apply_update`, emulator.py:203-208).

    `owner_walk` optionally restates the placement routing of
    emulator.py:256-262 (a list of per-worker tensor-index lists; the first
    holder computes); it never changes the numbers.
    """
    if not worker_batches:
        raise ValueError("need at least one worker batch")
    if len({np.asarray(x).shape[0] for x, _ in worker_batches}) != 1:
        raise ValueError("per-worker batch sizes must be equal")
    res = [mlp_forward_backward(weights, acts, x, t) for x, t in worker_batches]
    n = len(weights)
    facs, grads = {}, []
    for l in range(n):
        facs[("A", l)] = np.mean([factor_A(r[1][l]) for r in res], axis=0)
        facs[("G", l)] = np.mean([factor_G(r[2][l]) for r in res], axis=0)
        grads.append(np.mean([r[3][l] for r in res], axis=0))
    order = [(k, l) for l in range(n) for k in ("A", "G")]  # emulator.py:243-245
    inv = {}
    if owner_walk is None:
        for key in order:
            inv[key] = damped_inverse(facs[key], gamma)
    else:
        if sum(1 for _ in {i for w in owner_walk for i in w}) != len(order):
            raise ValueError("placement does not cover every tensor")
        for assigned in owner_walk:
            for idx in assigned:
                if order[idx] not in inv:
                    inv[order[idx]] = damped_inverse(facs[order[idx]], gamma)
    return [np.asarray(weights[l]) - alpha * precondition(grads[l], inv[("A", l)], inv[("G", l)]) for l in range(n)]


def kfac_step_centralized(weights, acts, inputs, targets, gamma, alpha):
    """`kfac_step_centralized` (emulator.py:266-275): the union-batch oracle."""
    _, ins, gs, dws = mlp_forward_backward(weights, acts, inputs, targets)
    out = []
    for l in range(len(weights)):
        a_inv = damped_inverse(factor_A(ins[l]), gamma)
        g_inv = damped_inverse(factor_G(gs[l]), gamma)
        out.append(np.asarray(weights[l]) - alpha * precondition(dws[l], a_inv, g_inv))
    return out


def run_fixture(fx: dict, owner_walk=None) -> float:
    """`run_fixture` (emulator.py:328-343): max |deviation| from the frozen
    centralized-oracle weights."""
    batches = list(zip(fx["worker_inputs"], fx["worker_targets"]))
    got = dkfac_step([np.array(w) for w in fx["weights"]], fx["activations"], batches,
                     fx["gamma"], fx["alpha"], owner_walk)
    return max(float(np.abs(g - np.array(e)).max()) for g, e in zip(got, fx["expected_weights"]))


def layer_kfac_update(weight, rank_a_rows: Sequence, rank_g_rows: Sequence, rank_grads: Sequence,
                      gamma: float, alpha: float, running=None, decay: float = 0.0):
    """One preconditioned layer update from captured per-rank tensors -- the
    rule of `dkfac_step` (emulator.py:234-263) applied to one layer:

      A = mean_r factor_A(a_rows_r), G = mean_r factor_G(g_rows_r),
      grad = mean_r grad_r, W' = W - alpha * G^-1 grad A^-1  (damped).

    `running=(A_old, G_old)` with `decay` restates the north-star running
    average A <- decay*A_old + (1-decay)*A (unpinned by the reference, which
    has no running average; decay=0 reduces to the reference).
    Returns (W', A, G, A^-1, G^-1, preconditioned grad).
    """
    A = np.mean([factor_A(r) for r in rank_a_rows], axis=0)
    G = np.mean([factor_G(r) for r in rank_g_rows], axis=0)
    if running is not None:
        A = decay * running[0] + (1.0 - decay) * A
        G = decay * running[1] + (1.0 - decay) * G
    grad = np.mean([np.asarray(g, dtype=np.float64) for g in rank_grads], axis=0)
    a_inv = damped_inverse(A, gamma)
    g_inv = damped_inverse(G, gamma)
    step = precondition(grad, a_inv, g_inv)
    return np.asarray(weight, dtype=np.float64) - alpha * step, A, G, a_inv, g_inv, step
