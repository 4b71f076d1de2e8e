"""Timed CPU reference of the SPD-KFAC step's linear algebra (TEST / BASELINE
INFRASTRUCTURE ONLY: used by bench.py's `cpu_baseline` leg and `--impl reference`).

Per layer l of the workload (shapes from paper_2107_06533_b200.workloads), exactly
the reference's float64 arithmetic (restated in oracle/linalg.py):
  compute_factor_A(rows[M, a]), compute_factor_G(rows[M, g])   linalg.py:116-127
  damped_inverse(A, gamma), damped_inverse(G, gamma)           linalg.py:130-149
  precondition(grad, A^-1, G^-1); W -= alpha * step            linalg.py:152-167, emulator.py:203-208
on synthetic rows of the layer's true (M, a, g), for every layer of the model in
each timed step (inputs generated once per distinct shape, outside the timing); the
reference has no conv layers, so the rows are fed as if already im2col'd (im2col
cost not charged to the reference).
"""

from __future__ import annotations

import os
import time
from collections import Counter

import numpy as np

from .linalg import damped_inverse, factor_A, factor_G, precondition

_REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def implementation():
    """The reference's own functions when its unmodified package is installed under
    baseline/_ref (pip install --no-deps --target baseline/_ref <reference pkg>), else the
    oracle port.  Returns (factor_A, factor_G, damped_inverse, precondition, kind)."""
    import sys
    if os.path.isdir(os.path.join(_REF_DIR, "kfacsched")):
        if _REF_DIR not in sys.path:
            sys.path.insert(0, _REF_DIR)
        try:
            import kfacsched as K
            return K.compute_factor_A, K.compute_factor_G, K.damped_inverse, K.precondition, "reference"
        except Exception:  # pragma: no cover - broken install: fall back to the port
            pass
    return factor_A, factor_G, damped_inverse, precondition, "port"


def distinct_shapes(shapes):
    """[(M, a, g)] -> Counter of multiplicities, in first-seen order."""
    return Counter((m, a, g) for _, m, a, g in shapes)


def layer_inputs(m: int, a: int, g: int, seed: int = 0):
    """Synthetic float64 inputs of one layer: A rows [m, a], G rows [m, g], gradient and weight [g, a]."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((m, a)), rng.standard_normal((m, g)), rng.standard_normal((g, a)), \
        rng.standard_normal((g, a))


def time_layer(m: int, a: int, g: int, gamma: float = 0.1, alpha: float = 0.1, seed: int = 0, inputs=None) -> float:
    """Seconds of the reference's per-layer step arithmetic on (m, a, g): factors, both damped
    inverses, preconditioning and the update (input generation is not timed)."""
    fa, fg, dinv, pre, _ = implementation()
    rows_a, rows_g, grad, w = inputs if inputs is not None else layer_inputs(m, a, g, seed)
    t0 = time.perf_counter()
    A = fa(rows_a)
    G = fg(rows_g)
    ai = dinv(A, gamma)
    gi = dinv(G, gamma)
    w -= alpha * pre(grad, ai, gi)
    return time.perf_counter() - t0


def threads() -> int:
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        if os.environ.get(k):
            return int(os.environ[k])
    return os.cpu_count() or 1


def full_step(shapes, cache=None) -> float:
    """One measured step of the whole workload: the reference's per-layer arithmetic for EVERY layer
    (all 54 of ResNet-50), so the step's time is the wall time actually spent.  `cache` keeps each
    distinct shape's synthetic inputs across layers and steps (generating them costs more than some
    layers); input generation is not timed."""
    cache = {} if cache is None else cache
    total = 0.0
    for _, m, a, g in shapes:
        k = (m, a, g)
        if k not in cache:
            cache[k] = layer_inputs(*k)
        total += time_layer(*k, inputs=cache[k])
    return total


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"
