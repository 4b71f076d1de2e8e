"""The reference-side binding of INTEGRATION.md section 3, as a module: what a kfacsched maintainer
adds (e.g. as `kfacsched/_b200.py`) to route `kfacsched.linalg`'s arithmetic through the C ABI of
libspdkfac.so (include/spdkfac.h).  Raw ctypes on the C ABI -- no paper_2107_06533_b200 Python --
with torch only for device memory and the stream.

Each function keeps the reference's signature, return type (SymMatrix / ndarray) and errors:
  compute_factor_A / compute_factor_G   linalg.py:106-127
  damped_inverse                        linalg.py:130-149 (NotPositiveDefiniteError(pivot))
  precondition                          linalg.py:152-167

`install()` monkeypatches them into `kfacsched.linalg` and the `kfacsched` package namespace;
tests/kfacsched_b200_plugin.py does that before the reference's own tests import them.

TEST INFRASTRUCTURE (the drop-in exercise of tests/test_gpu_reference_dropin.py).
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np
import torch

_LIB_PATH = os.environ.get("SPDKFAC_LIB",
                           str(pathlib.Path(__file__).resolve().parents[1] / "paper_2107_06533_b200" / "lib" /
                               "libspdkfac.so"))
_lib = C.CDLL(_LIB_PATH)
_lib.spdkfac_last_error.restype = C.c_char_p
_lib.spdkfac_factor_workspace_size.restype = C.c_size_t
_lib.spdkfac_inverse_workspace_size.restype = C.c_size_t
_lib.spdkfac_precond_workspace_size.restype = C.c_size_t


class _Geom(C.Structure):  # spdkfac_factor_geom
    _fields_ = [("layout", C.c_int32), ("n", C.c_int64), ("c", C.c_int64), ("h", C.c_int64), ("w", C.c_int64),
                ("kh", C.c_int32), ("kw", C.c_int32), ("stride_h", C.c_int32), ("stride_w", C.c_int32),
                ("pad_h", C.c_int32), ("pad_w", C.c_int32), ("dil_h", C.c_int32), ("dil_w", C.c_int32)]


def _check(rc, pivot=None):
    if rc == 0:
        return
    msg = _lib.spdkfac_last_error().decode()
    if rc == 1:  # SPDKFAC_ERR_NOT_PD
        from kfacsched.linalg import NotPositiveDefiniteError
        raise NotPositiveDefiniteError(pivot)
    if rc in (2, 3):  # SHAPE / ARG
        raise ValueError(msg)
    raise RuntimeError(msg)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _factor(batch, what):
    from kfacsched.linalg import unpack_upper
    try:
        x = np.asarray(batch, dtype=np.float64)
    except ValueError as e:  # ragged rows (linalg.py:108-112)
        raise ValueError(f"{what}: expected a batch of equal-length vectors") from e
    if x.ndim != 2:
        raise ValueError(f"{what}: expected a batch of equal-length vectors")
    if x.shape[0] < 1:
        raise ValueError(f"{what}: empty batch")
    b, d = x.shape
    xt = torch.tensor(x, dtype=torch.float32, device="cuda").contiguous()
    g = _Geom(layout=0, n=b, c=d, h=1, w=d)
    ws = torch.empty(max(int(_lib.spdkfac_factor_workspace_size(C.byref(g))), 256), dtype=torch.uint8, device="cuda")
    plan = C.c_void_p()
    s = _stream()
    _check(_lib.spdkfac_factor_plan_create(C.byref(plan), C.byref(g), C.c_void_p(ws.data_ptr()),
                                           C.c_size_t(ws.numel()), s))
    packed = torch.empty(d * (d + 1) // 2, device="cuda")
    try:
        _check(_lib.spdkfac_factor_plan_run(plan, C.c_void_p(xt.data_ptr()), C.c_float(1.0 / b), C.c_float(0.0),
                                            C.c_float(1.0), C.c_void_p(packed.data_ptr()), s))
    finally:
        _lib.spdkfac_factor_plan_destroy(plan)
    return unpack_upper(packed.double().cpu().numpy(), d)  # SymMatrix, as the reference returns


def compute_factor_A(activations):
    """Drop-in for linalg.compute_factor_A (linalg.py:116-122): SymMatrix((x^T x) / b)."""
    return _factor(activations, "compute_factor_A")


def compute_factor_G(output_grads):
    """Drop-in for linalg.compute_factor_G (linalg.py:125-127)."""
    return _factor(output_grads, "compute_factor_G")


def damped_inverse(m, gamma):
    """Drop-in for linalg.damped_inverse (linalg.py:130-149)."""
    from kfacsched.linalg import SymMatrix, pack_upper
    if gamma < 0:
        raise ValueError(f"damping must be nonnegative, got {gamma}")
    if not isinstance(m, SymMatrix):
        m = SymMatrix(m)
    d = m.dim
    packed = torch.tensor(pack_upper(m), dtype=torch.float32, device="cuda")
    out = torch.empty(d, d, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    dims = (C.c_int32 * 1)(d)
    ws = torch.empty(max(int(_lib.spdkfac_inverse_workspace_size(1, dims)), 256), dtype=torch.uint8, device="cuda")
    plan = C.c_void_p()
    s = _stream()
    _check(_lib.spdkfac_inverse_plan_create(C.byref(plan), 1, dims, (C.c_void_p * 1)(packed.data_ptr()),
                                            (C.c_void_p * 1)(out.data_ptr()), C.c_void_p(info.data_ptr()),
                                            C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()), s))
    try:
        _check(_lib.spdkfac_inverse_plan_run(plan, C.c_float(gamma), s))
    finally:
        torch.cuda.synchronize()
        _lib.spdkfac_inverse_plan_destroy(plan)
    if int(info.item()):
        _check(1, pivot=int(info.item()) - 1)
    x = out.double().cpu().numpy()
    return SymMatrix((x + x.T) / 2)


def precondition(grad, a_inv, g_inv):
    """Drop-in for linalg.precondition (linalg.py:152-167): G^-1 . grad . A^-1."""
    from kfacsched.linalg import SymMatrix
    g = np.asarray(grad, dtype=np.float64)
    if g.ndim != 2:
        raise ValueError(f"gradient must be 2-D, got shape {g.shape}")
    a = a_inv.values if isinstance(a_inv, SymMatrix) else np.asarray(a_inv, dtype=np.float64)
    gi = g_inv.values if isinstance(g_inv, SymMatrix) else np.asarray(g_inv, dtype=np.float64)
    d_out, d_in = g.shape
    if a.shape != (d_in, d_in) or gi.shape != (d_out, d_out):
        raise ValueError(f"shape mismatch: grad {d_out}x{d_in} needs A-side dim {d_in} (got {a.shape[0]}) "
                         f"and G-side dim {d_out} (got {gi.shape[0]})")
    dev = lambda v: torch.tensor(v, dtype=torch.float32, device="cuda").contiguous()  # noqa: E731
    gt, at, git = dev(g), dev(a), dev(gi)
    out = torch.empty(d_out, d_in, device="cuda")
    do, di = (C.c_int32 * 1)(d_out), (C.c_int32 * 1)(d_in)
    ws = torch.empty(max(int(_lib.spdkfac_precond_workspace_size(1, do, di)), 256), dtype=torch.uint8, device="cuda")
    plan = C.c_void_p()
    s = _stream()
    _check(_lib.spdkfac_precond_plan_create(C.byref(plan), 1, do, di, C.c_void_p(ws.data_ptr()),
                                            C.c_size_t(ws.numel()), s))
    ptr = lambda t: (C.c_void_p * 1)(t.data_ptr())  # noqa: E731
    try:
        _check(_lib.spdkfac_precond_plan_run(plan, ptr(git), ptr(gt), ptr(at), None, C.c_float(0.0), ptr(out), s))
    finally:
        torch.cuda.synchronize()
        _lib.spdkfac_precond_plan_destroy(plan)
    return out.double().cpu().numpy()


def install():
    """Route kfacsched's linear algebra through libspdkfac (module and package namespace)."""
    import kfacsched
    import kfacsched.linalg as KL
    for name in ("compute_factor_A", "compute_factor_G", "damped_inverse", "precondition"):
        setattr(KL, name, globals()[name])
        if hasattr(kfacsched, name):
            setattr(kfacsched, name, globals()[name])
