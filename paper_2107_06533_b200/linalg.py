"""Reference-facing operator API on CUDA tensors.

Mirrors the public functions of `kfacsched.linalg` (pkg/src/kfacsched/linalg.py)
-- same names, argument meaning and error behaviour -- with the arithmetic in
libspdkfac.so (include/spdkfac.h).  Inputs are torch tensors (any float dtype;
converted to contiguous float32 on the current CUDA device); outputs are
float32 CUDA tensors.  Symmetric results are returned as full d x d matrices
(the reference's `SymMatrix.values`); `pack_upper`/`unpack_upper` convert to and
from the reference's packed row-major upper layout.

The plan classes (`FactorPlan`, `InversePlan`, `PrecondPlan`) are what the
optimizer uses: they bind shapes once, own their device workspace and launch
on a given stream without host synchronisation.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import torch

from . import _lib as L


class NotPositiveDefiniteError(ValueError):
    """linalg.py:37-46: Cholesky hit a nonpositive pivot; `pivot` is 0-based."""

    def __init__(self, pivot: int):
        super().__init__(f"matrix is not positive definite (failing pivot index {pivot})")
        self.pivot = pivot


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _f32(t, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    if not t.is_cuda:
        t = t.cuda()
    return t.to(torch.float32).contiguous()


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ factors

class FactorPlan:
    """One Kronecker factor side of one layer (include/spdkfac.h factor plan)."""

    def __init__(self, layout: int, shape, kernel=(1, 1), stride=(1, 1), padding=(0, 0), dilation=(1, 1),
                 device=None, stream=None):
        lib = L.load(require_device=True)
        g = L.FactorGeom()
        g.layout = layout
        if layout == L.ROWS:
            g.n, g.c = int(shape[0]), int(shape[1])
            g.h, g.w = 1, int(shape[1])
        else:
            g.n, g.c, g.h, g.w = (int(v) for v in shape)
        g.kh, g.kw = (int(v) for v in kernel)
        g.stride_h, g.stride_w = (int(v) for v in stride)
        g.pad_h, g.pad_w = (int(v) for v in padding)
        g.dil_h, g.dil_w = (int(v) for v in dilation)
        rows, dim = C.c_int64(), C.c_int64()
        L.check(lib.spdkfac_factor_dims(C.byref(g), C.byref(rows), C.byref(dim)), "factor geometry")
        self.geom, self.rows, self.dim = g, rows.value, dim.value
        self.packed_size = self.dim * (self.dim + 1) // 2
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = _workspace(lib.spdkfac_factor_workspace_size(C.byref(g)), self.device)
        h = C.c_void_p()
        L.check(lib.spdkfac_factor_plan_create(C.byref(h), C.byref(g), self._ws.data_ptr(), self._ws.numel(),
                                               _stream(stream)), "factor plan")
        self._h = h
        self._lib = lib

    def run(self, x: torch.Tensor, packed: torch.Tensor, scale: float | None = None, decay: float = 0.0,
            world_scale: float = 1.0, stream=None) -> None:
        """packed <- world_scale*(decay*packed + (1-decay)*scale*X^T X); scale defaults to 1/rows."""
        fmt = torch.channels_last if self.geom.layout in (L.CONV_A_NHWC, L.SPATIAL_NHWC) else torch.contiguous_format
        if not (x.is_contiguous(memory_format=fmt) and x.dtype == torch.float32 and packed.dtype == torch.float32):
            raise ValueError("factor input must be float32 in the plan's memory format; packed float32")
        s = 1.0 / self.rows if scale is None else float(scale)
        L.check(self._lib.spdkfac_factor_plan_run(self._h, x.data_ptr(), s, float(decay), float(world_scale),
                                                  packed.data_ptr(), _stream(stream)), "factor run")

    def stage(self, x: torch.Tensor, stream=None) -> None:
        """First half of run(): consume x into the plan's split-precision staging buffer."""
        L.check(self._lib.spdkfac_factor_plan_stage(self._h, x.data_ptr(), _stream(stream)), "factor stage")

    def compute(self, packed: torch.Tensor, scale: float, decay: float = 0.0, world_scale: float = 1.0,
                stream=None) -> None:
        """Second half of run(): tensor-core SYRK from the staging buffer into `packed`."""
        L.check(self._lib.spdkfac_factor_plan_compute(self._h, float(scale), float(decay), float(world_scale),
                                                      packed.data_ptr(), _stream(stream)), "factor compute")

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.spdkfac_factor_plan_destroy(self._h)
            self._h = None


class FactorGroup:
    """Several factor sides staged one by one and computed by ONE tensor-core launch
    (include/spdkfac.h factor group).  `members`: list of (layout, shape, kernel, stride,
    padding, dilation); `packed`: per member, the fusion-buffer slice it writes; `scales`:
    per member, the factor normalisation (1/M, or b^2/M for output gradients).  A `packed` entry
    may also be a raw device address (int): a peer rank's inbox mapped through CUDA IPC
    (comm.PeerExchange), which the SYRK epilogue then writes over NVLink; `device` is then taken
    from the first tensor entry (or the current device)."""

    def __init__(self, members, packed, scales, stream=None):
        lib = L.load(require_device=True)
        n = len(members)
        geoms = (L.FactorGeom * n)()
        for k, (layout, shape, kernel, stride, padding, dilation) in enumerate(members):
            g = geoms[k]
            g.layout = layout
            if layout == L.ROWS:
                g.n, g.c, g.h, g.w = int(shape[0]), int(shape[1]), 1, int(shape[1])
            else:
                g.n, g.c, g.h, g.w = (int(v) for v in shape)
            g.kh, g.kw = (int(v) for v in kernel)
            g.stride_h, g.stride_w = (int(v) for v in stride)
            g.pad_h, g.pad_w = (int(v) for v in padding)
            g.dil_h, g.dil_w = (int(v) for v in dilation)
        self.n = n
        tensors = [p for p in packed if isinstance(p, torch.Tensor)]
        self.device = tensors[0].device if tensors else torch.device("cuda", torch.cuda.current_device())
        self._keep = tensors
        addrs = [int(p) if not isinstance(p, torch.Tensor) else p.data_ptr() for p in packed]
        self._ws = _workspace(lib.spdkfac_factor_group_workspace_size(n, geoms), self.device)
        sc = (C.c_float * n)(*[float(x) for x in scales])
        h = C.c_void_p()
        L.check(lib.spdkfac_factor_group_create(C.byref(h), n, geoms, L.ptr_array(addrs),
                                                sc, self._ws.data_ptr(), self._ws.numel(), _stream(stream)),
                "factor group")
        self._h, self._lib = h, lib

    def stage(self, member: int, x: torch.Tensor, stream=None) -> None:
        L.check(self._lib.spdkfac_factor_group_stage(self._h, int(member), x.data_ptr(), _stream(stream)),
                "factor group stage")

    def compute(self, decay: float = 0.0, world_scale: float = 1.0, stream=None) -> None:
        L.check(self._lib.spdkfac_factor_group_compute(self._h, float(decay), float(world_scale), _stream(stream)),
                "factor group compute")

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.spdkfac_factor_group_destroy(self._h)
            self._h = None


def _rows_batch(batch, what: str) -> torch.Tensor:
    x = _f32(batch, what)
    if x.dim() != 2:
        raise ValueError(f"{what}: expected a batch of equal-length vectors, got shape {tuple(x.shape)}")
    if x.shape[0] < 1:
        raise ValueError(f"{what}: empty batch")
    if x.shape[1] < 1:
        raise ValueError(f"{what}: vectors must have length >= 1")
    return x


def _factor_full(plan: FactorPlan, x: torch.Tensor, scale=None) -> torch.Tensor:
    packed = torch.empty(plan.packed_size, dtype=torch.float32, device=x.device)
    plan.run(x, packed, scale=scale)
    return unpack_upper(packed, plan.dim)


def compute_factor_A(activations) -> torch.Tensor:
    """linalg.py:116-122: (a^T a)/b over a [b, d_in] batch."""
    x = _rows_batch(activations, "compute_factor_A")
    return _factor_full(FactorPlan(L.ROWS, x.shape, device=x.device), x)


def compute_factor_G(output_grads) -> torch.Tensor:
    """linalg.py:125-127: (g^T g)/b over a [b, d_out] batch."""
    x = _rows_batch(output_grads, "compute_factor_G")
    return _factor_full(FactorPlan(L.ROWS, x.shape, device=x.device), x)


def _pair(v):
    return (v, v) if isinstance(v, int) else tuple(v)


def compute_factor_A_conv(x, kernel_size, stride=1, padding=0, dilation=1) -> torch.Tensor:
    """Conv restatement of compute_factor_A: rows = im2col patches (c, kh, kw
    order) of an NCHW input, divided by M = b*Hout*Wout."""
    x = _f32(x, "compute_factor_A_conv")
    if x.dim() != 4 or x.numel() == 0:
        raise ValueError(f"compute_factor_A_conv: expected a nonempty NCHW tensor, got {tuple(x.shape)}")
    plan = FactorPlan(L.CONV_A, x.shape, _pair(kernel_size), _pair(stride), _pair(padding), _pair(dilation),
                      device=x.device)
    return _factor_full(plan, x)


def compute_factor_G_spatial(g, row_scale: float = 1.0) -> torch.Tensor:
    """Conv restatement of compute_factor_G: rows = per-position output
    gradients of an NCHW tensor times `row_scale` (the batch size, undoing a
    batch-mean loss), divided by M = b*H*W."""
    g = _f32(g, "compute_factor_G_spatial")
    if g.dim() != 4 or g.numel() == 0:
        raise ValueError(f"compute_factor_G_spatial: expected a nonempty NCHW tensor, got {tuple(g.shape)}")
    plan = FactorPlan(L.SPATIAL, g.shape, device=g.device)
    return _factor_full(plan, g, scale=row_scale * row_scale / plan.rows)


# ------------------------------------------------------------------ packing

def pack_upper(m) -> torch.Tensor:
    """linalg.py:181-184."""
    m = _f32(m, "pack_upper")
    if m.dim() != 2 or m.shape[0] != m.shape[1] or m.shape[0] < 1:
        raise ValueError(f"expected a square matrix, got shape {tuple(m.shape)}")
    d = m.shape[0]
    out = torch.empty(d * (d + 1) // 2, dtype=torch.float32, device=m.device)
    L.check(L.load(True).spdkfac_pack_upper_f32(m.data_ptr(), d, d, out.data_ptr(), _stream()), "pack_upper")
    return out


def unpack_upper(arr, d: int) -> torch.Tensor:
    """linalg.py:187-199."""
    if d < 1:
        raise ValueError("dimension must be >= 1")
    a = _f32(arr, "unpack_upper")
    if a.dim() != 1 or a.numel() != d * (d + 1) // 2:
        raise ValueError(f"packed length {a.numel()} does not match dim {d} (expected {d * (d + 1) // 2})")
    out = torch.empty(d, d, dtype=torch.float32, device=a.device)
    L.check(L.load(True).spdkfac_unpack_upper_f32(a.data_ptr(), d, out.data_ptr(), d, _stream()), "unpack_upper")
    return out


# ------------------------------------------------------------------ inverse

class InversePlan:
    """Batched damped inverse bound to fixed packed inputs and full outputs."""

    def __init__(self, packed_in: Sequence[torch.Tensor], out_full: Sequence[torch.Tensor], stream=None):
        lib = L.load(require_device=True)
        self.n = len(packed_in)
        if self.n < 1 or len(out_full) != self.n:
            raise ValueError("need matching nonempty input/output lists")
        self.dims = [int(o.shape[0]) for o in out_full]
        for p, o, d in zip(packed_in, out_full, self.dims):
            if p.numel() != d * (d + 1) // 2 or tuple(o.shape) != (d, d) or not o.is_contiguous():
                raise ValueError("packed input / full output shape mismatch")
        self.device = out_full[0].device
        self._keep = (list(packed_in), list(out_full))
        self.info = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        dims = L.i32_array(self.dims)
        self._ws = _workspace(lib.spdkfac_inverse_workspace_size(self.n, dims), self.device)
        h = C.c_void_p()
        L.check(lib.spdkfac_inverse_plan_create(
            C.byref(h), self.n, dims, L.ptr_array([p.data_ptr() for p in packed_in]),
            L.ptr_array([o.data_ptr() for o in out_full]), self.info.data_ptr(), self._ws.data_ptr(),
            self._ws.numel(), _stream(stream)), "inverse plan")
        self._h = h
        self._lib = lib

    def run(self, gamma: float, stream=None) -> None:
        if gamma < 0:
            raise ValueError(f"damping must be nonnegative, got {gamma}")
        L.check(self._lib.spdkfac_inverse_plan_run(self._h, float(gamma), _stream(stream)), "inverse run")

    def check(self) -> None:
        """Host-synchronising read of the per-matrix pivots (raises like linalg.py:141-145)."""
        info = self.info.cpu()
        bad = torch.nonzero(info).flatten()
        if bad.numel():
            raise NotPositiveDefiniteError(int(info[bad[0]]) - 1)

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.spdkfac_inverse_plan_destroy(self._h)
            self._h = None


def damped_inverse_batched(mats: Sequence[torch.Tensor], gamma: float) -> list:
    """damped_inverse over a batch of symmetric matrices in one plan."""
    if gamma < 0:
        raise ValueError(f"damping must be nonnegative, got {gamma}")
    packed = [pack_upper(m) for m in mats]
    outs = [torch.empty(m.shape[0], m.shape[0], dtype=torch.float32, device=packed[0].device) for m in mats]
    plan = InversePlan(packed, outs)
    plan.run(gamma)
    plan.check()
    return outs


def damped_inverse(m, gamma: float) -> torch.Tensor:
    """linalg.py:130-149: (m + gamma I)^-1, symmetrised; raises
    NotPositiveDefiniteError(pivot) / ValueError(gamma < 0)."""
    if gamma < 0:
        raise ValueError(f"damping must be nonnegative, got {gamma}")
    m = _f32(m, "damped_inverse")
    if m.dim() != 2 or m.shape[0] != m.shape[1] or m.shape[0] < 1:
        raise ValueError(f"expected a square matrix, got shape {tuple(m.shape)}")
    return damped_inverse_batched([m], gamma)[0]


# ------------------------------------------------------------------ precondition

class PrecondPlan:
    """Batched P_l = G_l^-1 grad_l A_l^-1 (+ W_l -= alpha P_l) over fixed layer shapes."""

    def __init__(self, shapes: Sequence[tuple], device=None, stream=None):
        lib = L.load(require_device=True)
        self.shapes = [(int(o), int(i)) for o, i in shapes]
        self.n = len(self.shapes)
        if self.n < 1:
            raise ValueError("no layers to precondition")
        dout = L.i32_array([s[0] for s in self.shapes])
        din = L.i32_array([s[1] for s in self.shapes])
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = _workspace(lib.spdkfac_precond_workspace_size(self.n, dout, din), self.device)
        h = C.c_void_p()
        L.check(lib.spdkfac_precond_plan_create(C.byref(h), self.n, dout, din, self._ws.data_ptr(), self._ws.numel(),
                                                _stream(stream)), "precondition plan")
        self._h = h
        self._lib = lib

    def bind(self, g_inv, grads, a_inv, weights=None, out=None):
        """Pre-build the pointer tables for tensors whose storage stays fixed across steps."""
        self._bound = (L.ptr_array([t.data_ptr() for t in g_inv]), L.ptr_array([t.data_ptr() for t in grads]),
                       L.ptr_array([t.data_ptr() for t in a_inv]),
                       L.ptr_array([w.data_ptr() for w in weights]) if weights is not None else None,
                       L.ptr_array([o.data_ptr() for o in out]) if out is not None else None)
        self._bound_key = tuple(t.data_ptr() for t in grads)

    def run_bound(self, alpha: float, stream=None, inverses_staged: bool = False) -> None:
        """inverses_staged: every layer's inverses were already staged (stage_inverses) since
        they last changed, so only the gradients are split here."""
        gi, gr, ai, pw, po = self._bound
        if inverses_staged:
            gi = ai = None
        L.check(self._lib.spdkfac_precond_plan_run(self._h, gi, gr, ai, pw, float(alpha), po, _stream(stream)),
                "precondition run")

    def stage_inverses(self, which: str, layers: Sequence[int], inverses: Sequence[torch.Tensor], stream=None) -> None:
        """Split the given layers' inverses (which = "A" or "G") into the plan's bf16 hi/lo
        operands, on `stream` (e.g. right after the stream that inverted them)."""
        if not layers:
            return
        L.check(self._lib.spdkfac_precond_plan_stage_inverses(
            self._h, 0 if which == "A" else 1, len(layers), L.i32_array(layers),
            L.ptr_array([t.data_ptr() for t in inverses]), _stream(stream)), "stage inverses")

    def run(self, g_inv, grads, a_inv, weights=None, alpha: float = 0.0, out=None, stream=None) -> None:
        n = self.n
        assert len(g_inv) == n and len(grads) == n and len(a_inv) == n
        pw = L.ptr_array([w.data_ptr() for w in weights]) if weights is not None else None
        po = L.ptr_array([o.data_ptr() for o in out]) if out is not None else None
        L.check(self._lib.spdkfac_precond_plan_run(
            self._h, L.ptr_array([t.data_ptr() for t in g_inv]), L.ptr_array([t.data_ptr() for t in grads]),
            L.ptr_array([t.data_ptr() for t in a_inv]), pw, float(alpha), po, _stream(stream)), "precondition run")

    def stage_packed(self, which: str, layers: Sequence[int], packed: Sequence[torch.Tensor],
                     full_out: Sequence[torch.Tensor] | None = None, stream=None) -> None:
        """Packed upper inverses (a broadcast) -> operand planes and, optionally, full matrices."""
        if not layers:
            return
        L.check(self._lib.spdkfac_precond_plan_stage_packed(
            self._h, 0 if which == "A" else 1, len(layers), L.i32_array(layers),
            L.ptr_array([t.data_ptr() for t in packed]),
            L.ptr_array([t.data_ptr() for t in full_out]) if full_out is not None else None,
            _stream(stream)), "stage packed inverses")

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.spdkfac_precond_plan_destroy(self._h)
            self._h = None


def precondition(grad, a_inv, g_inv) -> torch.Tensor:
    """linalg.py:152-167: g_inv @ grad @ a_inv."""
    g = _f32(grad, "precondition")
    if g.dim() != 2:
        raise ValueError(f"gradient must be 2-D, got shape {tuple(g.shape)}")
    a = _f32(a_inv, "precondition")
    gi = _f32(g_inv, "precondition")
    d_out, d_in = g.shape
    if a.shape != (d_in, d_in) or gi.shape != (d_out, d_out):
        raise ValueError(f"shape mismatch: grad {d_out}x{d_in} needs A-side dim {d_in} (got {a.shape[0]}) "
                         f"and G-side dim {d_out} (got {gi.shape[0]})")
    out = torch.empty_like(g)
    PrecondPlan([(d_out, d_in)], device=g.device).run([gi], [g], [a], out=[out])
    return out
