"""float64 restatement of `kfacsched.linalg` (TEST INFRASTRUCTURE ONLY).

Every function takes and returns plain numpy arrays (the reference wraps
them in an immutable `SymMatrix`, linalg.py:49-103; the wrapper's only
arithmetic is the exact symmetrisation `(a + a.T) / 2` of linalg.py:66-72,
which `_sym` restates).
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import lapack, solve_triangular

_ASYM_TOL = 1e-12  # linalg.py:34 (_SYMMETRY_ATOL)


class NotPositiveDefinite(ValueError):
    """Restates `NotPositiveDefiniteError` (linalg.py:37-46): 0-based pivot."""

    def __init__(self, pivot: int):
        super().__init__(f"matrix is not positive definite (failing pivot index {pivot})")
        self.pivot = pivot


def _sym(a: np.ndarray) -> np.ndarray:
    """SymMatrix construction (linalg.py:60-72): reject asymmetry above
    1e-12*max(1, |a|_max), then average with the transpose."""
    a = np.array(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {a.shape}")
    if a.shape[0] < 1:
        raise ValueError("dimension must be >= 1")
    tol = _ASYM_TOL * max(1.0, float(np.abs(a).max()))
    if float(np.abs(a - a.T).max()) > tol:
        raise ValueError("matrix is not symmetric")
    return (a + a.T) / 2.0


def factor(rows, what: str = "factor") -> np.ndarray:
    """`_factor_from_batch` (linalg.py:106-113): (x^T x) / b over a [b, d]
    batch of row vectors; empty and ragged batches raise ValueError."""
    x = np.asarray(rows, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError(f"{what}: expected a batch of equal-length vectors, got shape {x.shape}")
    if x.shape[0] < 1:
        raise ValueError(f"{what}: empty batch")
    return _sym((x.T @ x) / x.shape[0])


def factor_A(activations) -> np.ndarray:
    """`compute_factor_A` (linalg.py:116-122)."""
    return factor(activations, "compute_factor_A")


def factor_G(output_grads) -> np.ndarray:
    """`compute_factor_G` (linalg.py:125-127)."""
    return factor(output_grads, "compute_factor_G")


def damped_inverse(m, gamma: float) -> np.ndarray:
    """`damped_inverse` (linalg.py:130-149): Cholesky of m + gamma*I
    (LAPACK dpotrf, lower), two triangular solves against I, symmetrise."""
    if gamma < 0:
        raise ValueError(f"damping must be nonnegative, got {gamma}")
    m = np.asarray(m, dtype=np.float64)
    d = m.shape[0]
    c, info = lapack.dpotrf(m + gamma * np.eye(d), lower=1)
    if info > 0:
        raise NotPositiveDefinite(info - 1)
    if info < 0:
        raise ValueError(f"illegal value in Cholesky argument {-info}")
    y = solve_triangular(c, np.eye(d), lower=True)
    x = solve_triangular(c.T, y, lower=False)
    return _sym((x + x.T) / 2.0)


def precondition(grad, a_inv, g_inv) -> np.ndarray:
    """`precondition` (linalg.py:152-167): G^-1 . grad . A^-1."""
    g = np.asarray(grad, dtype=np.float64)
    if g.ndim != 2:
        raise ValueError(f"gradient must be 2-D, got shape {g.shape}")
    a_inv = np.asarray(a_inv, dtype=np.float64)
    g_inv = np.asarray(g_inv, dtype=np.float64)
    if a_inv.shape[0] != g.shape[1] or g_inv.shape[0] != g.shape[0]:
        raise ValueError("shape mismatch")
    return g_inv @ g @ a_inv


def kron_vec_precondition(grad, a_inv, g_inv) -> np.ndarray:
    """Independent oracle used by the reference test (test_linalg.py:159-170):
    unvec of (A^-1 kron G^-1) vec_F(grad), column-major vec."""
    grad = np.asarray(grad, dtype=np.float64)
    big = np.kron(np.asarray(a_inv), np.asarray(g_inv))
    return (big @ grad.flatten(order="F")).reshape(grad.shape, order="F")


def pack_upper(m) -> np.ndarray:
    """`pack_upper` (linalg.py:181-184): row-major upper triangle incl. the
    diagonal, d(d+1)/2 entries; element (i<=j) sits at i*(2d-i+1)/2 + j-i."""
    m = np.asarray(m, dtype=np.float64)
    r, c = np.triu_indices(m.shape[0])
    return np.ascontiguousarray(m[r, c])


def unpack_upper(arr, d: int) -> np.ndarray:
    """`unpack_upper` (linalg.py:187-199)."""
    flat = np.asarray(arr, dtype=np.float64)
    if d < 1:
        raise ValueError("dimension must be >= 1")
    if flat.ndim != 1 or flat.size != d * (d + 1) // 2:
        raise ValueError(f"packed length {flat.size} does not match dim {d}")
    out = np.zeros((d, d))
    r, c = np.triu_indices(d)
    out[r, c] = flat
    out[c, r] = flat
    return _sym(out)


# --- conv restatement: the reference has FC semantics only
# (SPEC.md:111).  Conv layers are restated as FC layers over im2col rows, the
# Grosse-Martens KFC convention: A rows = input patches (c, kh, kw order, the
# order of torch's conv weight reshape [cout, cin*kh*kw]); G rows = per-position
# output gradients.  Each row set is fed to `factor` exactly as linalg.py:113
# divides by the row count M = b*Hout*Wout.  This normalisation is unpinned by
# the reference and stated in DESIGN.md.


def im2col_rows(x, kh: int, kw: int, stride=1, pad=0, dil=1) -> np.ndarray:
    """[B, C, H, W] -> [B*Ho*Wo, C*kh*kw] patch rows (zero padding); stride / pad / dil are ints
    or (h, w) pairs (Inception's 1x7 / 7x1 kernels pad one axis only)."""
    x = np.asarray(x, dtype=np.float64)
    b, c, h, w = x.shape
    sh, sw = (stride, stride) if np.isscalar(stride) else stride
    ph, pw = (pad, pad) if np.isscalar(pad) else pad
    dh, dw = (dil, dil) if np.isscalar(dil) else dil
    ho = (h + 2 * ph - dh * (kh - 1) - 1) // sh + 1
    wo = (w + 2 * pw - dw * (kw - 1) - 1) // sw + 1
    xp = np.zeros((b, c, h + 2 * ph, w + 2 * pw))
    xp[:, :, ph:ph + h, pw:pw + w] = x
    cols = np.empty((b, c, kh, kw, ho, wo))
    for i in range(kh):
        for j in range(kw):
            hs, ws = i * dh, j * dw
            cols[:, :, i, j] = xp[:, :, hs:hs + sh * (ho - 1) + 1:sh, ws:ws + sw * (wo - 1) + 1:sw]
    return cols.reshape(b, c * kh * kw, ho * wo).transpose(0, 2, 1).reshape(b * ho * wo, c * kh * kw)


def conv_grad_rows(g, scale: float = 1.0) -> np.ndarray:
    """[B, C, Ho, Wo] output gradients -> [B*Ho*Wo, C] rows, times `scale`
    (the batch size, undoing the 1/b of a batch-mean loss)."""
    g = np.asarray(g, dtype=np.float64)
    b, c, ho, wo = g.shape
    return scale * g.transpose(0, 2, 3, 1).reshape(b * ho * wo, c)
