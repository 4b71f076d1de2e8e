"""Host replica of the blocked-sweep update planner in csrc/inverse.cu (fused trailing updates,
kFuse steps per W pass), executed in float64: the plan's algebra must reproduce the inverse.
Pure CPU (no kernels): it pins the item logic (which tiles each step updates and with which
pending steps' panels) that the tcgen05 update launches follow."""
import numpy as np
import pytest


def plan(T, k, fuse):
    """(I, J, first pending step) of step k's update items (I <= J, upper block triangle)."""
    k0 = k - k % fuse
    last = min(k0 + fuse - 1, T - 1)

    def touched(s, I, J):
        return I == s or J == s or (s + 1 <= I <= last + 1) or (s + 1 <= J <= last + 1)

    items = []
    for I in range(T):
        for J in range(I, T):
            if I == k or J == k:
                continue
            eager = (k + 1 <= I <= last + 1) or (k + 1 <= J <= last + 1)
            first = k
            if k == last:
                first = next((s + 1 for s in range(k - 1, k0 - 1, -1) if touched(s, I, J)), k0)
            elif not eager:
                continue
            items.append((I, J, first))
    return items


def blocked_sweep_inverse(M, b, fuse):
    T = M.shape[0] // b
    W = M.copy()
    panA, panC = {}, {}
    blk = lambda i: slice(i * b, (i + 1) * b)  # noqa: E731
    for k in range(T):
        K = blk(k)
        Pinv = np.linalg.inv(W[K, K])
        panA[k] = W[:, K].copy()          # Wold[:, K] (current after every earlier step)
        panC[k] = panA[k] @ Pinv          # C = Wold[:, K] P^-1
        for R in range(T):
            if R != k:
                W[blk(R), K] = panC[k][blk(R)]
                W[K, blk(R)] = panC[k][blk(R)].T
        W[K, K] = -Pinv
        for I, J, first in plan(T, k, fuse):
            U = sum(panA[s][blk(I)] @ panC[s][blk(J)].T for s in range(first, k + 1))
            W[blk(I), blk(J)] -= U
            if I != J:
                W[blk(J), blk(I)] = W[blk(I), blk(J)].T
    return -W


@pytest.mark.parametrize("T", [1, 2, 3, 4, 5, 8, 9, 13, 16])
@pytest.mark.parametrize("fuse", [1, 2, 4])
def test_fused_update_plan_inverts(T, fuse):
    rng = np.random.default_rng(T * 10 + fuse)
    b = 4
    n = T * b
    X = rng.standard_normal((n, n))
    M = X @ X.T / n + 0.5 * np.eye(n)
    got = blocked_sweep_inverse(M, b, fuse)
    np.testing.assert_allclose(got, np.linalg.inv(M), atol=1e-11, rtol=0)


def test_fused_plan_cuts_read_modify_write_passes():
    """kFuse = 4 on d = 4608 (T = 36): the tile read-modify-writes fall by about a third versus
    per-pair fusion and the bulk contractions carry K = 512."""
    T = 36

    def rmw(fuse):
        return sum(len(plan(T, k, fuse)) for k in range(T))
    assert rmw(4) < 0.7 * rmw(2) < 0.7 * 0.7 * rmw(1) * 1.5
    ks = {k - first + 1 for k in range(T) for _, _, first in plan(T, k, 4)}
    assert max(ks) == 4
