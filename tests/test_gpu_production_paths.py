"""GPU parity of the tile-engine paths the ResNet-50 bench step actually selects.

The unit tests in test_gpu_linalg.py cover the operator API at small and medium sizes; these
cover the production engine choices at their production shapes:

  * CTA-pair SYRK (cta_group::2, 256x256 super tiles) with split-K > 1: 6272x2304 (layer3
    conv2 A), 6272x1024, 25088x512, and the 1-split 1568x4608 (layer4 conv2 A);
  * the single-CTA engine with many split-K slices: 100352x256 (layer1 1x1 convs) -- the
    shape whose last K slice used to be empty (uninitialised partial slot);
  * the stem: conv1 A = im2col of [32,3,224,224] k7 s2 p3 (401408 x 147, pair engine, T=2)
    and its spatial output-gradient G [32,64,112,112] (401408 x 64);
  * a mixed FactorGroup (pair and single-CTA members in ONE launch, like a fusion group);
  * the d = 4608 damped inverse of a rank-deficient factor (M = 1568 < d, as layer4 conv2's
    A is) at gamma = 0.1, and a d = 2048 one;
  * 512 x 4608 preconditioning (layer4 conv2).

Tolerances as in test_gpu_linalg.py (north_star): factors and preconditioned gradients
relative Frobenius <= 1e-4 against float64; inverses under the kappa-scaled bound.
"""

import ctypes as C
import math

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


def relf(got, want):
    got = got.detach().double().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def _describe(group, member=0):
    from paper_2107_06533_b200 import _lib as L
    out = (C.c_int64 * 4)()
    L.check(L.load().spdkfac_factor_group_describe(group._h, member, out), "describe")
    return {"pair": out[0] == 1, "f32_rows": out[0] == 2, "im2col": out[0] == 3, "splits": int(out[1]), "rows": int(out[2]), "dim": int(out[3])}


def _group(members, dims, rows):
    """A FactorGroup whose member k writes X_k^T X_k / rows[k] (the optimizer's 1/M scale)."""
    from paper_2107_06533_b200.linalg import FactorGroup
    packed = [torch.full((d * (d + 1) // 2,), float("nan"), device="cuda") for d in dims]
    return FactorGroup(members, packed, [1.0 / r for r in rows]), packed


def _rows_member(m, d):
    from paper_2107_06533_b200 import _lib as L
    return (L.ROWS, (m, d), (1, 1), (1, 1), (0, 0), (1, 1))


def _factor_rows_oracle(x):
    x64 = x.double()
    return (x64.T @ x64 / x.shape[0]).cpu().numpy()


def _correlated_rows(m, d, seed):
    """Post-ReLU-like rows with correlated columns (a realistic factor spectrum, not white noise)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    z = torch.randn(m, d, device="cuda", generator=g)
    mix = torch.randn(d, d, device="cuda", generator=g) / math.sqrt(d)
    return torch.relu(z + 0.5 * z @ mix)


@pytest.mark.parametrize("m,d,pair,min_splits", [(6272, 2304, True, 2), (6272, 1024, True, 2), (25088, 512, True, 2),
                                                 (1568, 4608, True, 1), (100352, 256, False, 2)])
def test_syrk_production_engines(m, d, pair, min_splits):
    x = _correlated_rows(m, d, seed=m + d)
    grp, packed = _group([_rows_member(m, d)], [d], [m])
    info = _describe(grp)
    assert info["pair"] == pair and info["splits"] >= min_splits, info
    # every split-K slice non-empty (the reduce sums all `splits` slots)
    nkb = (m + 63) // 64
    per = -(-nkb // info["splits"])
    assert (info["splits"] - 1) * per < nkb, info
    grp.stage(0, x)
    grp.compute()
    # the workspace is reused: a second run must give the same bits (counters re-armed, no stale partials)
    from paper_2107_06533_b200.linalg import unpack_upper
    first = packed[0].clone()
    grp.stage(0, x)
    grp.compute()
    torch.cuda.synchronize()
    assert torch.equal(first, packed[0])
    got = unpack_upper(packed[0], d)
    assert not torch.isnan(got).any()
    assert relf(got, _factor_rows_oracle(x)) <= TOL


def test_syrk_stem_conv_a_pair_engine():
    """conv1 A: channels-last [32,3,224,224], k7 s2 p3 -> 401408 x 147 (pair engine, T = 2)."""
    from paper_2107_06533_b200 import _lib as L
    from paper_2107_06533_b200.linalg import unpack_upper
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(32, 3, 224, 224, device="cuda", generator=g).contiguous(memory_format=torch.channels_last)
    grp, packed = _group([(L.CONV_A_NHWC, tuple(x.shape), (7, 7), (2, 2), (3, 3), (1, 1))], [147], [401408])
    info = _describe(grp)
    assert info["pair"] and info["rows"] == 401408 and info["splits"] > 1, info
    grp.stage(0, x)
    grp.compute()
    got = unpack_upper(packed[0], 147)
    rows = O.im2col_rows(x.cpu().numpy(), 7, 7, 2, 3)
    want = rows.T @ rows / rows.shape[0]
    perm = [ci * 49 + ki * 7 + kj for ki in range(7) for kj in range(7) for ci in range(3)]  # (kh, kw, c) order
    assert relf(got, want[np.ix_(perm, perm)]) <= TOL


def test_syrk_stem_spatial_g():
    """conv1 G: channels-last output gradients [32,64,112,112] -> 401408 x 64 (148 splits)."""
    from paper_2107_06533_b200 import _lib as L
    from paper_2107_06533_b200.linalg import unpack_upper
    g = torch.Generator(device="cuda").manual_seed(4)
    y = torch.randn(32, 64, 112, 112, device="cuda", generator=g).contiguous(memory_format=torch.channels_last)
    grp, packed = _group([(L.SPATIAL_NHWC, tuple(y.shape), (1, 1), (1, 1), (0, 0), (1, 1))], [64], [401408])
    info = _describe(grp)
    assert info["splits"] > 1, info
    grp.stage(0, y)
    grp.compute()
    rows = y.permute(0, 2, 3, 1).reshape(-1, 64)
    assert relf(unpack_upper(packed[0], 64), _factor_rows_oracle(rows)) <= TOL


_F32_CASES = [("rows", (1000, 100)), ("rows", (333, 36)), ("rows", (31, 256)), ("rows", (5, 4)), ("rows", (77, 252)),
              ("rows", (100352, 256)), ("spatial", (32, 64, 56, 56)), ("pointwise", (8, 128, 14, 14))]


@pytest.mark.parametrize("kind,shape", _F32_CASES)
@pytest.mark.parametrize("f32", ["2", "0"])
def test_syrk_f32_rows_engine(kind, shape, f32, monkeypatch):
    """Row layouts with d <= 256 (linear inputs, channels-last output gradients, 1x1 conv inputs)
    skip the staging pass: the SYRK's converter warps split TMA-loaded fp32 tiles (engine 2).
    SPDKFAC_F32_ROWS=0 stages them as in round 1 (engine 0).  Both against float64: ragged M
    (< one 32-row K block, not a multiple of 64), d not a multiple of 128, many split-K slices."""
    from paper_2107_06533_b200 import _lib as L
    from paper_2107_06533_b200.linalg import unpack_upper
    monkeypatch.setenv("SPDKFAC_F32_ROWS", f32)
    g = torch.Generator(device="cuda").manual_seed(sum(shape))
    if kind == "rows":
        x = torch.relu(torch.randn(*shape, device="cuda", generator=g) + 0.3)
        member, rows = _rows_member(*shape), x
    else:
        x = torch.randn(*shape, device="cuda", generator=g).contiguous(memory_format=torch.channels_last)
        layout = L.SPATIAL_NHWC if kind == "spatial" else L.CONV_A_NHWC
        member = (layout, tuple(x.shape), (1, 1), (1, 1), (0, 0), (1, 1))
        rows = x.permute(0, 2, 3, 1).reshape(-1, shape[1])
    m, d = rows.shape
    grp, packed = _group([member], [d], [m])
    info = _describe(grp)
    assert info["f32_rows"] == (f32 != "0") and not info["pair"], info
    grp.stage(0, x)
    grp.compute()
    first = packed[0].clone()
    grp.stage(0, x)
    grp.compute()
    torch.cuda.synchronize()
    assert torch.equal(first, packed[0])
    assert relf(unpack_upper(packed[0], d), _factor_rows_oracle(rows)) <= TOL


_I2C_CASES = [((32, 64, 56, 56), (3, 3), (1, 1), (1, 1), (1, 1)),    # ResNet-50 layer1 conv2
              ((32, 128, 56, 56), (3, 3), (2, 2), (1, 1), (1, 1)),   # layer2 first conv2 (stride 2)
              ((3, 64, 7, 9), (3, 3), (1, 1), (1, 1), (1, 1)),       # ragged: M = 189 rows
              ((4, 192, 17, 17), (1, 7), (1, 1), (0, 3), (1, 1)),    # Inception-v4 1x7
              ((4, 192, 17, 17), (7, 1), (1, 1), (3, 0), (1, 1)),    # and 7x1
              ((2, 64, 20, 20), (3, 3), (2, 2), (0, 0), (1, 1)),     # stride 2, no padding
              ((2, 64, 20, 20), (3, 3), (1, 1), (2, 2), (2, 2)),     # dilation 2
              ((2, 128, 12, 12), (5, 5), (1, 1), (2, 2), (1, 1))]    # 5x5


@pytest.mark.parametrize("shape,k,st,pd,dl", _I2C_CASES)
@pytest.mark.parametrize("i2c", ["1", "0"])
def test_syrk_im2col_tma_engine(shape, k, st, pd, dl, i2c, monkeypatch):
    """Channels-last k x k convolutions with C % 64 == 0 on the single-CTA engine: the staging pass
    writes the activation's hi / lo planes, and the SYRK gathers its im2col tiles with TMA im2col loads
    (engine 3: padding as out-of-bounds zeros, stride as the traversal step, taps as im2col offsets).
    SPDKFAC_IM2COL=0 (the default) stages the im2col rows instead (engine 0).  Both against float64."""
    from paper_2107_06533_b200 import _lib as L
    from paper_2107_06533_b200.linalg import unpack_upper
    monkeypatch.setenv("SPDKFAC_IM2COL", i2c)
    g = torch.Generator(device="cuda").manual_seed(sum(shape) + k[0])
    x = torch.relu(torch.randn(*shape, device="cuda", generator=g) + 0.2).contiguous(memory_format=torch.channels_last)
    n, c, h, w = shape
    ho = (h + 2 * pd[0] - dl[0] * (k[0] - 1) - 1) // st[0] + 1
    wo = (w + 2 * pd[1] - dl[1] * (k[1] - 1) - 1) // st[1] + 1
    d, m = c * k[0] * k[1], n * ho * wo
    grp, packed = _group([(L.CONV_A_NHWC, shape, k, st, pd, dl)], [d], [m])
    info = _describe(grp)
    assert info["im2col"] == (i2c == "1") and info["rows"] == m, info
    for _ in range(2):
        grp.stage(0, x)
        grp.compute()
    rows = O.im2col_rows(x.double().cpu().numpy(), k[0], k[1], st, pd, dl)
    perm = [ci * k[0] * k[1] + ki * k[1] + kj for ki in range(k[0]) for kj in range(k[1]) for ci in range(c)]
    want = (rows.T @ rows / rows.shape[0])[np.ix_(perm, perm)]
    assert relf(unpack_upper(packed[0], d), want) <= TOL


def test_f32_rows_members_beyond_launch_limit_are_staged(monkeypatch):
    """A factor group launch carries at most 40 fp32 row maps (Inception-v4's groups hold more row
    members): the members beyond it are staged instead, in the same launch."""
    from paper_2107_06533_b200.linalg import unpack_upper
    monkeypatch.setenv("SPDKFAC_F32_ROWS", "2")
    shapes = [(64 + 7 * k, 32 + 4 * (k % 5)) for k in range(45)]
    xs = [_correlated_rows(m, d, seed=k) for k, (m, d) in enumerate(shapes)]
    grp, packed = _group([_rows_member(m, d) for m, d in shapes], [d for _, d in shapes], [m for m, _ in shapes])
    eng = [_describe(grp, k)["f32_rows"] for k in range(len(shapes))]
    assert eng == [True] * 40 + [False] * 5, eng
    for k, x in enumerate(xs):
        grp.stage(k, x)
    grp.compute()
    for k, x in enumerate(xs):
        assert relf(unpack_upper(packed[k], shapes[k][1]), _factor_rows_oracle(x)) <= TOL, k


def test_mixed_factor_group_one_launch(monkeypatch):
    """Pair-engine, single-CTA staged, single-CTA fp32-rows and TMA-im2col members (split and unsplit)
    reduced by one group compute."""
    monkeypatch.setenv("SPDKFAC_F32_ROWS", "2")
    monkeypatch.setenv("SPDKFAC_IM2COL", "1")
    from paper_2107_06533_b200 import _lib as L
    from paper_2107_06533_b200.linalg import unpack_upper
    shapes = [(6272, 2304), (6272, 256), (1000, 300), (25088, 512), (32, 2048)]
    xs = [_correlated_rows(m, d, seed=k) for k, (m, d) in enumerate(shapes)]
    conv = torch.randn(8, 64, 28, 28, device="cuda").contiguous(memory_format=torch.channels_last)
    members = [_rows_member(m, d) for m, d in shapes] + [(L.CONV_A_NHWC, tuple(conv.shape), (3, 3), (1, 1), (1, 1),
                                                          (1, 1))]
    dims = [d for _, d in shapes] + [576]
    grp, packed = _group(members, dims, [m for m, _ in shapes] + [8 * 28 * 28])
    kinds = [_describe(grp, k)["pair"] for k in range(len(members))]
    assert any(kinds) and not all(kinds), kinds
    assert any(_describe(grp, k)["f32_rows"] for k in range(len(members)))  # (6272, 256): fp32 rows
    assert _describe(grp, len(members) - 1)["im2col"]  # the 3x3 conv, C = 64
    for k, x in enumerate(xs + [conv]):
        grp.stage(k, x)
    grp.compute(decay=0.0, world_scale=0.5)
    for k, x in enumerate(xs):
        assert relf(unpack_upper(packed[k], dims[k]), 0.5 * _factor_rows_oracle(x)) <= TOL, k
    rows = O.im2col_rows(conv.cpu().numpy(), 3, 3, 1, 1)
    perm = [ci * 9 + ki * 3 + kj for ki in range(3) for kj in range(3) for ci in range(64)]
    want = (rows.T @ rows / rows.shape[0])[np.ix_(perm, perm)]
    assert relf(unpack_upper(packed[-1], 576), 0.5 * want) <= TOL


def _kappa(m, gamma, inv):
    """kappa(M + gamma I) = ||M + gamma I||_2 ||(M + gamma I)^-1||_2 by power iteration (float64)."""
    def norm2(a):
        v = np.random.default_rng(0).standard_normal(a.shape[0])
        for _ in range(60):
            v = a @ v
            v /= np.linalg.norm(v)
        return float(v @ (a @ v))
    return norm2(m + gamma * np.eye(m.shape[0])) * norm2(inv)


@pytest.mark.parametrize("d,m", [(4608, 1568), (2048, 1568)])
def test_damped_inverse_production_factor(d, m):
    """A factor as layer4's (M = 1568 rows, rank-deficient for d = 4608), computed by the GPU
    SYRK, inverted at gamma = 0.1 by the blocked sweep (36 / 16 pivot steps)."""
    from paper_2107_06533_b200.linalg import FactorPlan, InversePlan
    from paper_2107_06533_b200 import _lib as L
    gamma = 0.1
    x = _correlated_rows(m, d, seed=d)
    plan = FactorPlan(L.ROWS, x.shape)
    packed = torch.empty(plan.packed_size, device="cuda")
    plan.run(x, packed)
    out = torch.empty(d, d, device="cuda")
    inv = InversePlan([packed], [out])
    inv.run(gamma)
    inv.check()
    from paper_2107_06533_b200.linalg import unpack_upper
    f64 = unpack_upper(packed, d).double().cpu().numpy()
    want = O.damped_inverse(f64, gamma)
    err = relf(out, want)
    kappa = _kappa(f64, gamma, want)
    bound = 16.0 * math.sqrt(d) * kappa * 2.0 ** -24
    t = torch.tensor(f64 + gamma * np.eye(d), dtype=torch.float32, device="cuda")
    ref = relf(torch.cholesky_inverse(torch.linalg.cholesky(t)), want)  # cuSOLVER fp32, calibration only
    print(f"d={d} kappa={kappa:.3g} err={err:.3g} bound={bound:.3g} cusolver={ref:.3g}")
    assert err <= max(bound, 8 * ref), (err, bound, ref, kappa)
    assert torch.equal(out, out.T)


def test_precondition_512x4608():
    """layer4 conv2: grad [512, 4608], A^-1 4608^2, G^-1 512^2, with the fused update W -= alpha P."""
    from paper_2107_06533_b200.linalg import PrecondPlan
    rng = np.random.default_rng(45)
    dout, din = 512, 4608

    def spd(d):
        b = rng.standard_normal((d, d)).astype(np.float32)
        m = b @ b.T / d + np.eye(d, dtype=np.float32)
        return (m + m.T) / 2

    g = rng.standard_normal((dout, din)).astype(np.float32)
    a, gi = spd(din), spd(dout)
    w0 = rng.standard_normal((dout, din)).astype(np.float32)
    gt, at, git = (torch.tensor(v, device="cuda") for v in (g, a, gi))
    w = torch.tensor(w0, device="cuda")
    out = torch.empty(dout, din, device="cuda")
    plan = PrecondPlan([(dout, din)])
    plan.run([git], [gt], [at], out=[out])
    want = O.precondition(g.astype(np.float64), a.astype(np.float64), gi.astype(np.float64))
    assert relf(out, want) <= TOL
    alpha = 0.01
    plan.run([git], [gt], [at], weights=[w], alpha=alpha)
    torch.cuda.synchronize()
    delta = w.double().cpu().numpy() - w0.astype(np.float64)
    assert relf(delta, -alpha * want) <= TOL
