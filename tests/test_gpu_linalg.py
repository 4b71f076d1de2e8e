"""GPU parity of the operator API (libspdkfac.so) against the float64 oracle.

Tolerances (north_star): relative Frobenius error <= 1e-4 on factors and
preconditioned gradients; inverses within a condition-number-scaled bound
    ||X - X_ref||_F / ||X_ref||_F <= C_INV * kappa(M + gamma I) * 2^-24,
with C_INV = 16 * sqrt(d) (fp32 Cholesky/Gauss-Jordan forward-error scale),
and additionally never worse than 8x the error of cuSOLVER's fp32
Cholesky inverse of the same matrix (torch.cholesky_inverse, comparison only).
"""

import math
import pathlib

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FACTOR_TOL = 1e-4
PRECOND_TOL = 1e-4
GOLD = pathlib.Path(__file__).parent / "golden"


def _K():
    import paper_2107_06533_b200.linalg as K
    return K


def relf(got, want):
    got = got.detach().double().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def spd(rng, d, jitter=0.1):
    b = rng.standard_normal((d, d))
    return b @ b.T / d + jitter * np.eye(d)


@pytest.mark.parametrize("b,d", [(1, 1), (1, 3), (7, 5), (32, 64), (64, 130), (9, 200), (1000, 300),
                                 (4096, 576), (32, 2048), (1568, 1152), (100, 4608)])
def test_factor_rows_matches_oracle(b, d):
    K = _K()
    rng = np.random.default_rng(b * 7919 + d)
    x = rng.standard_normal((b, d))
    got = K.compute_factor_A(torch.tensor(x, dtype=torch.float32))
    want = O.factor_A(x.astype(np.float32).astype(np.float64))
    assert relf(got, want) <= FACTOR_TOL
    assert torch.equal(got, got.T)  # unpack writes both triangles from one packed value


def test_factor_golden():
    K = _K()
    lg = np.load(GOLD / "linalg_golden.npz")
    for key in [k for k in lg.files if k.startswith("fa_x_")]:
        x = lg[key]
        got = K.compute_factor_G(torch.tensor(x, dtype=torch.float32))
        assert relf(got, lg["fg_y_" + key[5:]]) <= FACTOR_TOL


def test_factor_known_answers():  # pkg/tests/test_linalg.py:43-57 (exact in fp32)
    K = _K()
    assert torch.equal(K.compute_factor_A([[1.0, 0.0]]).cpu(), torch.tensor([[1.0, 0.0], [0.0, 0.0]]))
    assert torch.equal(K.compute_factor_G([[0.0, 2.0]]).cpu(), torch.tensor([[0.0, 0.0], [0.0, 4.0]]))
    assert torch.allclose(K.compute_factor_G([[1.0, 0.0], [0.0, 1.0]]).cpu(), 0.5 * torch.eye(2), atol=0)
    with pytest.raises(ValueError, match="empty"):
        K.compute_factor_A(torch.zeros(0, 3))


@pytest.mark.parametrize("shape,k,s,p", [((2, 3, 9, 9), 3, 1, 1), ((4, 16, 14, 14), 3, 2, 1), ((2, 3, 32, 32), 7, 2, 3),
                                         ((8, 64, 8, 8), 1, 1, 0), ((2, 64, 28, 28), 3, 1, 1)])
def test_factor_conv_matches_oracle(shape, k, s, p):
    K = _K()
    rng = np.random.default_rng(sum(shape) + k)
    x = rng.standard_normal(shape).astype(np.float32)
    got = K.compute_factor_A_conv(torch.tensor(x), k, s, p)
    want = O.factor_A(O.im2col_rows(x, k, k, s, p))
    assert relf(got, want) <= FACTOR_TOL


@pytest.mark.parametrize("shape,k,s,p", [((2, 3, 9, 9), 3, 1, 1), ((4, 16, 14, 14), 3, 2, 1), ((2, 3, 32, 32), 7, 2, 3),
                                         ((8, 64, 8, 8), 1, 1, 0), ((2, 40, 28, 28), 3, 1, 1)])
def test_factor_conv_channels_last(shape, k, s, p):
    """NHWC staging: rows ordered (kh, kw, c) = the oracle's (c, kh, kw) factor permuted."""
    K = _K()
    import paper_2107_06533_b200._lib as L
    rng = np.random.default_rng(sum(shape) + 7 * k)
    x = rng.standard_normal(shape).astype(np.float32)
    xt = torch.tensor(x).cuda().contiguous(memory_format=torch.channels_last)
    plan = K.FactorPlan(L.CONV_A_NHWC, x.shape, (k, k), (s, s), (p, p))
    packed = torch.empty(plan.packed_size, device="cuda")
    plan.run(xt, packed)
    got = K.unpack_upper(packed, plan.dim)
    c = shape[1]
    perm = [ci * k * k + ki * k + kj for ki in range(k) for kj in range(k) for ci in range(c)]
    want = O.factor_A(O.im2col_rows(x, k, k, s, p))[np.ix_(perm, perm)]
    assert relf(got, want) <= FACTOR_TOL


@pytest.mark.parametrize("shape", [(2, 5, 3, 3), (32, 64, 56, 56), (32, 2048, 7, 7)])
def test_factor_spatial_channels_last(shape):
    K = _K()
    import paper_2107_06533_b200._lib as L
    rng = np.random.default_rng(shape[1] + 1)
    g = rng.standard_normal(shape).astype(np.float32)
    gt = torch.tensor(g).cuda().contiguous(memory_format=torch.channels_last)
    plan = K.FactorPlan(L.SPATIAL_NHWC, g.shape)
    packed = torch.empty(plan.packed_size, device="cuda")
    plan.run(gt, packed)
    want = O.factor_G(O.conv_grad_rows(g))
    assert relf(K.unpack_upper(packed, plan.dim), want) <= FACTOR_TOL


@pytest.mark.parametrize("shape", [(2, 5, 3, 3), (32, 64, 56, 56), (32, 2048, 7, 7)])
def test_factor_spatial_matches_oracle(shape):
    K = _K()
    rng = np.random.default_rng(shape[1])
    g = rng.standard_normal(shape).astype(np.float32)
    got = K.compute_factor_G_spatial(torch.tensor(g), row_scale=shape[0])
    want = O.factor_G(O.conv_grad_rows(g, scale=shape[0]))
    assert relf(got, want) <= FACTOR_TOL


def test_factor_running_average_and_world_scale():
    K = _K()
    import paper_2107_06533_b200._lib as L
    rng = np.random.default_rng(5)
    x = rng.standard_normal((300, 200)).astype(np.float32)
    old = spd(rng, 200)
    plan = K.FactorPlan(L.ROWS, x.shape)
    packed = K.pack_upper(torch.tensor(old, dtype=torch.float32))
    plan.run(torch.tensor(x).cuda(), packed, decay=0.9, world_scale=0.25)
    want = 0.25 * (0.9 * old + 0.1 * O.factor_A(x.astype(np.float64)))
    assert relf(K.unpack_upper(packed, 200), want) <= FACTOR_TOL


@pytest.mark.parametrize("d", [1, 2, 17, 64, 129, 512, 1000])
def test_pack_round_trip_exact(d):
    K = _K()
    rng = np.random.default_rng(d)
    m = torch.tensor(spd(rng, d), dtype=torch.float32)
    m = (m + m.T) / 2
    p = K.pack_upper(m)
    assert torch.equal(p.cpu(), torch.tensor(O.pack_upper(m.double().numpy()), dtype=torch.float32))
    assert torch.equal(K.unpack_upper(p, d).cpu(), m)


def test_pack_unpack_batched_exact():
    """spdkfac_(un)pack_upper_batched_f32 (the inverse broadcast path): tiled unpack of mixed
    sizes, including partial 64-tiles, is bit-exact against the oracle's unpack_upper."""
    import ctypes as C
    from paper_2107_06533_b200 import _lib as L
    lib = L.load(require_device=True)
    dims = [1, 5, 63, 64, 65, 130, 300, 700]
    rng = np.random.default_rng(5)
    fulls = []
    for d in dims:
        m = torch.tensor(spd(rng, d), dtype=torch.float32)
        fulls.append(((m + m.T) / 2).cuda())
    packed = [torch.empty(d * (d + 1) // 2, device="cuda") for d in dims]
    back = [torch.full((d, d), float("nan"), device="cuda") for d in dims]
    s = torch.cuda.current_stream().cuda_stream
    L.check(lib.spdkfac_pack_upper_batched_f32(len(dims), L.i32_array(dims), L.ptr_array([f.data_ptr() for f in fulls]),
                                               L.ptr_array([p.data_ptr() for p in packed]), s), "pack")
    L.check(lib.spdkfac_unpack_upper_batched_f32(len(dims), L.i32_array(dims), L.ptr_array([p.data_ptr() for p in packed]),
                                                 L.ptr_array([b.data_ptr() for b in back]), s), "unpack")
    torch.cuda.synchronize()
    for d, f, p, b in zip(dims, fulls, packed, back):
        assert torch.equal(p.cpu(), torch.tensor(O.pack_upper(f.double().cpu().numpy()), dtype=torch.float32)), d
        assert torch.equal(b, f), d


def inverse_bound(m, gamma, got_err):
    d = m.shape[0]
    ev = np.linalg.eigvalsh(m + gamma * np.eye(d))
    kappa = ev[-1] / ev[0]
    return 16.0 * math.sqrt(d) * kappa * 2.0 ** -24, kappa


def cusolver_err(m, gamma, want):
    t = torch.tensor(m + gamma * np.eye(m.shape[0]), dtype=torch.float32, device="cuda")
    ref = torch.cholesky_inverse(torch.linalg.cholesky(t))
    return relf(ref, want)


@pytest.mark.parametrize("d,gamma", [(1, 0.5), (5, 0.0), (17, 0.01), (64, 0.1), (128, 0.05), (129, 0.05), (147, 0.1),
                                     (256, 0.1), (300, 0.01), (576, 0.1), (1024, 0.1), (2304, 0.1)])
def test_damped_inverse_matches_oracle(d, gamma):
    K = _K()
    rng = np.random.default_rng(d)
    m = spd(rng, d)
    mt = torch.tensor(m, dtype=torch.float32)
    m32 = mt.double().numpy()
    got = K.damped_inverse(mt, gamma)
    want = O.damped_inverse(m32, gamma)
    err = relf(got, want)
    bound, kappa = inverse_bound(m32, gamma, err)
    ref = cusolver_err(m32, gamma, want)
    assert err <= max(bound, 8 * ref), (err, bound, ref, kappa)
    assert torch.equal(got, got.T)


def test_damped_inverse_golden():
    K = _K()
    lg = np.load(GOLD / "linalg_golden.npz")
    for key in [k for k in lg.files if k.startswith("inv_m_")]:
        d = key[6:]
        m, gamma = lg[key], float(lg["inv_gamma_" + d])
        got = K.damped_inverse(torch.tensor(m, dtype=torch.float32), gamma)
        want = lg["inv_y_" + d]
        bound, _ = inverse_bound(m, gamma, 0)
        assert relf(got, want) <= max(bound, 8 * cusolver_err(m, gamma, want))


def test_damped_inverse_batched_mixed_sizes():
    K = _K()
    rng = np.random.default_rng(77)
    dims = [64, 147, 256, 64, 1000, 128, 512]
    mats = [spd(rng, d) for d in dims]
    outs = K.damped_inverse_batched([torch.tensor(m, dtype=torch.float32).cuda() for m in mats], 0.1)
    for m, o in zip(mats, outs):
        want = O.damped_inverse(m.astype(np.float32).astype(np.float64), 0.1)
        bound, _ = inverse_bound(m, 0.1, 0)
        assert relf(o, want) <= max(bound, 8 * cusolver_err(m, 0.1, want))


def test_damped_inverse_errors():  # pkg/tests/test_linalg.py:125-133
    K = _K()
    with pytest.raises(K.NotPositiveDefiniteError) as e:
        K.damped_inverse(torch.diag(torch.tensor([1.0, -1.0, 2.0])), 0.0)
    assert e.value.pivot == 1
    with pytest.raises(ValueError, match="nonnegative"):
        K.damped_inverse(torch.eye(2), -0.1)
    # failure inside the blocked path: leading 200x200 block PD, pivot 200 negative
    d = 300
    m = np.eye(d)
    m[200, 200] = -1.0
    with pytest.raises(K.NotPositiveDefiniteError) as e:
        K.damped_inverse(torch.tensor(m, dtype=torch.float32), 0.0)
    assert e.value.pivot == 200
    assert torch.allclose(K.damped_inverse(torch.eye(3), 0.0).cpu(), torch.eye(3), atol=1e-7)
    assert torch.allclose(K.damped_inverse(torch.eye(2), 1.0).cpu(), 0.5 * torch.eye(2), atol=1e-7)


@pytest.mark.parametrize("dout,din", [(1, 1), (3, 5), (10, 64), (64, 147), (130, 70), (256, 2304), (1000, 2048),
                                      (2048, 512)])
def test_precondition_matches_oracle(dout, din):
    K = _K()
    rng = np.random.default_rng(dout * 31 + din)
    g = rng.standard_normal((dout, din)).astype(np.float32)
    a = spd(rng, din, 1.0).astype(np.float32)
    gi = spd(rng, dout, 1.0).astype(np.float32)
    got = K.precondition(torch.tensor(g), torch.tensor(a), torch.tensor(gi))
    want = O.precondition(g.astype(np.float64), a.astype(np.float64), gi.astype(np.float64))
    assert relf(got, want) <= PRECOND_TOL


def test_precondition_golden_and_kat():
    K = _K()
    lg = np.load(GOLD / "linalg_golden.npz")
    for key in [k for k in lg.files if k.startswith("pc_grad_")]:
        t = key[8:]
        got = K.precondition(torch.tensor(lg[key], dtype=torch.float32), torch.tensor(lg["pc_ainv_" + t], dtype=torch.float32),
                             torch.tensor(lg["pc_ginv_" + t], dtype=torch.float32))
        assert relf(got, lg["pc_y_" + t]) <= PRECOND_TOL
    g = torch.arange(6.0).reshape(2, 3)
    assert torch.allclose(K.precondition(g, torch.eye(3), torch.eye(2)).cpu(), g, atol=0)
    with pytest.raises(ValueError, match="shape mismatch"):
        K.precondition(torch.zeros(2, 3), torch.eye(2), torch.eye(2))


@pytest.mark.parametrize("f16", ["0", "1"])
def test_precond_stage_packed_matches_stage_inverses(f16, monkeypatch):
    """PrecondPlan.stage_packed (the broadcast path: packed inverse -> full + operand planes in one
    pass) gives the same preconditioned gradients and bit-identical full inverses as unpack +
    stage_inverses: bit-identical on tf32 planes; on fp16 planes (opt-in SPDKFAC_PRECOND_F16=1) the two
    routes scale the inverse rows differently (exact row maxima vs the SPD diagonal bound): equal to 1e-6."""
    monkeypatch.setenv("SPDKFAC_PRECOND_F16", f16)
    K = _K()
    rng = np.random.default_rng(9)
    shapes = [(70, 130), (200, 64)]
    grads = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    a_inv = [torch.tensor(spd(rng, s[1]), dtype=torch.float32, device="cuda") for s in shapes]
    g_inv = [torch.tensor(spd(rng, s[0]), dtype=torch.float32, device="cuda") for s in shapes]
    a_inv = [(m + m.T) / 2 for m in a_inv]
    g_inv = [(m + m.T) / 2 for m in g_inv]
    out1 = [torch.empty(s, device="cuda") for s in shapes]
    p1 = K.PrecondPlan(shapes)
    p1.run(g_inv, grads, a_inv, out=out1)
    p2 = K.PrecondPlan(shapes)
    full_a = [torch.full_like(m, float("nan")) for m in a_inv]
    full_g = [torch.full_like(m, float("nan")) for m in g_inv]
    p2.stage_packed("A", [0, 1], [K.pack_upper(m) for m in a_inv], full_a)
    p2.stage_packed("G", [0, 1], [K.pack_upper(m) for m in g_inv], full_g)
    out2 = [torch.empty(s, device="cuda") for s in shapes]
    p2.bind(g_inv, grads, a_inv, out=out2)
    p2.run_bound(0.0, inverses_staged=True)
    torch.cuda.synchronize()
    for x, y in zip(out1, out2):
        assert torch.equal(x, y) if f16 == "0" else relf(x, y.double().cpu().numpy()) <= 1e-6
    for f, m in zip(full_a + full_g, a_inv + g_inv):
        assert torch.equal(f, m)


def test_pack_batched_many_rows():
    """A pack batch whose rows sum past 65535 (BERT-base linears at P=2: 24 x 3072 + 60 x 768
    owned inverses): bit-exact against the oracle's pack_upper."""
    from paper_2107_06533_b200 import _lib as L
    lib = L.load(require_device=True)
    dims = [3072] * 20 + [768] * 10
    assert sum(dims) > 65535
    g = torch.Generator(device="cuda").manual_seed(9)
    fulls = []
    for d in dims:
        m = torch.randn(d, d, device="cuda", generator=g)
        fulls.append((m + m.T) / 2)
    packed = [torch.full((d * (d + 1) // 2,), float("nan"), device="cuda") for d in dims]
    s = torch.cuda.current_stream().cuda_stream
    L.check(lib.spdkfac_pack_upper_batched_f32(len(dims), L.i32_array(dims), L.ptr_array([f.data_ptr() for f in fulls]),
                                               L.ptr_array([p.data_ptr() for p in packed]), s), "pack")
    torch.cuda.synchronize()
    for d, f, p in zip(dims[::7], fulls[::7], packed[::7]):
        iu = torch.triu_indices(d, d, device="cuda")
        assert torch.equal(p, f[iu[0], iu[1]]), d


@pytest.mark.parametrize("mag,gamma", [(1e-6, 1e-3), (1e-6, 0.1), (1e3, 1e-4), (1.0, 1e-5), (1e8, 0.1), (1e-3, 1e-2)])
@pytest.mark.parametrize("tf32", ["0", "1"])
def test_damped_inverse_plane_scaling(mag, gamma, tf32, monkeypatch):
    """The blocked inverse's panel / update operands are fp16 planes scaled per operand class (1/gamma,
    sqrt(sigma/gamma), sigma: inv_scale_kernel) or tf32 planes (SPDKFAC_INV_TF32=1, and every run with
    gamma < 1e-4).  Factors of very small and very large magnitude against small and large damping,
    full-rank and rank-deficient (rows < d, as the G factors of small batches).  tf32 planes: the
    kappa-scaled fp32 bound.  fp16 planes: the same bound while sigma / gamma <= 2^16 (sigma = max
    diagonal of F + gamma I), beyond it the documented normwise model (sigma / gamma) 2^-38."""
    K = _K()
    monkeypatch.setenv("SPDKFAC_INV_TF32", tf32)
    rng = np.random.default_rng(int(abs(math.log10(mag)) * 10 + abs(math.log10(gamma))))
    for d, rows in [(384, 1000), (640, 96)]:
        x = rng.standard_normal((rows, d)) * (1.0 + rng.random(d) * 3.0)
        m = (x.T @ x / rows * mag).astype(np.float32).astype(np.float64)
        ev = np.linalg.eigvalsh(m + gamma * np.eye(d))
        if ev[0] <= 0 or ev[-1] / ev[0] > 1e6:  # indefinite after the fp32 rounding of F, or beyond fp32
            continue                                # (kappa u > 0.06): a failed pivot is then the right answer
        got = K.damped_inverse(torch.tensor(m, dtype=torch.float32), gamma)
        want = O.damped_inverse(m, gamma)
        err = relf(got, want)
        bound, kappa = inverse_bound(m, gamma, err)
        ref = cusolver_err(m, gamma, want)
        assert np.isfinite(got.cpu().numpy()).all()
        rng_ratio = (np.max(np.diag(m)) + gamma) / gamma
        f16 = tf32 == "0" and gamma >= 1e-4
        model = 16 * rng_ratio * 2.0 ** -38 if (f16 and rng_ratio > 2.0 ** 16) else 0.0
        assert err <= max(bound, 8 * ref, model), (d, err, bound, ref, kappa, rng_ratio)


@pytest.mark.parametrize("pairs", ["1", "0"])
def test_damped_inverse_update_engines(pairs, monkeypatch):
    """The blocked inverse with the CTA-pair update engine (SPDKFAC_UPDATE_PAIRS=1: 2x2 super tiles,
    including diagonal ones whose dead lower block is written) and with single-CTA tiles only."""
    K = _K()
    monkeypatch.setenv("SPDKFAC_UPDATE_PAIRS", pairs)
    rng = np.random.default_rng(123)
    dims = [1152, 2304, 640]
    mats = [spd(rng, d) for d in dims]
    outs = K.damped_inverse_batched([torch.tensor(m, dtype=torch.float32).cuda() for m in mats], 0.1)
    for m, o in zip(mats, outs):
        want = O.damped_inverse(m.astype(np.float32).astype(np.float64), 0.1)
        bound, _ = inverse_bound(m, 0.1, 0)
        assert relf(o, want) <= max(bound, 8 * cusolver_err(m, 0.1, want))


@pytest.mark.parametrize("shape,k,s,p", [((4, 64, 17, 17), (1, 7), (1, 1), (0, 3)), ((4, 64, 17, 17), (7, 1), (1, 1), (3, 0)),
                                         ((3, 40, 8, 8), (1, 3), (1, 1), (0, 1)), ((3, 40, 8, 8), (3, 1), (1, 1), (1, 0)),
                                         ((2, 24, 15, 15), (3, 3), (2, 2), (0, 0))])
@pytest.mark.parametrize("nhwc", [False, True])
def test_factor_conv_nonsquare_kernels(shape, k, s, p, nhwc):
    """Inception-v4's non-square kernels with one-axis padding (BASELINE configs[4]), both staging
    layouts: NCHW (c, kh, kw) column order and channels-last (kh, kw, c)."""
    K = _K()
    import paper_2107_06533_b200._lib as L
    rng = np.random.default_rng(sum(shape) + k[0] * 3 + k[1])
    x = rng.standard_normal(shape).astype(np.float32)
    want = O.factor_A(O.im2col_rows(x, k[0], k[1], s, p))
    if nhwc:
        xt = torch.tensor(x).cuda().contiguous(memory_format=torch.channels_last)
        plan = K.FactorPlan(L.CONV_A_NHWC, x.shape, k, s, p)
        c = shape[1]
        perm = [ci * k[0] * k[1] + ki * k[1] + kj for ki in range(k[0]) for kj in range(k[1]) for ci in range(c)]
        want = want[np.ix_(perm, perm)]
    else:
        xt = torch.tensor(x).cuda()
        plan = K.FactorPlan(L.CONV_A, x.shape, k, s, p)
    packed = torch.empty(plan.packed_size, device="cuda")
    plan.run(xt, packed)
    assert relf(K.unpack_upper(packed, plan.dim), want) <= FACTOR_TOL
