"""GPU parity of the full optimizer step (SPDKFAC) against the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_golden_fixture_through_optimizer():
    from tests.smoke_impl import TOL, fixture_step
    errs = fixture_step()
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("seed,cl", [(0, False), (1, False), (0, True), (2, True)])
def test_conv_net_step_matches_oracle(seed, cl):
    from tests.smoke_impl import TOL, conv_step
    errs = conv_step(seed=seed, channels_last=cl)
    assert max(errs.values()) <= TOL, errs


def test_running_average_and_frequencies():
    """decay rho: A_t = rho A_{t-1} + (1-rho) A(batch_t); factors only every
    factor_update_freq steps; inverses only every inv_update_freq steps."""
    import oracle as O
    import torch.nn as nn
    from paper_2107_06533_b200.optimizer import SPDKFAC
    torch.manual_seed(3)
    lin = nn.Linear(20, 7, bias=False).cuda()
    opt = SPDKFAC(lin, lr=0.0, damping=0.1, factor_decay=0.8, factor_update_freq=2, inv_update_freq=4)
    xs = [torch.randn(16, 20, device="cuda") for _ in range(5)]
    running = None
    for i, x in enumerate(xs):
        opt.zero_grad()
        lin(x).pow(2).mean().backward()
        inv_before = opt.inv[0].clone()
        opt.step()
        if i % 2 == 0:
            fresh = O.factor_A(x.double().cpu().numpy())
            running = fresh if running is None else 0.8 * running + 0.2 * fresh
        got = opt.factor(0, "A").double().cpu().numpy()
        assert np.linalg.norm(got - running) / np.linalg.norm(running) < 1e-4, i
        if i % 4 != 0:
            assert torch.equal(opt.inv[0], inv_before)
    opt.remove_hooks()


def test_state_dict_round_trip():
    import torch.nn as nn
    from paper_2107_06533_b200.optimizer import SPDKFAC
    lin = nn.Linear(8, 4).cuda()
    opt = SPDKFAC(lin, lr=0.1, damping=0.1)
    lin(torch.randn(5, 8, device="cuda")).sum().backward()
    opt.step()
    sd = opt.state_dict()
    opt2 = SPDKFAC(nn.Linear(8, 4).cuda(), lr=0.1, damping=0.1)
    opt2.load_state_dict(sd)
    assert torch.equal(opt2.bufA, opt.bufA) and all(torch.equal(a, b) for a, b in zip(opt2.inv, opt.inv))
    assert opt2.steps == 1
    opt.remove_hooks()
    opt2.remove_hooks()


def test_nonpd_raises_on_next_step():
    import torch.nn as nn
    from paper_2107_06533_b200.linalg import NotPositiveDefiniteError
    from paper_2107_06533_b200.optimizer import SPDKFAC
    lin = nn.Linear(4, 3, bias=False).cuda()
    opt = SPDKFAC(lin, lr=0.1, damping=0.0)
    x = torch.zeros(2, 4, device="cuda")  # A = 0, gamma = 0: singular
    lin(x).sum().backward()
    opt.step()
    with pytest.raises(NotPositiveDefiniteError) as e:
        opt.check_inverses()
    assert e.value.pivot == 0
    opt.remove_hooks()


def test_nonpd_detected_after_next_inversion():
    """A failed inversion of step N is still reported when step N+1's forward pass has already
    launched (and finished) its own, successful A inversion: each eager step's info goes to its own
    pinned slot, so the next one cannot overwrite it before step() checks it."""
    import torch.nn as nn
    from paper_2107_06533_b200.linalg import NotPositiveDefiniteError
    from paper_2107_06533_b200.optimizer import SPDKFAC
    lin = nn.Linear(4, 3, bias=False).cuda()
    opt = SPDKFAC(lin, lr=0.1, damping=0.0)
    g = torch.Generator(device="cuda").manual_seed(3)
    # step 0: A = 0 (singular at gamma = 0), G full rank (random output weights)
    (lin(torch.zeros(64, 4, device="cuda")) * torch.randn(64, 3, device="cuda", generator=g)).sum().backward()
    opt.step()
    opt.zero_grad(set_to_none=False)
    # step 1: both factors full rank; its A inversion runs (and succeeds) in the forward hooks
    (lin(torch.randn(64, 4, device="cuda", generator=g)) * torch.randn(64, 3, device="cuda", generator=g)).sum().backward()
    torch.cuda.synchronize()
    with pytest.raises(NotPositiveDefiniteError):
        opt.step()
    opt.remove_hooks()


def test_graphed_step_matches_eager():
    """One CUDA-graph replay per iteration gives the same weights as the eager step."""
    import torch.nn as nn
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from tests.smoke_impl import SmallNet
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(7)
    m1 = SmallNet().cuda()
    m2 = SmallNet().cuda()
    m2.load_state_dict(m1.state_dict())
    crit = nn.CrossEntropyLoss()
    xs = [torch.randn(16, 3, 8, 8, device="cuda") for _ in range(5)]
    ys = [torch.randint(0, 10, (16,), device="cuda") for _ in range(5)]
    o1 = SPDKFAC(m1, lr=0.05, damping=0.1)
    for x, y in zip(xs, ys):
        o1.zero_grad(set_to_none=False)
        crit(m1(x), y).backward()
        o1.step()
    o2 = SPDKFAC(m2, lr=0.05, damping=0.1)
    gs = GraphedStep(m2, crit, o2, [xs[0]], [ys[0]], warmup=1)  # warmup = eager step 1 on xs[0]
    for x, y in zip(xs[1:], ys[1:]):
        gs([x], [y])
    torch.cuda.synchronize()
    o2.check_inverses()
    for p1, p2 in zip(m1.parameters(), m2.parameters()):
        assert torch.allclose(p1, p2, rtol=1e-5, atol=1e-6), (p1 - p2).abs().max()
    assert o2.steps == 5
    o1.remove_hooks()
    o2.remove_hooks()


def test_graphed_prefetch_matches_direct_inputs():
    """GraphedStep.prefetch (the next batch copied from pinned host memory on a copy stream while
    the current replay runs, then moved device-to-device into the graph inputs) gives the same
    weights as passing each batch to the call."""
    import torch.nn as nn
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from tests.smoke_impl import SmallNet
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(11)
    m1, m2 = SmallNet().cuda(), SmallNet().cuda()
    m2.load_state_dict(m1.state_dict())
    crit = nn.CrossEntropyLoss()
    xs = [torch.randn(16, 3, 8, 8) for _ in range(6)]
    ys = [torch.randint(0, 10, (16,)) for _ in range(6)]
    xh, yh = [x.pin_memory() for x in xs], [y.pin_memory() for y in ys]
    o1, o2 = SPDKFAC(m1, lr=0.05, damping=0.1), SPDKFAC(m2, lr=0.05, damping=0.1)
    g1 = GraphedStep(m1, crit, o1, [xs[0].cuda()], [ys[0].cuda()], warmup=1)
    g2 = GraphedStep(m2, crit, o2, [xs[0].cuda()], [ys[0].cuda()], warmup=1)
    l1 = [float(g1([xh[i]], [yh[i]]).item()) for i in range(1, 6)]
    l2 = []
    g2.prefetch([xh[1]], [yh[1]])
    for i in range(1, 6):
        loss = g2()
        if i + 1 < 6:
            g2.prefetch([xh[i + 1]], [yh[i + 1]])
        l2.append(float(loss.item()))
    torch.cuda.synchronize()
    assert l1 == l2
    for p1, p2 in zip(m1.parameters(), m2.parameters()):
        assert torch.equal(p1, p2)
    o1.remove_hooks()
    o2.remove_hooks()


@pytest.mark.parametrize("graphed", [False, True])
def test_update_in_backward_matches_step(graphed):
    """update_in_backward: early G groups precondition + update during the backward pass (on
    their own streams); the weights equal those of the plain step() path."""
    import torch.nn as nn
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.workloads import build_model
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(11)
    m1 = build_model("resnet20").cuda()
    m2 = build_model("resnet20").cuda()
    m2.load_state_dict(m1.state_dict())
    crit = nn.CrossEntropyLoss()
    xs = [torch.randn(8, 3, 32, 32, device="cuda") for _ in range(4)]
    ys = [torch.randint(0, 10, (8,), device="cuda") for _ in range(4)]
    freq = 1 if graphed else 2  # GraphedStep captures one step type
    o1 = SPDKFAC(m1, lr=0.05, damping=0.1, inv_update_freq=freq)
    o2 = SPDKFAC(m2, lr=0.05, damping=0.1, inv_update_freq=freq, update_in_backward=True,
                 early_g_fraction=(0.5, 0.9))
    assert len(o2._early) == 2
    for x, y in zip(xs, ys):
        o1.zero_grad(set_to_none=False)
        crit(m1(x), y).backward()
        o1.step()
    if graphed:
        gs = GraphedStep(m2, crit, o2, [xs[0]], [ys[0]], warmup=1)
        for x, y in zip(xs[1:], ys[1:]):
            gs([x], [y])
    else:
        for x, y in zip(xs, ys):
            o2.zero_grad(set_to_none=False)
            crit(m2(x), y).backward()
            assert any(o2._pc_done.values())  # early groups ran during backward
            o2.step()
    torch.cuda.synchronize()
    for p1, p2 in zip(m1.parameters(), m2.parameters()):
        assert torch.allclose(p1, p2, rtol=1e-5, atol=1e-6), (p1 - p2).abs().max()
    o1.remove_hooks()
    o2.remove_hooks()


@pytest.mark.parametrize("seed", [0, 1])
def test_token_linear_step_matches_oracle(seed):
    """Linears on [batch, seq, features] inputs (BASELINE configs[4], BERT-base linears)."""
    from tests.smoke_impl import TOL, token_linear_step
    errs = token_linear_step(seed=seed)
    assert max(errs.values()) <= TOL, errs


def test_second_capture_before_step_raises():
    """A second train-mode forward/backward before step() must not silently freeze a fusion
    group's SYRK: the optimizer raises, and the next proper step works."""
    import torch.nn as nn
    from paper_2107_06533_b200.optimizer import SPDKFAC
    torch.manual_seed(5)
    lin = nn.Sequential(nn.Linear(12, 9, bias=False), nn.ReLU(), nn.Linear(9, 4, bias=False)).cuda()
    opt = SPDKFAC(lin, lr=0.01, damping=0.1)
    for _ in range(2):  # first step: per-layer plans; second: fusion-group objects
        opt.zero_grad()
        lin(torch.randn(8, 12, device="cuda")).pow(2).mean().backward()
        opt.step()
    opt.zero_grad()
    lin(torch.randn(8, 12, device="cuda")).pow(2).mean().backward()
    with pytest.raises(RuntimeError, match="captured twice"):
        lin(torch.randn(8, 12, device="cuda")).pow(2).mean().backward()
    opt.step()
    x = torch.randn(8, 12, device="cuda")
    opt.zero_grad()
    lin(x).pow(2).mean().backward()
    opt.step()
    torch.cuda.synchronize()
    import oracle as O
    want = O.factor_A(x.double().cpu().numpy())
    got = opt.factor(0, "A").double().cpu().numpy()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-4
    opt.remove_hooks()


@pytest.mark.parametrize("ff,fi,uib", [(1, 3, False), (2, 4, True)])
def test_graphed_update_frequencies_match_eager(ff, fi, uib):
    """GraphedStep with factor_update_freq / inv_update_freq > 1 (one graph per step type:
    factors + inversion, factors only, reuse) gives the eager step's weights (simulator.py:126,377)."""
    import torch.nn as nn
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.workloads import build_model
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(13)
    m1 = build_model("resnet20").cuda()
    m2 = build_model("resnet20").cuda()
    m2.load_state_dict(m1.state_dict())
    crit = nn.CrossEntropyLoss()
    n = 10
    xs = [torch.randn(8, 3, 32, 32, device="cuda") for _ in range(n)]
    ys = [torch.randint(0, 10, (8,), device="cuda") for _ in range(n)]
    kw = dict(lr=0.05, damping=0.1, factor_decay=0.9, factor_update_freq=ff, inv_update_freq=fi)
    o1 = SPDKFAC(m1, **kw)
    o2 = SPDKFAC(m2, update_in_backward=uib, **kw)
    for x, y in zip(xs, ys):
        o1.zero_grad(set_to_none=True)
        crit(m1(x), y).backward()
        o1.step()
    gs = GraphedStep(m2, crit, o2, [xs[0]], [ys[0]], warmup=1)
    assert len(gs.graphs) == len({(s % ff == 0, s % fi == 0) for s in range(fi)})
    for x, y in zip(xs[1:], ys[1:]):
        gs([x], [y])
    torch.cuda.synchronize()
    o2.check_inverses()
    assert o2.steps == n
    for p1, p2 in zip(m1.parameters(), m2.parameters()):
        assert torch.allclose(p1, p2, rtol=1e-5, atol=1e-6), (p1 - p2).abs().max()
    assert torch.allclose(o1.bufA, o2.bufA, rtol=1e-5, atol=1e-7)
    o1.remove_hooks()
    o2.remove_hooks()


def test_graphed_step_rejects_lr_change():
    import torch.nn as nn
    from paper_2107_06533_b200.graph import GraphedStep
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from tests.smoke_impl import SmallNet
    torch.manual_seed(2)
    m = SmallNet().cuda()
    o = SPDKFAC(m, lr=0.05, damping=0.1)
    crit = nn.CrossEntropyLoss()
    x, y = torch.randn(16, 3, 8, 8, device="cuda"), torch.randint(0, 10, (16,), device="cuda")
    gs = GraphedStep(m, crit, o, [x], [y], warmup=1)
    gs([x], [y])
    o.param_groups[0]["lr"] = 0.01
    with pytest.raises(RuntimeError, match="learning rate changed"):
        gs([x], [y])
    gs.recapture = True
    gs([x], [y])  # captures again at the new lr
    assert gs.lr == 0.01
    o.remove_hooks()
