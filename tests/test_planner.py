"""Host plans: identical to the reference's plans on identical inputs
(golden plans.json from tests/golden/make_golden.py), plus the reference's
own planner/perf-model unit tests restated (pkg/tests/test_planner.py,
test_perfmodel.py)."""

import json
import pathlib
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2107_06533_b200 import perfmodel as PM
from paper_2107_06533_b200 import planner as P

GOLD = pathlib.Path(__file__).parent / "golden"
PLANS = json.loads((GOLD / "plans.json").read_text())
PROFILES = json.loads((GOLD / "profiles.json").read_text())
PARAMS = PM.PerfParams(PM.AllReduceParams(PLANS["params"]["alpha_ar"], PLANS["params"]["beta_ar"]),
                       PM.BcastParams(PLANS["params"]["alpha_bcast"], PLANS["params"]["beta_bcast"]),
                       PM.InverseParams(PLANS["params"]["alpha_inv"], PLANS["params"]["beta_inv"]),
                       PLANS["params"]["fitted_world_size"])
ALL_CT = (PM.InverseParams(1.0, 1e-6), PM.BcastParams(1e-9, 1e-12))


def layers(name):
    return [SimpleNamespace(**l) for l in PROFILES[name]["layers"]]


def inv_tasks(dims):
    return [P.InvTask(i, d, i // 2 + 1, P.FactorKind.A if i % 2 == 0 else P.FactorKind.G) for i, d in enumerate(dims)]


def fwd_tasks(times, dims=None):
    dims = dims or [2] * len(times)
    return [P.FactorTask(i + 1, P.FactorKind.A, d, c) for i, (c, d) in enumerate(zip(times, dims))]


@pytest.mark.parametrize("model", sorted(PLANS["models"]))
def test_fusion_plans_identical_to_reference(model):
    ly = layers(model)
    for policy in P.FusionPolicy:
        fwd = P.plan_fusion(P.factor_tasks(ly, P.FactorKind.A), [l.t_ff for l in ly], PARAMS.allreduce, policy)
        bwd = P.plan_fusion(P.factor_tasks(ly, P.FactorKind.G), [l.t_bp for l in reversed(ly)], PARAMS.allreduce, policy)
        want = PLANS["models"][model]["fusion"][policy.value]
        assert [[[t.layer_index, t.kind.value] for t in g] for g in fwd.groups] == want["forward"]
        assert [[[t.layer_index, t.kind.value] for t in g] for g in bwd.groups] == want["backward"]


@pytest.mark.parametrize("model", sorted(PLANS["models"]))
def test_placements_identical_to_reference(model):
    tasks = P.inverse_tasks(layers(model))
    for key, want in PLANS["models"][model]["placement"].items():
        parts = key.split("_")
        p = int(parts[1])
        if parts[0] == "lbp":
            plan = P.lbp_place(tasks, p, PARAMS.inverse, PARAMS.bcast, balance="_".join(parts[2:]))
        else:
            plan = P.seq_place(tasks, p)
        assert [list(w) for w in plan.workers] == want["workers"], key
        assert sorted(plan.nct) == want["nct"], key
        assert P.placement_makespan(plan, PARAMS.inverse, PARAMS.bcast) == pytest.approx(want["makespan"], rel=1e-12)


def test_perfmodel_known_answers():
    kat = PLANS["perfmodel_kat"]
    for m, t in kat["allreduce"]:
        assert PM.allreduce_time(m, PARAMS.allreduce) == t
    for d, t in kat["bcast"]:
        assert PM.bcast_time(d, PARAMS.bcast) == t
    for d, t in kat["inverse"]:
        assert PM.inverse_time(d, PARAMS.inverse) == t
    assert PM.nct_threshold(PARAMS.inverse, PARAMS.bcast) == kat["nct_threshold"]
    lf = PM.fit_linear([PM.BenchSample(int(s), t) for s, t in kat["fit_linear"]["samples"]])
    assert lf.alpha == pytest.approx(kat["fit_linear"]["alpha"], rel=1e-9)
    assert lf.beta == pytest.approx(kat["fit_linear"]["beta"], rel=1e-9)
    assert lf.r_squared == pytest.approx(kat["fit_linear"]["r_squared"], rel=1e-12)
    ef = PM.fit_exponential([PM.BenchSample(int(s), t) for s, t in kat["fit_exponential"]["samples"]])
    assert ef.alpha_inv == pytest.approx(kat["fit_exponential"]["alpha_inv"], rel=1e-9)
    assert ef.beta_inv == pytest.approx(kat["fit_exponential"]["beta_inv"], rel=1e-9)


def test_params_file_round_trip(tmp_path):
    path = tmp_path / "x.params"
    PM.write_params(path, PARAMS)
    assert PM.read_params(path) == PARAMS
    assert PM.read_params(path) == PM.SYNTHETIC_IB_PARAMS  # bundled calibration == reference data file
    (tmp_path / "bad.params").write_text("alpha_ar 1\nalpha_ar 2\n")
    with pytest.raises(ValueError, match="duplicate"):
        PM.read_params(tmp_path / "bad.params")


def test_bench_csv_round_trip(tmp_path):
    s = [PM.BenchSample(10, 0.5), PM.BenchSample(20, 0.25)]
    PM.write_bench_csv(tmp_path / "b.csv", s)
    assert PM.read_bench_csv(tmp_path / "b.csv") == s


# --- restated reference unit tests (pkg/tests/test_planner.py) -------------

def test_lbp_traces():
    assert P.lbp_place(inv_tasks([4, 3, 2, 1]), 2, *ALL_CT).workers == ((0,), (1, 2, 3))
    assert P.lbp_place(inv_tasks([4, 3, 2, 1]), 2, *ALL_CT, balance="dim").workers == ((0, 3), (1, 2))
    assert P.lbp_place(inv_tasks([64] * 4), 2, *ALL_CT).workers == ((0, 2), (1, 3))
    one = P.lbp_place(inv_tasks([4, 3, 2]), 1, *ALL_CT)
    assert one.workers == ((0, 1, 2),) and one.nct == {0, 1, 2}


def test_lbp_nct_replicated():
    plan = P.lbp_place(inv_tasks([8, 8, 200]), 3, PM.InverseParams(1e-4, 0.05), PM.BcastParams(0.1, 1e-9))
    assert {0, 1} <= plan.nct and 2 not in plan.nct
    assert all(0 in w and 1 in w for w in plan.workers)


def test_lbp_errors():
    with pytest.raises(ValueError, match="world_size"):
        P.lbp_place(inv_tasks([4]), 0, *ALL_CT)
    with pytest.raises(ValueError, match="no inversion tasks"):
        P.lbp_place([], 2, *ALL_CT)
    with pytest.raises(ValueError, match="balance"):
        P.lbp_place(inv_tasks([4]), 2, *ALL_CT, balance="cubic")


def test_seq_and_local():
    assert P.seq_place(inv_tasks([5, 6, 7, 8]), 2).workers == ((0, 2), (1, 3))
    assert P.seq_place(inv_tasks([5, 6]), 4).workers == ((0,), (1,), (), ())
    assert P.local_place(inv_tasks([5, 6]), 2).nct == {0, 1}


def test_plan_invariants():
    t = tuple(inv_tasks([4, 5]))
    with pytest.raises(ValueError, match="more than one worker"):
        P.PlacementPlan(t, ((0, 1), (0,)), frozenset())
    with pytest.raises(ValueError, match="missing from worker"):
        P.PlacementPlan(t, ((0, 1), ()), frozenset({0}))
    with pytest.raises(ValueError, match="does not cover"):
        P.PlacementPlan(t, ((0,), ()), frozenset())


def test_fusion_semantics():
    ar = PM.AllReduceParams(1e-3, 1e-9)
    assert [len(g) for g in P.plan_fusion(fwd_tasks([.1, .2, .3]), [.1] * 3, ar, P.FusionPolicy.LAYERWISE).groups] == [1, 1, 1]
    assert [len(g) for g in P.plan_fusion(fwd_tasks([.1, .2, .3]), [.1] * 3, ar, P.FusionPolicy.NAIVE).groups] == [3]
    zero = PM.AllReduceParams(0.0, 1e-9)
    assert [len(g) for g in P.plan_fusion(fwd_tasks([.1] * 4), [.1] * 4, zero, P.FusionPolicy.OPTIMAL).groups] == [1] * 4
    t3 = fwd_tasks([.1] * 3, [512] * 3)
    assert [len(g) for g in P.plan_fusion(t3, [.1] * 3, ar, P.FusionPolicy.THRESHOLD, threshold_bytes=2 ** 20).groups] == [1, 1, 1]
    assert [len(g) for g in P.plan_fusion(t3, [.1] * 3, ar, P.FusionPolicy.THRESHOLD).groups] == [3]
    plan = P.plan_fusion(fwd_tasks([0.5, 0.2, 2.0, 2.0], [13, 13, 19, 2]), [0.2, 0.9, 0.5, 0.5],
                         PM.AllReduceParams(1.0, 0.01), P.FusionPolicy.OPTIMAL)
    assert [[t.layer_index for t in g] for g in plan.groups] == [[1, 2], [3], [4]]


def test_fusion_errors():
    ar = PM.AllReduceParams(1e-3, 1e-9)
    with pytest.raises(ValueError, match="no factor tasks"):
        P.plan_fusion([], [], ar, P.FusionPolicy.NAIVE)
    with pytest.raises(ValueError, match="boundary"):
        P.plan_fusion([P.FactorTask(1, P.FactorKind.A, 2, .1), P.FactorTask(1, P.FactorKind.G, 2, .1)], [.1, .1], ar,
                      P.FusionPolicy.NAIVE)
    with pytest.raises(ValueError, match="forward order"):
        P.plan_fusion([P.FactorTask(2, P.FactorKind.A, 2, .1), P.FactorTask(1, P.FactorKind.A, 2, .1)], [.1, .1], ar,
                      P.FusionPolicy.NAIVE)


def test_greedy_within_four_thirds():
    rng = np.random.default_rng(31)

    def brute(loads, p):
        best = [sum(loads)]
        b = [0.0] * p

        def go(i):
            if i == len(loads):
                best[0] = min(best[0], max(b))
                return
            for q in range(p):
                b[q] += loads[i]
                if b[q] < best[0]:
                    go(i + 1)
                b[q] -= loads[i]
        go(0)
        return best[0]

    for _ in range(20):
        n, p = int(rng.integers(2, 8)), int(rng.integers(2, 4))
        dims = rng.integers(1, 40, n).tolist()
        plan = P.lbp_place(inv_tasks(dims), p, *ALL_CT)
        got = max(sum(plan.tasks[i].dim ** 2 for i in w) for w in plan.workers)
        assert got <= 4 / 3 * brute([d * d for d in dims], p) + 1e-9


def test_imbalance_report_resnet50_p8():
    # the d^2 floor at P=8 with whole-tensor LBP is 10.4%
    plan = P.lbp_place(P.inverse_tasks(layers("resnet50")), 8, *ALL_CT)
    rep = P.placement_imbalance(plan, weight=lambda d: float(d) ** 2)
    assert rep["max_over_mean_minus_1"] == pytest.approx(0.104, abs=2e-3)
    assert rep["makespan_over_lower_bound"] == pytest.approx(1.0, abs=1e-9)


def test_inversion_groups_partition_and_order():
    """schedule.inversion_groups: A + early G groups (backward order, cut at the cumulative
    sum-g^3 fractions) + the tail G group partition the 2L tensors."""
    from paper_2107_06533_b200.schedule import inversion_groups
    from paper_2107_06533_b200.workloads import layer_shapes
    sh = layer_shapes("resnet50", 32)
    a, g = [s[2] for s in sh], [s[3] for s in sh]
    r = inversion_groups(a, g, (0.85, 0.983, 0.9985))
    assert r["early"] == ["G1", "G2", "G3"] and r["tail"] == "G4" and r["n_g"] == [15, 15, 14, 10]
    sets = [r["A"]] + [r[k] for k in r["early"] + [r["tail"]]]
    assert sum(len(x) for x in sets) == 2 * len(sh) and set().union(*sets) == set(range(2 * len(sh)))
    # backward order: every member of an earlier group belongs to a later layer
    for e, f in zip(r["early"], r["early"][1:] + [r["tail"]]):
        assert min(r[e]) > max(r[f])
    # the tail holds only layer1 / conv1 output factors (g <= 256): a short inversion chain after backward
    assert max(g[t // 2] for t in r[r["tail"]]) == 256
    # single fraction == the two-group split
    r1 = inversion_groups(a, g, 0.85)
    assert r1["early"] == ["G1"] and r1["G1"] == r["G1"] and r1["n_g"] == [15, 39]
    with pytest.raises(ValueError):
        inversion_groups(a, g, (0.9, 0.8))


def test_lbp_dim_cube_balances_inversion_work():
    """balance="dim_cube" (extension): Algorithm 1 with d^3 bucket weights; on ResNet-50 it
    balances the inversion arithmetic exactly at P = 2, 4 and reaches the indivisible-task
    lower bound (one d = 4608 inverse per rank) at P = 8; d^2 stays the reference default."""
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.perfmodel import default_params
    from paper_2107_06533_b200.workloads import layer_shapes
    specs = [SPDKFAC._estimate_times(n, a, g) for n, m, a, g in layer_shapes("resnet50", 32)]
    tasks = P.inverse_tasks(specs)
    perf = default_params()
    for w, tol in ((2, 0.01), (4, 0.01)):
        r = P.placement_imbalance(P.lbp_place(tasks, w, perf.inverse, perf.bcast, balance="dim_cube"))
        assert r["max_over_mean_minus_1"] <= tol
        r2 = P.placement_imbalance(P.lbp_place(tasks, w, perf.inverse, perf.bcast, balance="dim_sq"))
        assert r2["max_over_mean_minus_1"] > 0.1  # the d^2 weights leave > 10 % on the table here
    r = P.placement_imbalance(P.lbp_place(tasks, 8, perf.inverse, perf.bcast, balance="dim_cube"))
    assert abs(r["makespan_over_lower_bound"] - 1.0) < 1e-9
    with pytest.raises(ValueError):
        P.lbp_place(tasks, 2, perf.inverse, perf.bcast, balance="dim_4")


def test_bert_base_linear_shapes():
    """configs[4]: the synthetic BERT-base linear stack has BERT-base's 72 encoder linears
    (q/k/v/o 768x768, ffn 768->3072->768) at bs32 x seq128 = 4096 rows, plus the classifier."""
    from collections import Counter
    from paper_2107_06533_b200.workloads import layer_shapes
    s = layer_shapes("bert_base_linears", 32)
    assert len(s) == 73
    assert Counter((m, a, g) for _, m, a, g in s[:-1]) == Counter(
        {(4096, 768, 768): 48, (4096, 768, 3072): 12, (4096, 3072, 768): 12})
    assert s[-1][1:] == (32, 768, 1000)


def test_marginal_inverse_model_makes_small_factors_nct(tmp_path):
    """B200 extension: the batched-inversion marginal model c3 d^3 against the
    marginal broadcast beta d(d+1)/2 gives a nonzero NCT set; the params file round-trips with the
    extension keys and reference-format files still read."""
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.workloads import layer_shapes
    bc = PM.BcastParams(1.7e-5, 7.3e-12)          # NCCL broadcast fit (P = 2)
    marg = PM.MarginalInverseParams(1.6e-14)       # ~7 ms for the 108 ResNet-50 factors in one plan
    thr = PM.nct_threshold(marg, bc)
    assert thr is not None and 100 < thr < 1000
    assert PM.nct_threshold(PM.InverseParams(1.36e-4, 9.2e-4), bc) == 1  # exponential: nothing NCT
    specs = [SPDKFAC._estimate_times(n, a, g) for n, m, a, g in layer_shapes("resnet50", 32)]
    tasks = P.inverse_tasks(specs)
    for w in (2, 4, 8):
        plan = P.lbp_place(tasks, w, marg, bc, balance="dim_cube")
        dims = {t.tensor_index: t.dim for t in tasks}
        assert plan.nct and all(dims[i] < thr for i in plan.nct) and all(dims[i] >= thr for i in dims if i not in plan.nct)
    params = PM.PerfParams(PM.AllReduceParams(2e-5, 8e-12), bc, PM.InverseParams(1.36e-4, 9.2e-4), 4, marg)
    path = tmp_path / "b200_p4.params"
    PM.write_params(path, params)
    back = PM.read_params(path)
    assert back.marginal == marg and back.placement_inverse == marg and back.fitted_world_size == 4
    ref = tmp_path / "ref.params"
    PM.write_params(ref, PM.PerfParams(params.allreduce, bc, params.inverse, 2))
    assert PM.read_params(ref).marginal is None and PM.read_params(ref).placement_inverse == params.inverse
    bad = tmp_path / "bad.params"
    bad.write_text(ref.read_text() + "inverse_model cubic\n")
    with pytest.raises(ValueError):
        PM.read_params(bad)
