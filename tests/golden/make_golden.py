"""Generate the golden fixtures under tests/golden/ by importing the reference.

Run in the dev container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (all committed, small):
  aggregated_step_w4.json  the reference's frozen step fixture (verbatim data,
                           pkg/tests/data/aggregated_step_w4.json)
  linalg_golden.npz        reference outputs of compute_factor_A/G,
                           damped_inverse, precondition, pack_upper on seeded
                           inputs (float64)
  plans.json               reference plan_fusion / lbp_place / seq_place /
                           local_place outputs on the bundled model profiles and
                           calibration, plus perf-model known answers
  profiles.json            per-layer (a_dim, g_dim, t_ff, t_bp, t_factorA,
                           t_factorG) of the bundled profiles
"""

from __future__ import annotations

import json
import pathlib
import shutil

import numpy as np

import kfacsched as K
from kfacsched import linalg as L
from kfacsched import simulator as S

HERE = pathlib.Path(__file__).parent
REF = pathlib.Path("/root/reference/pkg")


def linalg_golden():
    rng = np.random.default_rng(20260101)
    out = {}
    for b, d in [(1, 3), (7, 5), (32, 64), (64, 130), (9, 200)]:
        x = rng.standard_normal((b, d))
        out[f"fa_x_{b}_{d}"] = x
        out[f"fa_y_{b}_{d}"] = K.compute_factor_A(x).values
        out[f"fg_y_{b}_{d}"] = K.compute_factor_G(x).values
    for d, gamma in [(1, 0.5), (5, 0.0), (17, 0.01), (33, 0.1), (64, 0.1), (130, 0.05), (150, 0.2)]:
        b = rng.standard_normal((d, d))
        m = L.SymMatrix(b @ b.T / d + 0.1 * np.eye(d))
        out[f"inv_m_{d}"] = m.values
        out[f"inv_gamma_{d}"] = np.array(gamma)
        out[f"inv_y_{d}"] = K.damped_inverse(m, gamma).values
        out[f"pack_{d}"] = K.pack_upper(m)
    for dout, din in [(1, 1), (3, 5), (10, 64), (64, 147), (130, 70)]:
        g = rng.standard_normal((dout, din))
        ba = rng.standard_normal((din, din))
        bg = rng.standard_normal((dout, dout))
        a_inv = L.SymMatrix(ba @ ba.T / din + np.eye(din))
        g_inv = L.SymMatrix(bg @ bg.T / dout + np.eye(dout))
        out[f"pc_grad_{dout}_{din}"] = g
        out[f"pc_ainv_{dout}_{din}"] = a_inv.values
        out[f"pc_ginv_{dout}_{din}"] = g_inv.values
        out[f"pc_y_{dout}_{din}"] = K.precondition(g, a_inv, g_inv)
    np.savez_compressed(HERE / "linalg_golden.npz", **out)


def plans_golden():
    perf = K.bundled_params()
    res = {"params": {
        "alpha_ar": perf.allreduce.alpha_ar, "beta_ar": perf.allreduce.beta_ar,
        "alpha_bcast": perf.bcast.alpha_bcast, "beta_bcast": perf.bcast.beta_bcast,
        "alpha_inv": perf.inverse.alpha_inv, "beta_inv": perf.inverse.beta_inv,
        "fitted_world_size": perf.fitted_world_size}, "models": {}}
    for name in ("resnet50", "resnet152", "densenet201", "inceptionv4"):
        prof = K.bundled_profile(name)
        entry = {"fusion": {}, "placement": {}}
        for policy in K.FusionPolicy:
            cfg = S.SchemeConfig(scheme=S.Scheme.SPDKFAC, world_size=8, fusion_policy=policy,
                                 placement_mode="lbp", overlap_factor_comm=True)
            plans = S.build_plans(prof, cfg, perf)
            entry["fusion"][policy.value] = {
                "forward": [[[t.layer_index, t.kind.value] for t in g] for g in plans.forward_fusion.groups],
                "backward": [[[t.layer_index, t.kind.value] for t in g] for g in plans.backward_fusion.groups],
            }
        tasks = S.inverse_tasks(prof)
        for p in ((1, 2, 3, 4, 8, 16, 64) if name == "resnet50" else (1, 2, 4, 8)):
            for bal in ("dim_sq", "dim"):
                pl = K.lbp_place(tasks, p, perf.inverse, perf.bcast, balance=bal)
                entry["placement"][f"lbp_{p}_{bal}"] = {
                    "workers": [list(w) for w in pl.workers], "nct": sorted(pl.nct),
                    "makespan": K.placement_makespan(pl, perf.inverse, perf.bcast)}
            pl = K.seq_place(tasks, p)
            entry["placement"][f"seq_{p}"] = {"workers": [list(w) for w in pl.workers], "nct": sorted(pl.nct),
                                               "makespan": K.placement_makespan(pl, perf.inverse, perf.bcast)}
        res["models"][name] = entry
    # perf-model known answers
    kat = {"allreduce": [], "bcast": [], "inverse": [], "nct_threshold": None}
    for m in (0, 1, 2080, 10**6):
        kat["allreduce"].append([m, K.allreduce_time(m, perf.allreduce)])
    for d in (1, 64, 738, 4608):
        kat["bcast"].append([d, K.bcast_time(d, perf.bcast)])
        kat["inverse"].append([d, K.inverse_time(d, perf.inverse)])
    kat["nct_threshold"] = K.nct_threshold(perf.inverse, perf.bcast)
    samples = [K.BenchSample(s, 1e-4 + 2e-9 * s + (1e-6 if s % 3 else -1e-6)) for s in (10, 1000, 5000, 20000, 100000)]
    lf = K.fit_linear(samples)
    kat["fit_linear"] = {"samples": [[s.size, s.time] for s in samples], "alpha": lf.alpha, "beta": lf.beta,
                         "r_squared": lf.r_squared}
    es = [K.BenchSample(d, 2e-4 * np.exp(1.1e-3 * d) * (1.01 if d % 2 else 0.99)) for d in (64, 256, 1024, 2048, 4096)]
    ef = K.fit_exponential(es)
    kat["fit_exponential"] = {"samples": [[s.size, s.time] for s in es], "alpha_inv": ef.alpha_inv,
                              "beta_inv": ef.beta_inv}
    res["perfmodel_kat"] = kat
    (HERE / "plans.json").write_text(json.dumps(res, separators=(",", ":")) + "\n")


def profiles_golden():
    out = {}
    for name in ("resnet50", "resnet152", "densenet201", "inceptionv4"):
        prof = K.bundled_profile(name)
        out[name] = {"batch_size": prof.batch_size, "layers": [
            {"name": l.name, "a_dim": l.a_dim, "g_dim": l.g_dim, "t_ff": l.t_ff, "t_bp": l.t_bp,
             "t_factorA": l.t_factorA, "t_factorG": l.t_factorG} for l in prof.layers]}
    (HERE / "profiles.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    shutil.copyfile(REF / "tests/data/aggregated_step_w4.json", HERE / "aggregated_step_w4.json")
    linalg_golden()
    plans_golden()
    profiles_golden()
    print("golden fixtures written to", HERE)
