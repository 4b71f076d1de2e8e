#!/usr/bin/env python
"""SPD-KFAC iteration-time benchmark (BASELINE.json metric):

  "SPD-KFAC iteration time (ms) ResNet-50 bs32/GPU @1/2/4/8 B200; % roofline"

One step = one SPD-KFAC training iteration of torchvision ResNet-50 at batch 32
per GPU on synthetic 224x224 data: forward (A factors on a side stream), backward
(G factors, fused factor all-reduce per fusion group), gradient all-reduce,
load-balanced damped inverses + owner broadcast, preconditioning + weight update.
Factor and inverse update frequency 1 (every iteration does all of it).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Prints ONE JSON line on rank 0.  `value` = iteration ms (max over ranks, CUDA
events on the launching stream); `e2e` = the same through the public API with
the batch copied from pinned host memory and the loss read back every step;
`roofline` = the K-FAC kernel category with the largest live CUDA-event time in
the timed region (all categories in `roofline_kernels`, the SURVEY 8(d) iteration
roofline fraction in `iteration_roofline`); `cpu_baseline` = the reference's
float64 linear algebra on this host's cores for one full step of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

NPROC = os.cpu_count() or 1
for _k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_k, str(NPROC))

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPD-KFAC iteration time (ms) ResNet-50 bs32/GPU @1/2/4/8 B200; % roofline"
# scheme -> (fusion policy, placement) (simulator.py:145-193 SchemeConfig factories / ablation)
SCHEMES = {"spdkfac": ("optimal", "lbp"), "mpdkfac": ("naive", "seq"), "dkfac": ("naive", "local"),
           "spdkfac-nopipe": ("naive", "lbp"), "spdkfac-nolbp": ("optimal", "seq")}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--model", default="resnet50")
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--lr", type=float, default=0.01)
    p.add_argument("--damping", type=float, default=0.1)
    p.add_argument("--factor-freq", type=int, default=1)
    p.add_argument("--inv-freq", type=int, default=1)
    p.add_argument("--factor-decay", type=float, default=0.0,
                   help="running-average weight rho of the factors (0 = the reference's step)")
    p.add_argument("--placement", default="lbp")
    p.add_argument("--balance", choices=("dim_sq", "dim", "dim_cube"), default="dim_cube",
                   help="LBP bucket weight: d^2 / d (the reference's options) or d^3 (inversion arithmetic)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--profile", action="store_true", help="short run for ncu: no clocks/e2e/cpu legs")
    p.add_argument("--gc", choices=("freeze", "default"), default="freeze",
                   help="freeze: gc.freeze() after setup+warmup so generation-2 collections do not walk the "
                        "model/optimizer object graph mid-step")
    p.add_argument("--memory-format", choices=("channels_last", "nchw"), default="channels_last",
                   help="activation/weight memory format of the model (cuDNN runs NHWC natively on B200)")
    p.add_argument("--mode", choices=("graph", "eager"), default="graph",
                   help="graph: the whole step (fwd, bwd, K-FAC step) replayed as one CUDA graph")
    p.add_argument("--main-priority", type=int, default=-1,
                   help="CUDA priority of the forward/backward stream (negative = higher than the K-FAC side streams; "
                        "-1 measured 16.43/16.51 vs 16.70/16.56 ms for 0 at N=1)")
    p.add_argument("--trace", default=None,
                   help="diagnostic: torch.profiler (CUPTI) trace of 3 steps after the timed region; writes a "
                        "kernel-timeline summary JSON to this path")
    p.add_argument("--g-fractions", default="0.85,0.983,0.9985",
                   help="cumulative shares of the output-side inversion work (sum g^3) at which the early G "
                        "inversion groups are cut (comma list; the rest is inverted in step())")
    p.add_argument("--scheme", default="spdkfac",
                   choices=("spdkfac", "mpdkfac", "dkfac", "spdkfac-nopipe", "spdkfac-nolbp"),
                   help="measured baselines of simulator.py:145-193: dkfac = naive fusion + every worker inverts "
                        "everything; mpdkfac = naive fusion + round-robin placement; the ablations toggle the "
                        "pipelined (optimal) fusion and LBP separately")
    p.add_argument("--launch-groups", choices=("auto", "fusion", "inversion"), default="auto",
                   help="factor SYRK launch groups: the fusion plan (P>1 default) or few large groups (P=1 default)")
    p.add_argument("--update-in-backward", choices=("auto", "on", "off"), default="auto",
                   help="precondition + update the early G groups' layers during backward (auto: on at P=1)")
    p.add_argument("--ncu-range", action="store_true",
                   help="wrap the last timed step in cudaProfilerStart/Stop (ncu --profile-from-start off)")
    p.add_argument("--clocks", choices=("nvml", "smi", "off"), default="nvml")
    p.add_argument("--timeline", action="store_true", help="diagnostic: per-phase CUDA-event timeline of one eager step")
    p.add_argument("--stats-off", action="store_true", help="no per-launch CUDA events in the timed region (diagnostic)")
    p.add_argument("--perf-params", default=None,
                   help="planner cost-model file (perfmodel.read_params); default data/b200_p{N}.params")
    p.add_argument("--factor-comm", choices=("auto", "reduce", "allreduce", "peer"), default="auto",
                   help="P > 1 factor aggregation: 'peer' (each group's SYRK output pushed into the owner's inbox over "
                        "NVLink peer memory, owner-side sum), NCCL 'reduce' onto the owner, or 'allreduce'; auto follows "
                        "SPDKFAC_FACTOR_COMM, else peer (factor_decay 0, P <= 8) / allreduce")
    p.add_argument("--optimizer", choices=("spdkfac", "sgd"), default="spdkfac",
                   help="sgd = diagnostic floor (forward/backward + SGD, no K-FAC); never the headline")
    return p.parse_args(argv)


def make_optimizer(a, model, world):
    """The SPDKFAC configuration the bench times (also used by the config-level parity tests,
    tests/test_gpu_config_parity.py, so the checked step IS the measured step)."""
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.planner import FusionPolicy
    fusion, placement = SCHEMES[a.scheme]
    if a.scheme == "spdkfac":
        placement = a.placement
    perf = None
    if getattr(a, "perf_params", None):
        from paper_2107_06533_b200.perfmodel import read_params
        perf = read_params(a.perf_params)
    return SPDKFAC(model, lr=a.lr, damping=a.damping, factor_update_freq=a.factor_freq, perf=perf,
                   factor_decay=getattr(a, "factor_decay", 0.0), factor_comm=getattr(a, "factor_comm", "auto"),
                   inv_update_freq=a.inv_freq, placement=placement, balance=a.balance,
                   fusion=FusionPolicy(fusion),
                   early_g_fraction=tuple(float(f) for f in a.g_fractions.split(",")), launch_groups=a.launch_groups,
                   update_in_backward=a.update_in_backward == "on" or (a.update_in_backward == "auto" and world == 1))


def launch_groups_of(a, world):
    """The optimizer's resolved launch groups (SPDKFAC auto rule) for the bench line."""
    if a.launch_groups != "auto":
        return a.launch_groups
    fc = a.factor_comm if a.factor_comm != "auto" else os.environ.get(
        "SPDKFAC_FACTOR_COMM", ("peer" if world <= 8 else "reduce") if a.factor_decay == 0 else "allreduce")
    return "inversion" if world == 1 or (world == 2 and fc == "peer" and SCHEMES[a.scheme][0] == "optimal") else "fusion"


def workload_config(a, world):
    idx = {"resnet20": "0", "resnet50": "1" if world == 1 else "2", "densenet201": "3",
           "bert_base_linears": "4", "inceptionv4": "4"}.get(a.model)
    data = {"resnet20": "32x32", "bert_base_linears": "seq128 x 768 token embeddings",
            "inceptionv4": "299x299"}.get(a.model, "224x224")
    return {"workload": f"{a.model} SPD-KFAC bs{a.batch}/GPU synthetic {data}"
                        + (f" (BASELINE.json configs[{idx}])" if idx else " (not a BASELINE.json config)"),
            "per_gpu_batch": a.batch, "global_batch": a.batch * world, "damping": a.damping, "lr": a.lr,
            "factor_update_freq": a.factor_freq, "inv_update_freq": a.inv_freq, "factor_decay": a.factor_decay,
            "scheme": a.scheme,
            "fusion": (SCHEMES[a.scheme][0] if launch_groups_of(a, world) == "fusion" else
                       "SYRK / aggregation launch groups = A in 2 halves, G at the inversion groups"
                       + (" (P=1: no factor comm)" if world == 1 else " (peer aggregation, P=2)")),
            "g_inversion_fractions": a.g_fractions,
            "update_in_backward": a.update_in_backward == "on" or (a.update_in_backward == "auto" and world == 1),
            "placement": SCHEMES[a.scheme][1] if a.scheme != "spdkfac" else a.placement, "lbp_balance": a.balance, "parallelism": f"dp{world}", "python_gc": a.gc,
            "execution": (f"one CUDA graph per iteration (fwd+bwd+{'K-FAC' if a.optimizer == 'spdkfac' else 'SGD'} step)"
                          if a.mode == "graph" else "eager"),
            "memory_format": a.memory_format,
            "main_stream_priority": a.main_priority,
            "factor_comm": (None if world == 1 else
                            (a.factor_comm if a.factor_comm != "auto" else
                             os.environ.get("SPDKFAC_FACTOR_COMM", ("peer" if world <= 8 else "reduce")
                                            if a.factor_decay == 0 else "allreduce"))),
            "l2": "per-iteration working set (activations, 0.3 GB packed factors, im2col staging) >> 126 MB L2; no flush"}


# ---------------------------------------------------------------- clocks
class NvmlClocks:
    """Clock / throttle-reason sampler on a background thread via NVML (light queries only;
    an `nvidia-smi -lms` loop with power/reason fields stalled the GPU ~50-100 ms per sample)."""

    def __init__(self, index: int, period_s: float = 0.1):
        import threading
        import pynvml as N
        self.N = N
        N.nvmlInit()
        self.h = N.nvmlDeviceGetHandleByIndex(index)
        self.max = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        self.samples = []
        self.stop_ev = threading.Event()
        self.period = period_s
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        N = self.N
        while not self.stop_ev.is_set():
            self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                 N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            self.stop_ev.wait(self.period)

    def stop(self):
        self.stop_ev.set()
        self.t.join()
        N = self.N
        bits = {"hw_slowdown": getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        reasons = sorted({k for _, r in self.samples for k, b in bits.items() if r & b})
        sm = [c for c, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max, "reasons": reasons,
                "samples": len(sm), "source": "nvml"}


class Clocks:
    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU reference
def cpu_reference(model, batch, steps=1, warmup=0):
    """Time the reference's float64 K-FAC algebra (oracle/cpu_step.py) for `steps` full steps; each
    step times every layer of the model (each its own call).  Warm-up runs the
    smallest shape (BLAS thread pool, first-touch pages), not a full step."""
    from oracle import cpu_step
    from paper_2107_06533_b200.workloads import layer_shapes
    shapes = layer_shapes(model, batch)
    keys = list(cpu_step.distinct_shapes(shapes))
    small = min(keys, key=lambda k: k[0] * (k[1] + k[2]) + k[1] ** 3 + k[2] ** 3)
    for _ in range(warmup):
        cpu_step.time_layer(*small)
    cache = {}
    # full steps until `steps` are done or the wall budget is spent (at least one): every reported step is a
    # whole step actually timed, and the arm still ends within a few minutes at the driver's K
    budget = float(os.environ.get("SPDKFAC_REF_BUDGET_S", "240"))
    t_start, per_step = time.perf_counter(), []
    while len(per_step) < max(1, steps):
        per_step.append(cpu_step.full_step(shapes, cache=cache))
        if time.perf_counter() - t_start > budget:
            break
    kind = cpu_step.implementation()[4]
    sample = (f"full step per timed step: all {len(shapes)} {model} K-FAC layers (bs{batch}; {len(keys)} distinct "
              f"shapes), each layer's factor A+G, 2 damped inverses, precondition and update timed (float64 "
              f"numpy/scipy LAPACK); im2col and forward/backward not charged; host CPU {cpu_step.cpu_model()}")
    return statistics.mean(per_step) * 1e3, sample, per_step, kind


# ---------------------------------------------------------------- diagnostics
def trace_summary(step, path, torch, n=3, comm_tags=None):
    """CUPTI kernel timeline of n steps: GPU busy union per step, per-stream busy, top kernels,
    and the six-category breakdown of the last step (breakdown.py) next to `path`."""
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(n):
            torch.cuda._sleep(1000)  # step delimiter kernel (outside the graph)
            step(i)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", 0)) for e in evs))
    if path is None:
        return
    marks = [k for k in ks if "spin_kernel" in k[2] or "sleep" in k[2].lower()]
    if len(marks) >= n:
        from paper_2107_06533_b200 import breakdown as BD
        w0 = marks[-1][1]
        last = [(s0, e0, nm, sid) for s0, e0, nm, sid in ks if s0 >= w0]
        if comm_tags is None or sum(BD.is_nccl(k[2]) for k in last) != len(comm_tags):
            comm_tags = ["inverse" if "broadcast" in k[2].lower() else "factor" for k in last if BD.is_nccl(k[2])]
        lab = BD.label_events(last, comm_tags)
        tot = BD.breakdown(lab, start=w0)
        base = os.path.splitext(path)[0]
        open(base + "_breakdown.csv", "w").write(BD.breakdown_to_csv({k: v * 1e-6 for k, v in tot.items()}))
        open(base + "_timeline.csv", "w").write(BD.timeline_to_csv([(s0 * 1e-6, e0 * 1e-6, nm, sid, c)
                                                                    for s0, e0, nm, sid, c in lab], t0=w0 * 1e-6))
    ks = [k for k in ks if k not in marks]
    if not ks:
        json.dump({"error": "no CUDA events"}, open(path, "w"))
        return
    t0, t1 = ks[0][0], max(k[1] for k in ks)
    busy, cur_s, cur_e = 0.0, None, None
    for s0, e0, _, _ in ks:
        if cur_e is None or s0 > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s0, e0
        else:
            cur_e = max(cur_e, e0)
    busy += cur_e - cur_s
    per_name, per_stream = {}, {}
    for s0, e0, nm, sid in ks:
        key = nm[:90]
        c = per_name.setdefault(key, [0.0, 0])
        c[0] += e0 - s0
        c[1] += 1
        per_stream[str(sid)] = per_stream.get(str(sid), 0.0) + (e0 - s0)
    top = sorted(per_name.items(), key=lambda kv: -kv[1][0])[:40]
    # phase windows of the LAST traced step (from its first kernel), by kernel family
    import re
    fam = {"fwd_bwd (cudnn/cutlass/aten)": r"cudnn|cutlass3x|sm80_xmma|at::native|Memset|max_pool",
           "factor stage": r"stage_rows|stage_im2col|stage_spatial", "factor syrk": r"tc3_gemm_kernel<\(spd::Kind\)1, 3|tc3_pair",
           "factor reduce": r"reduce_pack", "inv pivot": r"pivot_kernel|pivot_tc_kernel<false>", "inv update": r"Kind\)2, 3, true",
           "precond": r"split_rows_batched|apply_update|Kind\)2, 3, false, 4", "inv panel": r"stage_panel|Kind\)2, 3, false, 0",
           "inv unpack/finalize": r"damp_unpack|finalize_kernel|small_inverse|pivot_tc_kernel<true>", "nccl": r"nccl",
           "pack/unpack": r"pack_upper|unpack_upper"}
    step_len = (t1 - t0) / n
    last0 = t0 + (n - 1) * step_len
    phases = {}
    for s0, e0, nm, sid in ks:
        if s0 < last0:
            continue
        for f, rx in fam.items():
            if re.search(rx, nm):
                w = phases.setdefault(f"{f} @stream{sid}", [s0, e0, 0.0])
                w[0], w[1], w[2] = min(w[0], s0), max(w[1], e0), w[2] + (e0 - s0)
                break
    phases = {f: {"first_ms": round((w[0] - last0) / 1e3, 3), "last_ms": round((w[1] - last0) / 1e3, 3),
                  "busy_ms": round(w[2] / 1e3, 3)} for f, w in sorted(phases.items(), key=lambda kv: kv[1][1])
              if w[2] > 20.0}
    out = {"steps": n, "span_ms_per_step": (t1 - t0) / 1e3 / n, "gpu_busy_union_ms_per_step": busy / 1e3 / n,
           "kernel_sum_ms_per_step": sum(v[0] for v in per_name.values()) / 1e3 / n,
           "per_stream_ms_per_step": {k: v / 1e3 / n for k, v in sorted(per_stream.items(), key=lambda kv: -kv[1])},
           "last_step_phases": phases,
           "top": [{"name": k, "ms_per_step": v[0] / 1e3 / n, "count_per_step": v[1] / n} for k, v in top]}
    json.dump(out, open(path, "w"), indent=1)


# ---------------------------------------------------------------- rooflines
# K-FAC kernel categories timed live in the timed region (libspdkfac stats categories)
ROOF_CATS = ("factor_stage", "factor_syrk", "inv_pivot", "inv_panel", "inv_update", "precond_gemm")
# bound and peak of each category: the tensor-core contractions against the measured GEMM peak of
# the MMA kind they issue (bf16 for the factor SYRK, f16 for the inverse panel / update, tf32 for the
# preconditioning),
# the staging pass against HBM
_INV_PEAK = "tf32_tflops" if os.environ.get("SPDKFAC_INV_TF32") == "1" else "bf16_tflops_sustained"
_INV_KIND = "TF32" if os.environ.get("SPDKFAC_INV_TF32") == "1" else "F16"
_PREC_PEAK = "bf16_tflops_sustained" if os.environ.get("SPDKFAC_PRECOND_F16") == "1" else "tf32_tflops"
_PREC_KIND = "F16 row-scaled" if os.environ.get("SPDKFAC_PRECOND_F16") == "1" else "TF32"
_ROOF_SPEC = {"factor_syrk": ("tensor", "bf16_tflops_sustained"),
              "inv_pivot": ("fp32", "fp32_ffma_tflops") if os.environ.get("SPDKFAC_PIVOT") != "tc" else ("tensor", "tf32_tflops"),
              # the inverse panel / update issue kind::f16 MMAs on scaled fp16 planes (SPDKFAC_INV_TF32=1: tf32)
              "inv_panel": ("tensor", _INV_PEAK), "inv_update": ("tensor", _INV_PEAK),
              "precond_gemm": ("tensor", _PREC_PEAK), "factor_stage": ("hbm", "hbm_gbs")}
_KERNEL_NAMES = {"factor_syrk": "tc3_gemm_kernel<BF16> + tc3_pair_kernel (factor SYRK, 3 x bf16, tcgen05)",
                 "inv_pivot": ("pivot_kernel (128-pivot block: 16 pipelined 8-pivot sweeps, rank-8 updates on FFMA2)"
                               if os.environ.get("SPDKFAC_PIVOT") != "tc" else
                               "pivot_tc_kernel<false> (128-pivot block: warp sweeps + rank-32 tcgen05 updates)"),
                 "inv_panel": f"stage_panel_kernel + tc3_gemm_kernel<{_INV_KIND}> (inverse panel C = W[:,K] P^-1)",
                 "inv_update": f"tc3_gemm_kernel<{_INV_KIND}, C-tile> (inverse trailing update, 3 x {_INV_KIND.lower()}"
                               + (" planes scaled per matrix)" if _INV_KIND == "F16" else ")"),
                 "precond_gemm": f"tc3_gemm_kernel<{_PREC_KIND}, chunked accumulation> (G^-1 grad A^-1, W -= lr P)",
                 "factor_stage": "stage_rows / stage_im2col / stage_spatial (fp32 -> bf16 hi/lo planes)"}


def torch_sm_count():
    try:
        import torch
        return torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        return None


def kernel_roofline(cat, rec, per, peaks, world, model):
    """Roofline of one kernel category from its live CUDA-event time and the algorithmic work the
    library declares per launch (flops: SURVEY 8(d) per-unit figures x units; bytes: staging)."""
    bound, peak_key = _ROOF_SPEC[cat]
    ms = rec["ms"] / per
    launches = rec["launches"] / per
    work = rec["bytes"] / per if bound == "hbm" else rec["flops"] / per
    ach = (work / (ms * 1e-3)) / (1e9 if bound == "hbm" else 1e12) if ms > 0 else 0.0
    peak = peaks.get(peak_key)
    out = {"kernel": _KERNEL_NAMES[cat], "category": cat, "bound": bound, "achieved": round(ach, 2),
           "peak": round(peak, 1) if peak else None, "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
           "frac": round(ach / peak, 4) if peak and ms > 0 else None, "peak_source": peak_key + (
               " (MEASURED_PEAKS.json)" if peak_key in ("hbm_gbs", "bf16_tflops_sustained") else " (measured by this run)"),
           "kernel_ms_per_step": round(ms, 4), "launches_per_step": launches,
           "timing": "in-kernel launch probes (first CTA start to last CTA end, %globaltimer) over the timed region's "
                     "last step (graph mode) or all timed steps (eager)",
           ("algorithmic_bytes_per_step" if bound == "hbm" else "algorithmic_flops_per_step"): work,
           "traffic": None}
    if cat == "inv_pivot" and peak and ms > 0 and launches > 0:
        # one CTA (one SM) per active 128-block: the kernel is a latency chain that occupies few SMs, so also
        # report the fraction of the FFMA rate of the SMs it actually holds (2*128^3 flop per CTA)
        ctas = (work / launches) / (2.0 * 128 ** 3)
        sms = torch_sm_count()
        out["ctas_per_launch"] = round(ctas, 1)
        out["frac_of_occupied_sms"] = round(ach / (peak * min(1.0, ctas / sms)), 4) if sms else None
    try:  # DRAM bytes per launch from a committed `ncu --set full` capture of the same launches
        t = json.load(open(os.path.join(ROOT, "profiles", f"traffic_{model}_n{world}.json")))[cat]
        out["traffic"] = round(t["dram_bytes_per_step"] / max(launches, 1e-9))
        out["traffic_per_step"] = t["dram_bytes_per_step"]
        out["traffic_source"] = t.get("source")
    except Exception:
        out["traffic_source"] = "no committed ncu capture for this category/config"
    return out


def iteration_roof(bst, nb, peaks, ffbp_flops, ms):
    """iteration roofline time = sum over the step's work of max(F / peak, B / BW);
    fraction = that / measured iteration time.  K-FAC categories from the library's declared
    algorithmic work (per-launch event pass), forward/backward from torch's FLOP counter at the
    TF32 GEMM peak (the convolutions run TF32), communication not included (N = 1: none)."""
    tf32, bf16, hbm = peaks.get("tf32_tflops"), peaks.get("bf16_tflops_sustained"), peaks.get("hbm_gbs")
    if not (tf32 and bf16 and hbm):
        return None
    parts = {}
    for cat, rec in bst.items():
        if not isinstance(rec, dict) or not (rec["flops"] or rec["bytes"]):
            continue
        pk = bf16 if cat == "factor_syrk" else (peaks.get("fp32_ffma_tflops") or tf32) if cat in ("inv_pivot", "inv_small") \
            and os.environ.get("SPDKFAC_PIVOT") != "tc" else tf32
        parts[cat] = max(rec["flops"] / nb / (pk * 1e12), rec["bytes"] / nb / (hbm * 1e9)) * 1e3
    if ffbp_flops:
        parts["forward_backward"] = ffbp_flops / (tf32 * 1e12) * 1e3
    t = sum(parts.values())
    return {"roofline_ms": round(t, 4), "measured_ms": round(ms, 4), "frac": round(t / ms, 4) if ms else None,
            "parts_ms": {k: round(v, 4) for k, v in parts.items()}, "ffbp_flops_per_step": ffbp_flops,
            "peaks": {"tf32_tflops": tf32, "bf16_tflops_sustained": bf16, "hbm_gbs": hbm}}


def measure_peaks(torch, dev, world):
    """FP32 (cuBLAS SGEMM: FFMA) and TF32 (cuBLAS, tensor cores) GEMM peaks on this GPU, the way
    MEASURED_PEAKS.json measures bf16 (8192^3, best of several, CUDA events); at N > 1 the NCCL
    all-reduce bus bandwidth of a 256 MiB fp32 buffer (max over ranks)."""
    out = {}
    n = 8192
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    old = torch.backends.cuda.matmul.allow_tf32
    try:
        for name, tf32, reps in (("fp32_ffma_tflops", False, 3), ("tf32_tflops", True, 6)):
            torch.backends.cuda.matmul.allow_tf32 = tf32
            torch.matmul(a, b)
            torch.cuda.synchronize()
            best = float("inf")
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(a, b)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            out[name] = round(2.0 * n ** 3 / (best * 1e-3) / 1e12, 1)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    del a, b
    out["how"] = "cuBLAS fp32 matmul 8192^3 with TF32 off (FFMA) / on (tf32 tensor cores), best of 3 / 6"
    if world > 1:
        import torch.distributed as dist
        buf = torch.ones(64 << 20, device=dev)  # 256 MiB
        for _ in range(3):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(5):
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dist.all_reduce(buf)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = min(best, float(t.item()))
        nbytes = buf.numel() * 4
        out["nccl_allreduce_busbw_gbs"] = round(2.0 * (world - 1) / world * nbytes / (best * 1e-3) / 1e9, 1)
        out["nccl_allreduce_bytes"] = nbytes
        del buf
    return out


def count_ffbp_flops(torch, model, crit, x, y):
    """Forward + backward FLOPs of one step (torch.utils.flop_counter; convolutions and matmuls)."""
    try:
        from torch.utils.flop_counter import FlopCounterMode
        with FlopCounterMode(display=False) as fc:
            crit(model(x), y).backward()
        model.zero_grad(set_to_none=True)
        return int(fc.get_total_flops())
    except Exception:
        return None


# ---------------------------------------------------------------- our arm
def run_ours(a):
    import torch
    import torch.distributed as dist
    import torch.nn as nn

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cudnn.benchmark = True

    from paper_2107_06533_b200 import _lib
    from paper_2107_06533_b200.optimizer import SPDKFAC
    from paper_2107_06533_b200.workloads import build_model, input_shape, num_classes

    measured_peaks = measure_peaks(torch, dev, world) if not a.profile else None
    torch.manual_seed(0)
    model = build_model(a.model).to(dev)
    cl = a.memory_format == "channels_last" and len(input_shape(a.model, 1)) == 4
    if cl:
        model = model.to(memory_format=torch.channels_last)
    ffbp_flops = None
    if not a.profile:  # before the optimizer exists: its hooks would capture this pass
        xf = torch.randn(input_shape(a.model, a.batch), device=dev)
        xf = xf.contiguous(memory_format=torch.channels_last) if cl else xf
        ffbp_flops = count_ffbp_flops(torch, model, nn.CrossEntropyLoss(), xf,
                                      torch.zeros(a.batch, dtype=torch.long, device=dev))
        del xf
    if a.optimizer == "sgd":
        opt = torch.optim.SGD(model.parameters(), lr=a.lr)
        opt.check_inverses = lambda: None
        opt.placement = None
    else:
        opt = make_optimizer(a, model, world)
        peer = getattr(opt, "_peer", None)
        if peer is not None and measured_peaks is not None:
            # NVLink evidence for the peer-memory factor aggregation: every rank pushes one fusion-buffer-sized
            # range into the next rank's inbox row (copy engine, all ranks at once), before any step writes
            # or reads those rows; plus the bytes the step pushes (CT factors owned by another rank)
            import torch.distributed as dist
            src = opt.bufA
            dst = peer.remote_ptr((rank + 1) % world, "A", 0)
            cs_ = torch.cuda.Stream()
            best = float("inf")
            for it in range(4):
                dist.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cs_)
                _lib.check(_lib.load().spdkfac_peer_copy(dst, src.data_ptr(), src.numel() * 4, cs_.cuda_stream),
                           "peer copy")
                e1.record(cs_)
                torch.cuda.synchronize()
                t = torch.tensor([e0.elapsed_time(e1)], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                if it:
                    best = min(best, float(t.item()))
            pushed = sum(e - s_ for k in ("A", "G") for segs in opt._peer_out[k] for s_, e, _ in segs) * 4
            measured_peaks["peer_push_gbs_per_gpu"] = round(src.numel() * 4 / (best * 1e-3) / 1e9, 1)
            measured_peaks["peer_push_test_bytes"] = src.numel() * 4
            measured_peaks["peer_push_bytes_per_step_per_gpu"] = pushed
            measured_peaks["peer_push_how"] = ("cudaMemcpyAsync into the next rank's CUDA-IPC inbox (copy engine), all "
                                               "ranks concurrently, max over ranks, best of 3")
    crit = nn.CrossEntropyLoss()
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    shp = input_shape(a.model, a.batch)
    xs = [torch.randn(shp, device=dev, generator=g) for _ in range(2)]
    if cl:
        xs = [x.contiguous(memory_format=torch.channels_last) for x in xs]
    ys = [torch.randint(0, num_classes(a.model), (a.batch,), device=dev, generator=g) for _ in range(2)]

    host_phases = []

    def step(i, x=None, y=None):
        x = xs[i % 2] if x is None else x
        y = ys[i % 2] if y is None else y
        t0 = time.perf_counter()
        opt.zero_grad(set_to_none=False)
        loss = crit(model(x), y)
        t1 = time.perf_counter()
        loss.backward()
        t2 = time.perf_counter()
        opt.step()
        t3 = time.perf_counter()
        host_phases.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2), round((t3 - t2) * 1e3, 2)))
        return loss

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    graphed = a.mode == "graph"  # the SGD diagnostic is graphed too, so the two compare like for like
    if graphed:
        from paper_2107_06533_b200.graph import GraphedStep
        gs = GraphedStep(model, crit, opt, [xs[0]], [ys[0]], warmup=a.warmup,
                         before_capture=lambda: (_lib.stats_probes(() if a.stats_off else ROOF_CATS, slots=4096),
                                                 _lib.stats_reset(timing=())),
                         priority=a.main_priority)
        eager_step = step

        def step(i, x=None, y=None):
            x = xs[i % 2] if x is None else x
            y = ys[i % 2] if y is None else y
            return gs([x], [y])
        step(0)
    else:
        for i in range(a.warmup):
            step(i)
    torch.cuda.synchronize()
    barrier()
    if a.gc == "freeze":
        import gc
        gc.collect()
        gc.freeze()

    clocks = None
    if not a.profile and a.clocks == "nvml":
        try:
            clocks = NvmlClocks(local)
        except Exception:
            clocks = Clocks(local)
    elif not a.profile and a.clocks == "smi":
        clocks = Clocks(local)
    # live roofline timing of the dominant kernel only (events pre-created, outside the region);
    # in graph mode the event nodes were captured into the graph (stats reset before capture)
    if not graphed:
        _lib.stats_probes(() if a.stats_off else ROOF_CATS, slots=1000 * a.steps)
        _lib.stats_reset(timing=())
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ms0 = torch.cuda.memory_stats()
    w0 = time.perf_counter()
    e0.record(stream)
    evs = []
    for i in range(a.steps):
        if a.ncu_range and i == a.steps - 1:  # ncu --profile-from-start off: the last timed step only
            torch.cuda.cudart().cudaProfilerStart()
        loss = step(i)
        if a.ncu_range and i == a.steps - 1:
            torch.cuda.cudart().cudaProfilerStop()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        evs.append(ev)
    e1.record(stream)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3 / a.steps
    wall_ms = max_over_ranks(wall_ms)
    ms1 = torch.cuda.memory_stats()
    alloc_diag = {k: ms1.get(k, 0) - ms0.get(k, 0) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries",
                                                              "num_sync_all_streams")}
    barrier()
    ms = e0.elapsed_time(e1) / a.steps
    per_step = [round(e0.elapsed_time(evs[0]), 2)] + [round(evs[i - 1].elapsed_time(evs[i]), 2) for i in range(1, len(evs))]
    clk = clocks.stop() if clocks else None
    st = _lib.stats()
    # graph mode: launch counts / flops were accounted once at capture (= per replay) and the
    # captured event nodes hold the last replay's timestamps
    per = 1 if graphed else a.steps
    launches = st["total_launches"] * (a.steps if graphed else 1)
    if a.trace:  # every rank steps (collectives); rank 0 writes
        tags = None
        if world > 1:  # program order of this rank's collectives over one (eager) iteration
            opt.comm.log.clear()
            eager_step(0)
            torch.cuda.synchronize()
            tags = list(opt.comm.log)
        trace_summary(step, a.trace if rank == 0 else None, torch, comm_tags=tags)
    # per-category breakdown: a separate 2-step eager pass with every launch bracketed by events
    nb = 2
    _lib.stats_probes(())  # the breakdown pass times every launch with CUDA events
    _lib.stats_reset(timing=True, reserve=600 * nb)
    for i in range(nb):
        (eager_step if graphed else step)(i)
    torch.cuda.synchronize()
    bst = _lib.stats()
    ms_max = max_over_ranks(ms)
    final_loss = float(loss.item())
    opt.check_inverses()

    # ---- e2e through the public API: pinned host batch -> device every step, loss read back
    e2e = None
    if not a.no_e2e and not a.profile:
        xh = [x.cpu().pin_memory() for x in xs]  # keeps the channels-last strides
        yh = [y.cpu().pin_memory() for y in ys]
        xd, yd = torch.empty_like(xs[0]), torch.empty_like(ys[0])
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w1 = time.perf_counter()
        f0.record(stream)
        if graphed:  # step i+1's pinned host batch moves over PCIe on a copy stream while step i computes
            gs.prefetch([xh[0]], [yh[0]])
        for i in range(a.steps):
            if graphed:
                loss = gs()  # waits for the prefetched batch, device-to-device into the static buffers
                if i + 1 < a.steps:
                    gs.prefetch([xh[(i + 1) % 2]], [yh[(i + 1) % 2]])
            else:
                xd.copy_(xh[i % 2], non_blocking=True)
                yd.copy_(yh[i % 2], non_blocking=True)
                loss = step(i, xd, yd)
            _ = float(loss.item())
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_wall = (time.perf_counter() - w1) * 1e3 / a.steps
        e2e_ms = max_over_ranks(f0.elapsed_time(f1) / a.steps)
        e2e = {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": xh[0].numel() * 4 + yh[0].numel() * 8,
               "d2h_bytes_per_step": 4, "host_wall_ms": round(max_over_ranks(e2e_wall), 3),
               "pipeline": ("graph mode: each step's pinned host batch is copied on a copy stream while the previous "
                            "step computes (GraphedStep.prefetch: double-buffered device slots, then a device-to-device "
                            "copy into the graph inputs); the loss is read back every step" if graphed else
                            "eager: pinned host batch copied on the compute stream before each step; loss read back")}

    # ---- rooflines: every K-FAC kernel category timed live in the timed region (CUDA events on the
    # launching streams; graph mode: the event nodes of the last replay), the dominant one as the
    # headline `roofline`, and the iteration roofline fraction of SURVEY 8(d)
    peaks = dict(measured_peaks) if measured_peaks else {}
    try:
        peaks.update({k: v for k, v in json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).items()
                      if k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained")})
    except Exception:
        pass
    kern = {cat: kernel_roofline(cat, st[cat], per, peaks, world, a.model) for cat in ROOF_CATS if st[cat]["launches"]}
    timed = {c: r for c, r in kern.items() if r["kernel_ms_per_step"] > 0}
    dom = max(timed, key=lambda c: timed[c]["kernel_ms_per_step"]) if timed else None
    roofline = dict(timed[dom]) if dom else None
    step_ms_total = sum(v["ms"] for k, v in bst.items() if isinstance(v, dict)) / nb
    if roofline is not None:
        roofline["share_of_library_kernel_time"] = round(bst[dom]["ms"] / nb / step_ms_total, 4) if step_ms_total else None
        roofline["why_this_kernel"] = "largest live CUDA-event time per step among the K-FAC kernel categories"
    iteration_roofline = iteration_roof(bst, nb, peaks, ffbp_flops, ms_max)
    breakdown = {k: {"ms_per_step": round(v["ms"] / nb, 4), "launches_per_step": v["launches"] / nb,
                     "tflops": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] > 0 and v["flops"] else None}
                 for k, v in bst.items() if isinstance(v, dict)}
    breakdown["note"] = "separate 2-step pass with CUDA events around every library launch (not the timed region)"

    timeline = None
    if a.timeline and a.optimizer == "spdkfac":
        opt.timeline = {}
        (eager_step if graphed else step)(0)
        torch.cuda.synchronize()
        timeline = opt.timeline_ms()
        opt.timeline = None

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and not a.profile:
        cpu_ms, sample, _, kind = cpu_reference(a.model, a.batch, steps=1, warmup=1)
        cpu = {"value": round(cpu_ms, 1), "unit": "ms", "cores": int(os.environ["OPENBLAS_NUM_THREADS"]),
               "kind": kind, "sample": sample}

    if rank == 0:
        out = {"metric": METRIC, "value": round(ms_max, 3), "unit": "ms", "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": round(ms_max, 3), "higher_is_better": False, "scaling": "weak",
               "vs_baseline": None, "dtype": "f32",
               "dtype_note": "fp32-class: split-precision tcgen05 contractions with fp32 accumulate -- factors 3xbf16, "
                             "inverse panels / updates 3xfp16 on power-of-two-scaled planes (3xtf32 for gamma < 1e-4), "
                             "preconditioning 3xtf32; "
                             "forward/backward fp32 with TF32 convolutions (cuDNN default)",
               "data": "synthetic (random N(0,1) images, uniform labels; random-init torchvision weights)",
               "config": workload_config(a, world), "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
               "roofline_kernels": kern, "iteration_roofline": iteration_roofline, "peaks_measured": measured_peaks,
               "cpu_baseline": cpu, "clocks": clk, "kernel_breakdown": breakdown,
               "placement_imbalance": _imbalance(opt) if opt.placement is not None else None,
               "placement_nct_tensors": len(opt.placement.nct) if opt.placement is not None and world > 1 else None,
               "perf_params": (a.perf_params or "data/b200_p{N}.params (perfmodel.default_params)")
               if a.optimizer == "spdkfac" else None,
               "host_wall_ms_per_step": round(wall_ms, 3), "per_step_ms": per_step, "allocator_in_region": alloc_diag,
               "host_phase_ms_fwd_bwd_step": host_phases[a.warmup:a.warmup + a.steps] if a.profile is False else None,
               "final_loss": final_loss, "timeline_ms": timeline}
        if a.optimizer != "spdkfac":
            out["diagnostic"] = f"optimizer={a.optimizer}: not the SPD-KFAC metric"
        if world > 1:
            out["grad_allreduce"] = "NCCL (libspdkfac comm), grouped per step"

        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _imbalance(opt):
    from paper_2107_06533_b200.planner import placement_imbalance
    r = placement_imbalance(opt.placement, weight=lambda d: float(d) ** 3)
    r2 = placement_imbalance(opt.placement, weight=lambda d: float(d) ** 2)
    return {"d3_max_over_mean_minus_1": round(r["max_over_mean_minus_1"], 4),
            "d3_makespan_over_lower_bound": round(r["makespan_over_lower_bound"], 4),
            "d2_max_over_mean_minus_1": round(r2["max_over_mean_minus_1"], 4)}


# ---------------------------------------------------------------- reference arm
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    w0 = time.perf_counter()
    ms, sample, per_step, kind = cpu_reference(a.model, a.batch, steps=max(1, a.steps), warmup=a.warmup)
    wall = time.perf_counter() - w0
    cores = int(os.environ["OPENBLAS_NUM_THREADS"])
    out = {"metric": METRIC, "impl": "reference", "value": round(ms, 1), "unit": "ms", "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 1), "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(a, world),
           "cpu_baseline": {"value": round(ms, 1), "unit": "ms", "cores": cores, "kind": kind, "sample": sample},
           "e2e": {"value": round(ms, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "per_step_ms": [round(x * 1e3, 1) for x in per_step], "wall_s": round(wall, 1),
           "steps_timed": len(per_step),
           "steps_note": ("every timed step is a full step; steps beyond the wall budget (SPDKFAC_REF_BUDGET_S, "
                          "default 240 s) are not run, so steps_timed may be < steps"),
           "note": "reference kfacsched is CPU-only numpy/scipy (no GPU path): its own functions from "
                   "baseline/_ref (kind=reference) or the oracle port (kind=port); every timed step is a full "
                   "step (every layer of the model) on this rank's host cores"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    # a hung collective should end the run, not hold the GPUs: dump every thread's stack and exit
    # after SPD_WATCHDOG seconds (default 900; 0 disables, e.g. under ncu)
    _wd = int(os.environ.get("SPD_WATCHDOG", "900"))
    if _wd > 0:
        import faulthandler
        faulthandler.dump_traceback_later(_wd, exit=True)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
