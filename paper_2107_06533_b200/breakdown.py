"""Measured six-category iteration breakdown.

The reference splits a *simulated* iteration into FFBP / GradComm / FactorComp /
FactorComm / InverseComp / InverseComm (simulator.py:80-96) and charges
communication only for its part not overlapped by compute (`breakdown`,
simulator.py:529-544); `breakdown_to_csv` / `timeline_to_csv`
(simulator.py:673-704) are its export formats.

Here the same categories come from a MEASURED kernel timeline (CUPTI, one
iteration of the CUDA graph).  The GPU runs several compute streams at once, so
"sum of compute durations" would count an instant twice; instead every instant
of the iteration is charged to exactly one category, compute before
communication, in the order below.  The categories then partition the
iteration span, as the reference's do, plus two rows the reference does not
model: preconditioning/update and idle gaps.
"""

from __future__ import annotations

import csv as _csv
import io
import re
from typing import Iterable, Sequence

CATEGORY_ORDER = ("FFBP", "GradComm", "FactorComp", "FactorComm", "InverseComp", "InverseComm")
EXTRA = ("Precondition", "Idle")
# charge priority for an instant covered by several categories: compute first
_PRIORITY = ("FFBP", "FactorComp", "InverseComp", "Precondition", "GradComm", "FactorComm", "InverseComm")
_COMM = {"GradComm", "FactorComm", "InverseComm"}

_K = r"tc3_gemm_kernel<(?:\(spd::Kind\))?"
_RULES = (
    # peer-memory factor aggregation (csrc/peer.cu): flag signal / wait and the owner-side inbox sum
    ("FactorComm", r"peer_signal_kernel|peer_wait_kernel|peer_sum_kernel|epoch_advance_kernel"),
    ("Precondition", r"split_rows_batched|split_rows_f16|packed_row_bounds|apply_update|stage_packed|" + _K +
     r"[02], \d+, false, [1-9]"),  # TF32 / F16, chunked accumulation
    ("FactorComp", r"stage_rows|stage_im2col|stage_spatial|reduce_pack|tc3_pair|" + _K + "1,"),  # bf16 SYRK
    ("InverseComp", r"pivot_kernel|pivot_tc_kernel|stage_panel|small_inverse|damp_unpack|finalize_kernel|inv_scale|"
                    r"unpack_upper|pack_upper|tc3_pair_ctile|" + _K + "[02],"),  # TF32 / F16 panel + update
)


# comm tags recorded by NcclComm -> category
COMM_TAGS = {"factor": "FactorComm", "inverse": "InverseComm", "grad": "GradComm"}


def classify(name: str, on_main: bool = False) -> str:
    """Category of one non-NCCL kernel; everything that is not ours is forward/backward (FFBP).
    on_main: the kernel ran on the main (forward/backward) stream."""
    for cat, rx in _RULES:
        if re.search(rx, name):
            return cat
    return "FFBP"


def is_nccl(name: str) -> bool:
    return "nccl" in name.lower()


def main_stream(kernels: Sequence[tuple]):
    """The stream carrying most forward/backward (non-library) kernel time."""
    busy = {}
    for s, e, name, stream in kernels:
        if not is_nccl(name) and classify(name) == "FFBP":
            busy[stream] = busy.get(stream, 0.0) + (e - s)
    return max(busy, key=busy.get) if busy else None


def label_events(kernels: Sequence[tuple], comm_tags: Sequence[str]) -> list:
    """kernels: (start, end, name, stream) of ONE iteration, any order.  NCCL kernels are
    matched in start order to `comm_tags` (the optimizer's program order of collective
    launches, one tag per NCCL kernel / group); returns (start, end, name, stream, category)."""
    ks = sorted(kernels, key=lambda k: (k[0], k[1]))
    main = main_stream(ks)
    n_comm = sum(1 for k in ks if is_nccl(k[2]))
    if n_comm != len(comm_tags):
        raise ValueError(f"{n_comm} NCCL kernels in the window but {len(comm_tags)} comm tags")
    out, ci = [], 0
    for s, e, name, stream in ks:
        if is_nccl(name):
            cat = COMM_TAGS[comm_tags[ci]]
            ci += 1
        else:
            cat = classify(name, stream == main)
        out.append((s, e, name, stream, cat))
    return out


def breakdown(events: Iterable[tuple], start: float | None = None, end: float | None = None) -> dict:
    """Charge each instant of [start, end] to one category (priority: compute, then comm).

    events: (start, end, name, stream, category).  Returns {category: seconds-or-units}
    over CATEGORY_ORDER + EXTRA; the values sum to end - start."""
    evs = [e for e in events if e[1] > e[0]]
    if not evs:
        return {c: 0.0 for c in CATEGORY_ORDER + EXTRA}
    t0 = min(e[0] for e in evs) if start is None else start
    t1 = max(e[1] for e in evs) if end is None else end
    cuts = sorted({t0, t1, *(max(t0, min(t1, e[0])) for e in evs), *(max(t0, min(t1, e[1])) for e in evs)})
    totals = {c: 0.0 for c in CATEGORY_ORDER + EXTRA}
    rank = {c: i for i, c in enumerate(_PRIORITY)}
    # sweep: active count per category
    bounds = sorted([(e[0], 1, e[4]) for e in evs] + [(e[1], -1, e[4]) for e in evs], key=lambda b: (b[0], b[1]))
    active = {c: 0 for c in _PRIORITY}
    bi = 0
    for a, b in zip(cuts, cuts[1:]):
        while bi < len(bounds) and bounds[bi][0] <= a:
            active[bounds[bi][2]] += bounds[bi][1]
            bi += 1
        live = [c for c in _PRIORITY if active[c] > 0]
        cat = min(live, key=rank.__getitem__) if live else "Idle"
        totals[cat] += b - a
    return totals


def _fmt(seconds: float) -> str:
    return f"{seconds:.9f}"


def breakdown_to_csv(totals: dict, extra: bool = True) -> str:
    """simulator.py:684-691 format (category,seconds); the two extra rows follow the six."""
    out = io.StringIO()
    w = _csv.writer(out, lineterminator="\n")
    w.writerow(["category", "seconds"])
    for cat in CATEGORY_ORDER + (EXTRA if extra else ()):
        w.writerow([cat, _fmt(totals.get(cat, 0.0))])
    return out.getvalue()


def timeline_to_csv(events: Sequence[tuple], t0: float = 0.0) -> str:
    """simulator.py:674-681 format (event,category,resource,start,end,layer); times in seconds
    from t0; `layer` carries the CUDA stream id."""
    out = io.StringIO()
    w = _csv.writer(out, lineterminator="\n")
    w.writerow(["event", "category", "resource", "start", "end", "layer"])
    for s, e, name, stream, cat in sorted(events, key=lambda x: (x[0], x[1])):
        res = "comm" if cat in _COMM else "compute"
        w.writerow([name[:120], cat, res, _fmt(s - t0), _fmt(e - t0), f"stream{stream}"])
    return out.getvalue()
