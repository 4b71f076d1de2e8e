"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv
python bench.py --profile --mode eager ...`) into profiles/: per-kernel and per-category
(breakdown.py) time per step.  Steps are counted by pivot_kernel launches (66 per step on
ResNet-50 at P = 1).  Usage: python scripts/launch_list_summary.py LAUNCHES.csv OUT.json [pivots_per_step]"""
import collections
import csv
import json
import sys

sys.path.insert(0, ".")
from paper_2107_06533_b200 import breakdown as BD  # noqa: E402


def main(path, out, pivots_per_step=66):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, si = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Stream")
    data = [(r[ki], float(r[vi].replace(",", "")), r[si]) for r in rows[1:] if r[vi] not in ("", "nan")]
    busy = collections.Counter()
    for n, v, s in data:
        if not BD.is_nccl(n) and BD.classify(n) == "FFBP":
            busy[s] += v
    main_stream = busy.most_common(1)[0][0]
    nsteps = sum(1 for n, _, _ in data if "pivot_kernel" in n) / float(pivots_per_step)
    per = collections.defaultdict(lambda: [0, 0.0, ""])
    cat = collections.defaultdict(float)
    for n, v, s in data:
        c = BD.classify(n, s == main_stream)
        k = (n.split("(")[0][:110], c)
        per[k][0] += 1
        per[k][1] += v
        per[k][2] = c
        cat[c] += v
    tot = sum(cat.values())
    res = {"source": f"{path.split('/')[-1]}: ncu gpu__time_duration.sum, --clock-control none (serialised, cold "
                     f"caches); every eager step of the run incl. warm-up and the breakdown pass, normalised per step "
                     f"by {pivots_per_step} pivot launches/step",
           "steps_seen": nsteps,
           "per_step_ms_by_category": {k: round(v / 1e6 / nsteps, 3) for k, v in cat.items()},
           "share_of_step_by_category": {k: round(v / tot, 4) for k, v in cat.items()},
           "kernels": [{"name": k[0], "category": k[1], "launches_per_step": round(v[0] / nsteps, 1),
                        "ms_per_step": round(v[1] / 1e6 / nsteps, 4), "us_per_launch": round(v[1] / v[0] / 1e3, 2)}
                       for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])[:60]]}
    json.dump(res, open(out, "w"), indent=1)
    print(res["per_step_ms_by_category"], res["share_of_step_by_category"], nsteps)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(int(x) for x in sys.argv[3:]))
