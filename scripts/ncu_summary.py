"""Summarise an `ncu --set full` report into profiles/: per-kernel launch count, mean duration,
DRAM bytes per launch (read + write, the bench `roofline.traffic` figure) and tensor-pipe /
DRAM utilisation.  Usage:
  python scripts/ncu_summary.py REPORT.ncu-rep|RAW.csv OUT.json [kernel-regex]
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out, rx=None):
    if rep.endswith(".csv"):  # `ncu -i X.ncu-rep --page raw --csv` export
        txt = open(rep).read()
        txt = txt[txt.index('"ID"'):]
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in data:
        name = r[col["Kernel Name"]]
        if rx and not re.search(rx, name):
            continue
        key = name.split("(")[0]
        d = per.setdefault(key, {"launches": 0, "us": 0.0, "dram_bytes": 0.0, "tensor_active_pct": 0.0,
                                 "tensor_elapsed_pct": 0.0, "dram_pct": 0.0, "sm_pct": 0.0})
        def val(m):
            if m not in col or r[col[m]] in ("", "n/a"):
                return 0.0
            return float(r[col[m]].replace(",", "")) * SCALE.get(units[col[m]], 1.0)
        d["launches"] += 1
        d["us"] += val("gpu__time_duration.sum")
        d["dram_bytes"] += val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        d["tensor_active_pct"] += val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        d["tensor_elapsed_pct"] += val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        d["dram_pct"] += val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
        d["sm_pct"] += val("sm__throughput.avg.pct_of_peak_sustained_elapsed")
    res = {}
    for k, d in per.items():
        n = d["launches"]
        res[k] = {"launches": n, "mean_us": round(d["us"] / n, 3), "dram_bytes_per_launch": round(d["dram_bytes"] / n),
                  "achieved_dram_gbs": round(d["dram_bytes"] / (d["us"] * 1e3), 1),
                  "tensor_pipe_active_pct": round(d["tensor_active_pct"] / n, 2),
                  "tensor_pipe_elapsed_pct": round(d["tensor_elapsed_pct"] / n, 2),
                  "dram_pct_of_peak": round(d["dram_pct"] / n, 2), "sm_throughput_pct": round(d["sm_pct"] / n, 2)}
    json.dump({"report": rep.split("/")[-1], "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))




def step_traffic(raw_csv, out, launches_per_step, model="resnet50", note=""):
    """profiles/syrk_traffic_n1.json for bench.py's roofline.traffic: DRAM bytes of the LAST
    `launches_per_step` factor-SYRK launches (one whole step) of an ncu --set full capture of
    eager steps; the factor stream is the one the CTA-pair engine launches on (the
    preconditioning GEMMs share the single-CTA kernel but run on the main stream)."""
    txt = open(raw_csv).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    pair_streams = [r[col["Stream"]] for r in data if "tc3_pair" in r[col["Kernel Name"]]]
    fs = max(set(pair_streams), key=pair_streams.count)
    syrk = [r for r in data if r[col["Stream"]] == fs][-int(launches_per_step):]

    def val(r, m):
        return float(r[col[m]].replace(",", "")) * SCALE.get(units[col[m]], 1.0)
    b = sum(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum") for r in syrk)
    us = sum(val(r, "gpu__time_duration.sum") for r in syrk)
    res = {"model": model, "launches_per_step": len(syrk), "dram_bytes_per_step": round(b),
           "ncu_us_per_step": round(us, 1),
           "source": f"ncu --set full --clock-control none, last {len(syrk)} factor-SYRK launches (one eager step) "
                     f"of {raw_csv.split('/')[-1]}" + (f"; {note}" if note else "")}
    json.dump(res, open(out, "w"), indent=1)
    print(res)


if __name__ == "__main__":
    if sys.argv[1] == "--step":
        step_traffic(sys.argv[2], sys.argv[3], int(sys.argv[4]))
    else:
        main(*sys.argv[1:])
