"""Summarise an ncu metrics CSV of one eager bench step (scripts/r2_profiles.sh) into per-category
kernel time and DRAM bytes per step, in the libspdkfac stats categories bench.py reports.

  python scripts/traffic_summary.py gpurun_out/r2_step_traffic.csv profiles/traffic_resnet50_n1.json
"""
import csv
import json
import re
import sys

CATS = [  # (category, kernel-name regex) -- first match wins
    ("factor_stage", r"stage_rows|stage_im2col|stage_spatial"),
    ("factor_syrk", r"tc3_gemm_kernel<(\(spd::Kind\))?1,|tc3_pair_kernel"),
    ("factor_reduce", r"reduce_pack"),
    ("inv_pivot", r"pivot_kernel(<[^>]*>)?\(|pivot_tc_kernel<(\(bool\))?(0|false)>"),
    ("inv_small", r"small_inverse|pivot_tc_kernel<(\(bool\))?(1|true)>"),
    ("inv_panel", r"stage_panel|inv_scale|tc3_gemm_kernel<(\(spd::Kind\))?[02], (\(int\))?3, (\(bool\))?(0|false), (\(int\))?0[,>]"),
    ("inv_update", r"tc3_gemm_kernel<(\(spd::Kind\))?[02], (\(int\))?3, (\(bool\))?(1|true)|tc3_pair_ctile"),
    ("inv_unpack_finalize", r"damp_unpack|finalize_kernel"),
    ("precond_gemm", r"tc3_gemm_kernel<(\(spd::Kind\))?[02], (\(int\))?3, (\(bool\))?(0|false), (\(int\))?[1-9]"),
    ("precond_split", r"split_rows_batched|split_rows_f16|packed_row_bounds|stage_packed"),
    ("pack", r"pack_|unpack_"),
]


def main(src, dst):
    rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
    hdr = rows[0]
    ik, im, iu, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3,
             "usecond": 1.0, "msecond": 1e3}
    launches = {}
    for r in rows[1:]:
        k = launches.setdefault(r[iid], {"name": r[ik]})
        k[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    out = {c: {"kernel_us": 0.0, "dram_bytes_per_step": 0.0, "launches_per_step": 0} for c, _ in CATS}
    other = {"kernel_us": 0.0, "dram_bytes_per_step": 0.0, "launches_per_step": 0}
    for k in launches.values():
        tgt = other
        if "spd::" in k["name"] or "pivot_kernel" in k["name"]:
            for c, rx in CATS:
                if re.search(rx, k["name"]):
                    tgt = out[c]
                    break
        tgt["kernel_us"] += k.get("gpu__time_duration.sum", 0.0)
        tgt["dram_bytes_per_step"] += k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        tgt["launches_per_step"] += 1
    total = sum(v["kernel_us"] for v in out.values()) + other["kernel_us"]
    for v in list(out.values()) + [other]:
        v["share_of_step_kernel_time"] = round(v["kernel_us"] / total, 4) if total else None
        v["source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum over one eager "
                       "bench step (--ncu-range), serialised and cold: compare shares, not absolute times")
    res = {k: v for k, v in out.items() if v["launches_per_step"]}
    res["forward_backward_and_other"] = other
    res["total_kernel_us_serialised"] = total
    json.dump(res, open(dst, "w"), indent=1)
    for c, v in res.items():
        if isinstance(v, dict):
            print(f"{c:28s} {v['launches_per_step']:5d} launches {v['kernel_us'] / 1e3:8.3f} ms "
                  f"{v['dram_bytes_per_step'] / 1e9:7.3f} GB  share {v['share_of_step_kernel_time']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
