#!/usr/bin/env python3
"""Summarise one measurement pass (tools/measure.sh <tag>) into profiles/:

  profiles/<tag>_ncu_summary.txt      key counters + stall mix per `ncu --set full` report
  profiles/<tag>_stage_traffic.json   DRAM bytes per RK stage of the element kernels (bench.py's `traffic`)
  profiles/<tag>_launches_summary.csv per-kernel totals of the launch list (share of the step)
  profiles/<tag>_launches.csv         the raw launch list
  profiles/<tag>_bench*.json          the bench lines

usage: tools/summarize_ncu.py <tag> [dof]
"""
import csv
import re
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return [{h: (u, v) for h, u, v in zip(hdr, units, r)} for r in vals]


def fp64_flops(rec):
    """FP64 flops of one launch from the SASS thread-instruction rates (FMA = 2)."""
    try:
        cyc = float(rec["smsp__cycles_elapsed.avg"][1].replace(",", ""))
        tot = 0.0
        for op, w in (("dfma", 2), ("dadd", 1), ("dmul", 1)):
            tot += w * cyc * float(rec[f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"][1]
                                   .replace(",", ""))
        return tot
    except (KeyError, ValueError):
        return None


def summarize(tag, dof):
    lines, kernels, bytes_k, flops_k = [], [], [], []
    # Exactly this pass's element-kernel captures (measure.sh names them <tag>_<kernel>_raw.csv);
    # a bare prefix match would also take another pass's files whose tag extends this one.
    pat = re.compile(re.escape(tag) + r"_k_[a-z0-9_]+?(_raw\.csv|\.ncu-rep)$")
    for rep in sorted(f for f in os.listdir(OUT) if pat.fullmatch(f) and not f.startswith(tag + "_k_launch")):
        for rec in raw(os.path.join(OUT, rep)):
            name = rec["Kernel Name"][1]
            lines.append(f"---- {name}")
            for k in KEYS:
                if k in rec:
                    u, v = rec[k]
                    lines.append(f"  {k:<62s} {v} {u}")
            stalls = {}
            for k, (u, v) in rec.items():
                pre = "smsp__average_warps_issue_stalled_"
                if k.startswith(pre) and k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls[k[len(pre):-len("_per_issue_active.ratio")]] = float(v)
                    except ValueError:
                        pass
            tot = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
            lines.append("  stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
            rd = float(rec["dram__bytes_read.sum"][1].replace(",", "")) * SCALE[rec["dram__bytes_read.sum"][0]]
            wr = float(rec["dram__bytes_write.sum"][1].replace(",", "")) * SCALE[rec["dram__bytes_write.sum"][0]]
            kernels.append(name)
            bytes_k.append(rd + wr)
            flops_k.append(fp64_flops(rec))
            if flops_k[-1] is not None:
                lines.append(f"  fp64 flops (2 dfma + dadd + dmul thread instructions)           {flops_k[-1]:.6g}")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.txt"), "w") as f:
        f.write(f"# {tag}: ncu --set full --clock-control none --import-source on, one launch per kernel\n")
        f.write("# command: tools/measure.sh (python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e)\n")
        f.write("\n".join(lines) + "\n")
    # The workload the captures ran (bench.py keys its roofline.traffic lookup on it).
    key, bj = None, os.path.join(OUT, f"{tag}_bench.json")
    if os.path.exists(bj):
        try:
            c = json.loads(open(bj).read())["config"]
            key = {"mesh": c.get("mesh"), "degree": c.get("degree"), "elements_per_gpu": c.get("elements_per_gpu")}
            dof = c.get("elements_per_gpu", 0) * (c.get("degree", 0) + 1) ** 3 or dof
        except Exception:
            key = None
    if kernels:
        tr = {
            "workload": key,
            "kernels": kernels,
            "bytes_per_kernel": bytes_k,
            "dram_bytes_per_stage": sum(bytes_k),
            "dof": dof,
            "dram_bytes_per_dof": sum(bytes_k) / dof,
            "fp64_flops_per_kernel": flops_k,
            "fp64_flops_per_dof": (sum(flops_k) / dof) if all(f is not None for f in flops_k) else None,
            "note": f"ncu --set full (profiles/{tag}_ncu_summary.txt); one launch of each element kernel; "
                    "mortar/pairing kernels add <1%",
        }
        json.dump(tr, open(os.path.join(PROF, f"{tag}_stage_traffic.json"), "w"), indent=1)

    src = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(PROF, f"{tag}_launches.csv"))
        txt = open(src).read()
        start = txt.find('"ID"')
        rows = list(csv.DictReader(io.StringIO(txt[start:])))
        agg = OrderedDict()
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0]
            v = float(r["Metric Value"].replace(",", ""))
            ms = v * {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6}.get(
                r["Metric Unit"], 1.0)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += ms
        tot = sum(v[1] for v in agg.values()) or 1.0
        with open(os.path.join(PROF, f"{tag}_launches_summary.csv"), "w") as f:
            f.write(f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none; "
                    "cold-cache, serialised)\n")
            f.write("# command: python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e\n")
            f.write("kernel, launches, total_ms, mean_ms, share\n")
            for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{k}, {n}, {ms:.4f}, {ms / n:.4f}, {ms / tot:.4f}\n")
    for suf in ("bench", "bench_ref"):
        p = os.path.join(OUT, f"{tag}_{suf}.json")
        if os.path.exists(p):
            d = json.loads(open(p).read())
            json.dump(d, open(os.path.join(PROF, f"{tag}_{suf}.json"), "w"), indent=1)


if __name__ == "__main__":
    summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 56623104)
