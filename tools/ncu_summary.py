"""Summarise ncu outputs (run here, on the CPU box) into profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [<traffic.json> <workload-name>]
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def _rows(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def launches(path, out):
    rows = _rows(open(path).read())
    per = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("ellm::", "").strip()
        if "paged_attn" in r["Kernel Name"]:
            name = "paged_attn_kernel"
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "nsecond" or unit == "ns" else v if unit in ("usecond", "us") else v * 1e3
        d = per.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += us
    total = sum(v[1] for v in per.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({path})\n\n`ncu --metrics gpu__time_duration.sum --clock-control none "
                "--profile-from-start off` over the timed decode steps of `bench.py --profile` "
                "(cold-cache, serialised launches: compare shares, not absolutes).\n\n")
        f.write("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
        for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {us:.1f} | {us / n:.2f} | {100 * us / total:.1f}% |\n")
        f.write(f"\nTotal kernel time {total:.1f} us over {sum(v[0] for v in per.values())} launches.\n")
    print(open(out).read())


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed_pipe_tensor_op_hmma.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def full(rep, out, traffic_json=None, wl_name=None):
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [ln for ln in raw.splitlines() if ln.startswith('"')]
    rd = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, data = rd[0], rd[1], rd[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    with open(out, "w") as f:
        f.write(f"# ncu --set full ({rep})\n\n")
        for row in data:
            f.write(f"## {row[idx['Kernel Name']][:90]}\n\n| metric | value | unit |\n|---|---|---|\n")
            for m in WANT:
                if m in idx:
                    f.write(f"| {m} | {row[idx[m]]} | {units[idx[m]]} |\n")
            stalls = sorted(((h, row[i]) for h, i in idx.items() if h.startswith("smsp__average_warp_latency_issue_stalled_")
                             or h.startswith("smsp__pcsamp_warps_issue_stalled_")), key=lambda x: -_num(x[1]))[:8]
            f.write("\nTop stall counters:\n\n")
            for h, v in stalls:
                f.write(f"- {h}: {v}\n")
            f.write("\n")
        if traffic_json and wl_name and data:
            row = data[-1]
            rb = _num(row[idx["dram__bytes_read.sum"]]) * _scale(units[idx["dram__bytes_read.sum"]])
            wb = _num(row[idx["dram__bytes_write.sum"]]) * _scale(units[idx["dram__bytes_write.sum"]])
            try:
                tj = json.load(open(traffic_json))
            except Exception:
                tj = {}
            tj[wl_name] = int(rb + wb)
            json.dump(tj, open(traffic_json, "w"), indent=1)
            f.write(f"traffic (dram read + write) per launch: {int(rb + wb)} B -> {traffic_json}\n")
    print(open(out).read())


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return 0.0


def _scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) > 5 else []))
