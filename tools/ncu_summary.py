"""Summaries of ncu output for profiles/ (run here, on the files gpurun brings back).

  python tools/ncu_summary.py launches gpurun_out/launches.csv   # launch-list table (markdown)
  python tools/ncu_summary.py full gpurun_out/prof_full.ncu-rep  # key metrics + stall shares
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(double2 \*, T3\)$", "", name)
    name = name.replace("qtb::", "").replace("(int)", "").replace("(bool)", "")
    return re.sub(r"\(.*\)$", "", name)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        k = short(r[4])
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[13], 1e-6)
        tot[k] += float(r[14].replace(",", "")) * scale
        cnt[k] += 1
    allms = sum(tot.values())
    print("| kernel | launches | total (ms) | share |")
    print("|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / allms:.1f}% |")


KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
        "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    print(f"{'Kernel Name':64s} {short(d['Kernel Name'][0])}")
    for k in KEYS:
        if k in d:
            print(f"{k:64s} {d[k][0]} {d[k][1]}")
    pre = "smsp__average_warps_issue_stalled_"
    st = {k[len(pre):].replace("_per_issue_active.ratio", ""): float(v[0])
          for k, v in d.items() if k.startswith(pre) and k.endswith("_per_issue_active.ratio")}
    tot = sum(st.values()) or 1.0
    print("stall reasons (share of samples):")
    for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]:
        print(f"  {k:30s} {100 * v / tot:.1f}%")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
