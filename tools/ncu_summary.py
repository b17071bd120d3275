"""Summarise one kernel of an ncu report (raw metrics + SASS mix) into the text
format kept under profiles/.

    python tools/ncu_summary.py report.ncu-rep "<header line>" > profiles/rNN_x.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
    "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"# {header}")
    print(f"# report: {rep} (kernel: {vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else '?'})")
    print()
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            print(f"{m:70s} {vals[i]:>16s} {units[i]}")
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(vals[i])
            except ValueError:
                pass
    if stalls:
        top = sorted(stalls.items(), key=lambda x: -x[1])[:9]
        print("stalls/issue: " + ", ".join(f"{k}={v:.2f}" for k, v in top))
    src = ncu_csv(rep, "source")
    shdr = src[1]
    ci = {h: i for i, h in enumerate(shdr)}
    mix, stall = defaultdict(int), defaultdict(float)
    for r in src[2:]:
        try:
            n = int(r[ci["Instructions Executed"]])
            smp = float(r[ci["Warp Stall Sampling (All Samples)"]])
        except (ValueError, KeyError, IndexError):
            continue
        op = r[ci["Source"]].strip().split()
        if not op:
            continue
        mn = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        mn = mn.split(".")[0]
        mix[mn] += n
        stall[mn] += smp
    tot, tots = sum(mix.values()), sum(stall.values()) or 1.0
    print()
    print("# SASS instruction mix (executed warp-instructions, share of stall samples)")
    print(f"total inst {tot} samples {int(tots)}")
    for mn, n in sorted(mix.items(), key=lambda x: -x[1])[:18]:
        print(f"{mn:12s} {n:12d} {100 * n / max(tot, 1):5.1f}%  stall {100 * stall[mn] / tots:5.1f}%")


if __name__ == "__main__":
    main()
