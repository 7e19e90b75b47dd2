"""Summarise an ncu --set full capture (read here, no GPU): key throughput
metrics, stall reasons and the executed instruction mix of one kernel."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def main(rep, want_kernel="fast_attention"):
    h, rows = raw(rep)
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
    for r in rows:
        d = dict(zip(h, r))
        if want_kernel not in d.get("Kernel Name", ""):
            continue
        for k in keys:
            print(f"{k:70s} {d.get(k)}")
        stalls = sorted(((float(v), k) for k, v in d.items()
                         if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio") and v not in ("", "n/a")),
                        reverse=True)
        for v, k in stalls[:10]:
            print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', ''):60s} {v:.3f}")
        break
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    hdr, mix, tot = None, Counter(), 0
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Address":
            if hdr is not None:
                break
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                n = int(d["Instructions Executed"] or 0)
            except ValueError:
                n = 0
            op = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip())
            op = op.split()[0].split(".")[0] if op else "?"
            mix[op] += n
            tot += n
    print(f"warp-instructions executed: {tot}")
    for op, n in mix.most_common(16):
        print(f"  {op:10s} {n:11d} {100 * n / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
