"""Hottest SASS instructions (stall samples) of an ncu source-page capture.
python tools/ncu_hot.py REP [N] [PAGES]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
pages = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {k: i for i, k in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    ins.append((int(r[0], 16), r[1].strip(), int(r[idx["Instructions Executed"]] or 0),
                int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)))
base = ins[0][0]
tot = sum(x[3] for x in ins)
print("samples", tot, "instructions / page", round(sum(x[2] for x in ins) / pages, 1))
for a, s, e, st in sorted(ins, key=lambda x: -x[3])[:n]:
    print(f"{a - base:#7x} {st:6d} {100 * st / tot:5.2f}%  x{e / pages:5.2f}  {s[:80]}")
