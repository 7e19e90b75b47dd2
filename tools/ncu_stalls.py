"""Stall-reason samples per warp role (outermost source line ranges) from an
ncu source-page capture.  python tools/ncu_stalls.py REP OBJ KERNEL role=a-b ..."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, __import__("os").path.dirname(__file__))
import ncu_lines as nl  # noqa: E402


def main(rep, obj, func, *roles):
    lm = nl.line_map(obj, func)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {k: i for i, k in enumerate(hdr)}
    spans = [(r.split("=")[0], *map(int, r.split("=")[1].split("-"))) for r in roles]
    agg = defaultdict(lambda: defaultdict(int))
    base = None
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        a = int(r[0], 16)
        base = a if base is None else base
        _, outer = lm.get(a - base, (("?", -1), ("?", -1)))
        role = next((nm for nm, lo, hi in spans if lo <= outer[1] <= hi), "other")
        for cname in cols:
            agg[role][cname] += int(r[idx[cname]] or 0)
    for role, d in agg.items():
        tot = sum(d.values())
        print(f"{role}: {tot} samples  " + ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.0f}%" for k, v in
                                                     sorted(d.items(), key=lambda kv: -kv[1]) if v * 50 > tot))


if __name__ == "__main__":
    main(*sys.argv[1:])
