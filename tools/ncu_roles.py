"""Per-page instruction budget of the page kernel by source line and opcode,
from an ncu source-page capture (outermost call site, see ncu_lines.py).

    python tools/ncu_roles.py REP.ncu-rep OBJ.o KERNEL_MANGLED PAGES role=a-b ...
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, __import__("os").path.dirname(__file__))
import ncu_lines as nl  # noqa: E402


def main(rep, obj, func, pages, *roles):
    pages = float(pages)
    lm = nl.line_map(obj, func)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    idx = {k: i for i, k in enumerate(hdr)}
    src_file = [l for l in open(obj.replace("build/", "").replace(".o", ".cu")).read().split("\n")]
    base = None
    per = defaultdict(int)
    ops = defaultdict(lambda: defaultdict(int))
    spans = [(r.split("=")[0], *map(int, r.split("=")[1].split("-"))) for r in roles]
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        a = int(r[0], 16)
        base = a if base is None else base
        inner, outer = lm.get(a - base, (("?", -1), ("?", -1)))
        n = int(r[idx["Instructions Executed"]] or 0)
        per[outer] += n
        toks = r[idx["Source"]].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        role = next((nm for nm, lo, hi in spans if lo <= outer[1] <= hi), "other")
        ops[role][op.split(".")[0]] += n
    for nm, lo, hi in spans:
        tot = sum(v for k, v in per.items() if lo <= k[1] <= hi)
        print(f"{nm}: {tot / pages:.0f} warp-instr / page")
        for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
            if lo <= k[1] <= hi and v / pages >= 6:
                print(f"  {k[1]:5d} {v / pages:7.1f}  {src_file[k[1] - 1].strip()[:96]}")
        print("  ops:", ", ".join(f"{o} {v / pages:.0f}" for o, v in sorted(ops[nm].items(), key=lambda kv: -kv[1])[:16]))


if __name__ == "__main__":
    main(*sys.argv[1:])
