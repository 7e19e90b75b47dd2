"""Attribute an ncu source-page capture (SASS) to CUDA source lines and to
warp-role line ranges, using nvdisasm line info (with inlining) of the built
object.  Each instruction is charged to its innermost source line (helpers
such as mbar_wait or mma_codes) and, for the role split and the call-site
table, to the outermost line of the kernel that called it.

    python tools/ncu_lines.py REP.ncu-rep OBJ.o KERNEL_MANGLED [role=a-b ...]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

PAIR = re.compile(r'File "([^"]+)", line (\d+)')


def line_map(obj, func):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True, check=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "--print-line-info-inline", os.path.join(tmp, cubin)], capture_output=True,
                         text=True).stdout
    m, block, cur, inside = {}, [], None, False
    for ln in out.splitlines():
        if ln.startswith(".text."):
            inside = ln.strip().rstrip(":") == ".text." + func
            continue
        if not inside:
            continue
        if "//##" in ln:
            block.append([(os.path.basename(f), int(n)) for f, n in PAIR.findall(ln)])
            continue
        if block:
            inner = block[0][0]
            outer = block[-1][-1]
            cur = (inner, outer)
            block = []
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if a and cur is not None:
            m[int(a.group(1), 16)] = cur
    return m


def main(rep, obj, func, *roles):
    lm = line_map(obj, func)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    idx = {k: i for i, k in enumerate(hdr)}
    base = None
    inner_l = defaultdict(lambda: [0, 0])
    outer_l = defaultdict(lambda: [0, 0])
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        addr = int(r[0], 16)
        base = addr if base is None else base
        inner, outer = lm.get(addr - base, (("?", -1), ("?", -1)))
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(r[idx["Instructions Executed"]] or 0)
        for d, k in ((inner_l, inner), (outer_l, outer)):
            d[k][0] += s
            d[k][1] += n
    tot_s = sum(v[0] for v in inner_l.values())
    tot_i = sum(v[1] for v in inner_l.values())
    spans = []
    for rr in roles:
        name, ab = rr.split("=")
        a, b = (int(x) for x in ab.split("-"))
        spans.append((name, a, b))
    agg = defaultdict(lambda: [0, 0])
    for line, (s, n) in outer_l.items():
        name = next((nm for nm, a, b in spans if a <= line[1] <= b), "other")
        agg[name][0] += s
        agg[name][1] += n
    print(f"{'role':12s} {'stall samples':>14s} {'%':>6s} {'warp-instr':>12s} {'%':>6s}")
    for name, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{name:12s} {s:14d} {100 * s / max(tot_s, 1):6.1f} {n:12d} {100 * n / max(tot_i, 1):6.1f}")
    for title, d in (("call sites (outermost line)", outer_l), ("innermost lines", inner_l)):
        print(f"\ntop {title} by samples:")
        for line, (s, n) in sorted(d.items(), key=lambda kv: -kv[1][0])[:30]:
            print(f"  {line[0]}:{line[1]:<5d}  samples {s:8d} ({100 * s / max(tot_s, 1):5.1f}%)  instr {n:10d}")


if __name__ == "__main__":
    main(*sys.argv[1:])
