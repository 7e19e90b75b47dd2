"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import io
import sys
from collections import defaultdict


def main(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    tot = sum(sum(v) for k, v in agg.items() if "prefill" not in k)
    print(f"{'kernel':55s} {'launches':>8s} {'avg us':>9s} {'total us':>10s} {'share of decode':>15s}")
    for k, v in agg.items():
        share = "" if "prefill" in k else f"{100 * sum(v) / tot:14.1f}%"
        print(f"{k:55s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / 1e3:10.1f} {share:>15s}")


if __name__ == "__main__":
    main(sys.argv[1])
