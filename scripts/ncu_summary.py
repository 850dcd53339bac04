"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
launches, total / mean device time and share of the listed time."""
import csv
import sys
from collections import OrderedDict


def main(path, skip_regex=None):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        rows.append((r["Kernel Name"].split("(")[0], ns))
    agg = OrderedDict()
    for name, ns in rows:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {len(rows)} launches, {tot/1e3:.1f} us total")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {n} | {ns/1e3:.1f} | {ns/n/1e3:.1f} | {ns/tot:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1])
