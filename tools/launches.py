"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/launches.py FILE.csv [--seq N]
"""
import collections
import csv
import sys


def load(path):
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    out = []
    for x in csv.DictReader(lines):
        if x.get("Metric Name") == "gpu__time_duration.sum":
            name = x["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
            v = float(x["Metric Value"].replace(",", ""))
            unit = x.get("Metric Unit", "nsecond")
            us = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
            out.append((name, us))
    return out


def main():
    path = sys.argv[1]
    rows = load(path)
    agg = collections.OrderedDict()
    for n, us in rows:
        a = agg.setdefault(n, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += us
        a[2] = max(a[2], us)
    tot = sum(us for _, us in rows)
    print(f"{path}: {len(rows)} launches, {tot:.1f} us total")
    for n, (c, s, m) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {n[:60]:60s} n={c:4d} sum={s:9.1f} us max={m:8.1f} share={s / tot:6.1%}")
    if "--seq" in sys.argv:
        k = int(sys.argv[sys.argv.index("--seq") + 1])
        for n, us in rows[:k]:
            print(f"    {n[:60]:60s} {us:9.1f}")


if __name__ == "__main__":
    main()
