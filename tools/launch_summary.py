"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(lines[start:]))


def main(path):
    rows = load(path)
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        n = r["Kernel Name"].split("(")[0].split("<")[0]
        agg[n][0] += 1
        agg[n][1] += float(r["Metric Value"]) / 1e6
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:28s} {c:8d} {t:10.3f} {t / c:9.4f} {100 * t / tot:5.1f}%")
    print(f"{'total':28s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
