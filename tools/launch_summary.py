"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time per kernel name,
launch count and share of the summed kernel time. Usage: launch_summary.py launches.csv [top]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        if "cub::" in short:
            short = short.split("<")[0]
        elif "<" in name.split("(")[0]:
            short = name.split("(")[0].replace("void ", "")
        rows.append((short, float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)))
    agg = defaultdict(lambda: [0.0, 0])
    for k, us in rows:
        agg[k][0] += us
        agg[k][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"{len(rows)} launches, {tot:.1f} us summed (serialised, cold-cache)")
    print(f"{'kernel':60s} {'us':>9s} {'n':>5s} {'share':>6s}")
    for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[:60]:60s} {us:9.1f} {n:5d} {100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main()
