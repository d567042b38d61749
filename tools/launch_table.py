"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
usage: launch_table.py LAUNCHES.csv [top]"""
import collections
import csv
import sys


def main(path, top=30):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        n = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("vp::", "")
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(top)]:
        print(f"{n:32s} {c:5d} {v / 1e6:8.3f} ms {v / c / 1e3:9.1f} us/launch {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
