"""Summarise an `ncu --csv --log-file` launch list: per-kernel count, time,
share, DRAM bytes and GB/s; optionally print the first launches in order."""
import csv
import collections
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rd = csv.DictReader(lines)
    by = {}
    for d in rd:
        e = by.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d["Grid Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [by[i] for i in sorted(by)]


def main(path, first=0):
    ks = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k in ks:
        nm = k["name"].split("(")[0][:48]
        t = k.get("gpu__time_duration.sum", 0.0)
        b = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        agg[nm][0] += 1
        agg[nm][1] += t
        agg[nm][2] += b
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':48s} {'n':>5s} {'total_us':>10s} {'share':>6s} {'us/launch':>9s} {'GB/s':>8s}")
    for nm, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{nm:48s} {n:5d} {t/1e3:10.1f} {t/tot:6.3f} {t/n/1e3:9.2f} {b/t if t else 0:8.1f}")
    print(f"total {tot/1e3:.1f} us over {len(ks)} launches")
    for k in ks[:first]:
        t = k.get("gpu__time_duration.sum", 0.0)
        b = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        print(f"  {k['name'][:40]:40s} grid={k['grid']:14s} {t/1e3:8.2f}us {b/1e6:9.2f}MB {b/t if t else 0:8.1f}GB/s")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
