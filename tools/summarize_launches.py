"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel mean time and share."""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    m = re.search(r"gemm_(tc|simt)<(\d+)?,? ?gorila::(\w+)", name)
    return name if not m else name


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1000.0 if unit == "ns" else v * 1000.0 if unit == "ms" else v if unit in ("us", "usecond") else v
        rows.append((r["Kernel Name"], v))
    agg = collections.OrderedDict()
    for n, v in rows:
        key = n[:150]
        agg.setdefault(key, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{len(rows)} launches, total {tot:.1f} us")
    for n, vs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(vs)/tot*100:5.1f}%  n={len(vs):4d}  mean={sum(vs)/len(vs):7.2f} us  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
