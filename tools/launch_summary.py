"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0][:60]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:60s} n={len(v):4d} total={sum(v)/1e3:9.1f}us ({100*sum(v)/tot:5.1f}%) mean={sum(v)/len(v)/1e3:8.2f}us")


if __name__ == "__main__":
    main()
