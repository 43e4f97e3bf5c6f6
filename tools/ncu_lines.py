"""Per-source-line instructions and stall samples of an ncu report for one .cu file.
Usage: python tools/ncu_lines.py report.ncu-rep file.cu [N] [tiles]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, path = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    tiles = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    src = open(path).read().splitlines()
    base = path.split("/")[-1]
    file, hdr = None, None
    agg, stall, kinds = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            d = dict(zip(hdr, r))
            try:
                ins = float(d["Instructions Executed"] or 0)
                s = float(d["Warp Stall Sampling (All Samples)"] or 0)
            except ValueError:
                continue
            key = (file, int(d["Line No"]))
            agg[key] += ins
            stall[key] += s
            for k, v in d.items():
                if k.startswith("stall_") and v:
                    try:
                        kinds[key][k[6:]] += float(v)
                    except ValueError:
                        pass
    ti, ts = sum(agg.values()) or 1, sum(stall.values()) or 1
    keys = sorted(set(agg) | set(stall), key=lambda k: -(stall[k] / ts + agg[k] / ti))[:n]
    for k in sorted(keys, key=lambda k: (k[0] != base, k[1])):
        txt = src[k[1] - 1].strip()[:80] if k[0] == base and k[1] <= len(src) else ""
        top = ",".join(f"{a}={b:.0f}" for a, b in kinds[k].most_common(2))
        print(f"{k[0][:16]:16s}:{k[1]:4d} ins {100*agg[k]/ti:4.1f}% ({agg[k]/tiles:6.0f}) stall {100*stall[k]/ts:4.1f}% {top:28s} {txt}")


if __name__ == "__main__":
    main()
