"""Summarise an ncu --page source --csv export (CUDA-source level): top lines by stall samples
and by excessive shared-memory wavefronts.  Usage: python tools/ncu_source_summary.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    rows, file = [], None
    lines = out.splitlines()
    i = 0
    while i < len(lines):
        ln = lines[i]
        if ln.startswith('"File Path"'):
            file = ln.split(",", 1)[1].strip('"')
            i += 1
            continue
        if ln.startswith('"Line No"'):
            hdr = next(csv.reader([ln]))
            hdr[1] = "Source"
            i += 1
            while i < len(lines) and not lines[i].startswith('"File Path"'):
                vals = next(csv.reader([lines[i]]))
                if len(vals) == len(hdr) and vals[0]:  # CUDA-line rows carry the aggregated metrics
                    rows.append((file, dict(zip(hdr, vals))))
                i += 1
            continue
        i += 1

    def num(d, k):
        try:
            return float(d.get(k, "0") or 0)
        except ValueError:
            return 0.0

    tot = sum(num(d, "Warp Stall Sampling (All Samples)") for _, d in rows) or 1
    print(f"total stall samples {tot:.0f}")
    print("--- top lines by stall samples")
    for f, d in sorted(rows, key=lambda x: -num(x[1], "Warp Stall Sampling (All Samples)"))[:n]:
        s = num(d, "Warp Stall Sampling (All Samples)")
        stalls = {k[6:]: num(d, k) for k in d if k.startswith("stall_") and "Not Issued" not in k}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        print(f"{100*s/tot:5.1f}% {f.split('/')[-1]}:{d['Line No']:>4} {d['Source'].strip()[:70]:70s} "
              + " ".join(f"{k}={v:.0f}" for k, v in top))
    itot = sum(num(d, "Instructions Executed") for _, d in rows) or 1
    print(f"--- top lines by warp instructions executed (total {itot:.0f})")
    for f, d in sorted(rows, key=lambda x: -num(x[1], "Instructions Executed"))[:n]:
        print(f"{100*num(d, 'Instructions Executed')/itot:5.1f}% {f.split('/')[-1]}:{d['Line No']:>4} "
              f"{d['Source'].strip()[:90]}")
    print("--- top lines by excessive shared wavefronts")
    for f, d in sorted(rows, key=lambda x: -num(x[1], "L1 Wavefronts Shared Excessive"))[:12]:
        print(f"{num(d, 'L1 Wavefronts Shared Excessive'):12.0f} / {num(d, 'L1 Wavefronts Shared'):12.0f} "
              f"{f.split('/')[-1]}:{d['Line No']:>4} {d['Source'].strip()[:80]}")


if __name__ == "__main__":
    main()
