"""Tabulate gpurun_out/abk1.log (tools/ab_k1.sh): GB/s per (lib, bits) over the repetitions."""
import collections
import json
import sys

res, lib = collections.defaultdict(list), ""
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/abk1.log"):
    if line.startswith("lib="):
        lib = line.strip()[4:] or "default"
        continue
    try:
        d = json.loads(line)
    except ValueError:
        if line.strip():
            print("!", line.strip()[:160])
        continue
    res[(d["bits"], d.get("rope"), lib)].append(round(d["alg_GBps"]))
for k in sorted(res, key=str):
    print(k, res[k])
