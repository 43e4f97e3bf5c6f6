"""Tabulate gpurun_out/ab.log (tools/ab_attn.sh): GB/s per (lib, bits, hq) over the repetitions."""
import collections
import json
import sys

res, lib = collections.defaultdict(list), ""
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.log"):
    if line.startswith("lib="):
        lib = line.strip()[4:] or "default"
        continue
    try:
        d = json.loads(line)
    except ValueError:
        if line.strip():
            print("!", line.strip()[:120])
        continue
    res[(d["bits"], d["hq"], lib)].append(round(d["alg_GBps"]))
for k in sorted(res):
    print(k, res[k])
