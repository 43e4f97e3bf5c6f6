"""Drop-in append_tokens timing: the flag-checked append (current) against the same append preceded by the
isfinite pre-pass the round-1 drop-in ran (two full reads of the input, eager reduce kernels, two syncs).

python tools/dropin_append_bench.py --tokens 32768 --bits 4 --iters 5
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04642_b200 as tk  # noqa: E402


def run(k, v, bits, R, prepass):
    cache = tk.CompressedLayerCache(8, 128, bits, R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if prepass:
        for t in (k, v):
            if not bool(torch.isfinite(t).all()):
                raise tk.DataError("non-finite")
    cache.append_tokens(k, v)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--R", type=int, default=128)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    k = torch.randn((a.tokens, 8, 128), generator=g, device="cuda").bfloat16()
    v = torch.randn((a.tokens, 8, 128), generator=g, device="cuda").bfloat16()
    out = {"tokens": a.tokens, "bits": a.bits, "R": a.R}
    for name, pre in (("checked_ms", False), ("prepass_ms", True)):
        ts = [run(k, v, a.bits, a.R, pre) for _ in range(a.iters + 2)][2:]
        out[name] = sorted(ts)[len(ts) // 2]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
