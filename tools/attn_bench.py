"""Single-layer decode-attention micro-benchmark: B sequences x T compressed tokens, one width.

python tools/attn_bench.py --bits 4 --batch 16 --tokens 32768 --hq 32 --mode 2
Prints achieved algorithmic GB/s (SURVEY §8d bytes) for the K2(+K3) launch, CUDA-event timed.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04642_b200 as tk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--layers", type=int, default=4, help="distinct layer pools cycled (defeats L2)")
    ap.add_argument("--reps", type=int, default=5, help="timed repetitions; the median is reported")
    args = ap.parse_args()
    B, T, H, D = args.batch, args.tokens, args.heads, args.dim
    store = tk.PagedKVCache(args.layers, H, D, [args.bits] * args.layers, 128, batch=B, page_tokens=64,
                            max_tokens=T + 130, shuffle_pages=True)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for layer in range(args.layers):
        for b0 in range(0, T, 8192):
            n = min(8192, T - b0)
            k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
            v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
            store.append(layer, k, v)
    q = torch.randn((B, args.hq, D), generator=g, device="cuda").bfloat16()
    out = torch.empty((B, args.hq, D), dtype=torch.bfloat16, device="cuda")
    splits = args.splits or store.suggest_splits(0, args.hq, args.mode)
    for i in range(3):
        store.attend(i % args.layers, q, out=out, num_splits=splits, mode=args.mode)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.iters):
            store.attend(i % args.layers, q, out=out, num_splits=splits, mode=args.mode)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / args.iters)
    times.sort()
    ms = times[len(times) // 2]
    c, r = store.lengths(0)
    tokb = 4 * D + H * (D * args.bits // 8) + 8 * H
    alg = B * (2 * c * tokb + 2 * r * H * D * 2 + 2 * args.hq * D * 2)
    print(json.dumps({"bits": args.bits, "batch": B, "tokens": c + r, "hq": args.hq, "heads": H, "dim": D, "mode": args.mode,
                      "splits": splits, "ms": ms, "ms_min": times[0], "alg_GBps": alg / ms / 1e6}))


if __name__ == "__main__":
    main()
