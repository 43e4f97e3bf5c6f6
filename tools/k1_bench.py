"""Bulk quantize-append micro-benchmark (config 3 shape per layer): B sequences x T tokens, one width.

python tools/k1_bench.py --bits 4 --batch 8 --tokens 32768
Prints algorithmic GB/s: read B*T*H*D*2*2 (bf16 K and V) + write B*T*2*(4D + H*D*b/8 + 8H).
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
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--rope", action="store_true", help="fused RoPE of the keys (tada_quant_append_rope)")
    ap.add_argument("--rope-composed", action="store_true",
                    help="unfused: tada_apply_rope to an f32 copy in HBM, then tada_quant_append")
    args = ap.parse_args()
    B, T, H, D = args.batch, args.tokens, 8, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    k = torch.randn((B, T, H, D), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, T, H, D), generator=g, device="cuda").bfloat16()
    if args.rope or args.rope_composed:
        from paper_2506_04642_b200.rope import _positions

        pos, top = _positions(torch.arange(T).repeat(B, 1), T, B)
        rope = tk.RopeParams(D, 500000.0)
    times = []
    for it in range(args.iters + 2):
        store = tk.PagedKVCache(1, H, D, [args.bits], 0, batch=B, page_tokens=64, max_tokens=T, shuffle_pages=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if args.rope:
            store.append_rope(0, k, v, pos, top, rope)
        elif args.rope_composed:
            store.append(0, store._rotate(k, pos, tk.rope_table(rope, top)), v.float())
        else:
            store.append(0, k, v)
        e1.record()
        e1.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
        del store
    ms = sorted(times)[len(times) // 2]
    tokb = 4 * D + H * D * args.bits // 8 + 8 * H
    alg = B * T * (H * D * 2 * 2 + 2 * tokb)
    print(json.dumps({"bits": args.bits, "batch": B, "tokens": T, "rope": "fused" if args.rope else ("composed" if args.rope_composed else None), "ms": ms,
                      "alg_GBps": alg / ms / 1e6}))


if __name__ == "__main__":
    main()
