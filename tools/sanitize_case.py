"""Small decode-attention + append workload for compute-sanitizer (racecheck / synccheck / memcheck).

python tools/sanitize_case.py --bits 4 --hq 32   (B=2, T=300 incl. tail tiles and empty splits, R=8)
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04642_b200 as tk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--tokens", type=int, default=300)
    ap.add_argument("--residual", type=int, default=8, help="odd values give odd compressed lengths")
    args = ap.parse_args()
    B, T, H, D, R = 2, args.tokens, args.heads, args.dim, args.residual
    rng = np.random.default_rng(1)
    k = torch.from_numpy(rng.normal(size=(B, T, H, D)).astype(np.float32)).cuda().bfloat16()
    v = torch.from_numpy(rng.normal(size=(B, T, H, D)).astype(np.float32)).cuda().bfloat16()
    store = tk.PagedKVCache(1, H, D, (args.bits,), R, batch=B, page_tokens=64, max_tokens=T + 16)
    store.append(0, k, v)
    pos = torch.arange(T, T + 1).repeat(B, 1)
    from paper_2506_04642_b200.rope import _positions

    for step in range(3):
        q = torch.from_numpy(rng.normal(size=(B, args.hq, D)).astype(np.float32)).cuda().bfloat16()
        kn = torch.from_numpy(rng.normal(size=(B, 1, H, D)).astype(np.float32)).cuda().bfloat16()
        vn = torch.from_numpy(rng.normal(size=(B, 1, H, D)).astype(np.float32)).cuda().bfloat16()
        store.append_attend(0, q, kn, vn, out_dtype=torch.bfloat16, num_splits=7, mode=args.mode)
    p, top = _positions((pos + 1).numpy(), 1, B)
    store.append_rope(0, kn, vn, p, top, tk.RopeParams(D))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
