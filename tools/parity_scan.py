"""Attention error of library variants at a long context against the oracle (GPU box; A/B experiments).

python tools/parity_scan.py --bits 2 --tokens 131072 --hq 32 --variants default variants/rc0/libtadakv_b200.so ...
The parent builds the bf16 inputs and the oracle's attend once; each variant runs in a subprocess with
TADA_LIB_PATH pointing at its library and reports the max-abs error of mode 2 (bf16 and f32 out).
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(path, bits, hq, splits):
    import torch

    import paper_2506_04642_b200 as tk

    z = np.load(path)
    k, v, q = z["k"], z["v"], z["q"]
    B, n, H, D = k.shape
    store = tk.PagedKVCache(1, H, D, (bits,), 128, batch=B, page_tokens=64, max_tokens=n + 8, shuffle_pages=True)
    store.append(0, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16())
    qd = torch.from_numpy(q).cuda().bfloat16()
    o16 = store.attend(0, qd, out_dtype=torch.bfloat16, num_splits=splits or None).float().cpu().numpy()
    o32 = store.attend(0, qd, out_dtype=torch.float32, num_splits=splits or None).cpu().numpy()
    np.savez(path + ".out.npz", o16=o16, o32=o32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--variants", nargs="+", default=["default"])
    ap.add_argument("--child", default="")
    args = ap.parse_args()
    if args.child:
        child(args.child, args.bits, args.hq, args.splits)
        return
    from oracle import tada_oracle as orc

    rng = np.random.default_rng(77)
    n = args.tokens + 37
    k = orc.bf16_round(rng.normal(size=(1, n, 8, 128)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(1, n, 8, 128)).astype(np.float32))
    q = orc.bf16_round(rng.normal(size=(1, args.hq, 128)).astype(np.float32))
    st = orc.LayerState(8, 128, args.bits, 128)
    orc.append(st, k[0], v[0])
    want = orc.attend(q[0], st, args.hq)[0]
    path = os.path.join(tempfile.mkdtemp(), "in.npz")
    np.savez(path, k=k, v=v, q=q)
    for var in args.variants:
        env = dict(os.environ)
        if var != "default":
            env["TADA_LIB_PATH"] = os.path.abspath(var)
        subprocess.run([sys.executable, __file__, "--child", path, "--bits", str(args.bits), "--hq", str(args.hq),
                        "--splits", str(args.splits)], env=env, check=True)
        z = np.load(path + ".out.npz")
        print(json.dumps({"variant": var, "bits": args.bits, "tokens": n, "hq": args.hq,
                          "max_abs_bf16": float(np.abs(z["o16"][0] - want).max()),
                          "max_abs_f32": float(np.abs(z["o32"][0] - want).max()),
                          "out_absmax": float(np.abs(want).max())}), flush=True)


if __name__ == "__main__":
    main()
