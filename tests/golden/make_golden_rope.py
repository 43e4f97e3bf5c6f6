"""Golden vectors for the RoPE + compress row, generated from the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_rope.py

Writes ``tests/golden/rope.npz`` + ``tests/golden/rope_manifest.json``:

* ``ar*``  tadakv.tensor.apply_rope on (tokens, D) rows: D in {2, 8, 64, 128}, bases 1e4 / 5e5,
  positions up to 131071, f32 and bf16-gridded inputs.
* ``rh*``  tadakv.tensor.rotate_heads on (tokens, H, D).
* ``af*``  append_fused's cache effect (model.py:176-178: rotate_heads, then append_tokens) into a
  CompressedLayerCache (H=8, D=128, widths 2/4/8, R in {0, 128}, chunks 130/1/1/6 from
  tests/golden_io.rope_af_inputs, the value rows given directly since the BLAS projection's
  summation order is host-specific) -> sha256 of the TADAKV1 bytes.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from tadakv import cache as ref_cache  # noqa: E402
from tadakv import tensor as ref_tensor  # noqa: E402

from oracle.tada_oracle import bf16_round  # noqa: E402

sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..")))
from golden_io import ROPE_AF_CHUNKS, rope_af_inputs  # noqa: E402  (seeded generators, no reference logic)

F32 = np.float32


def main():
    rng = np.random.default_rng(8001)
    arrays: dict[str, np.ndarray] = {}
    manifest: dict[str, dict] = {}
    n = 0
    for d in (2, 8, 64, 128):
        for base in (10000.0, 500000.0):
            for grid in (False, True):
                t = 37
                x = rng.normal(size=(t, d)).astype(F32) * F32(3.0)
                if grid:
                    x = bf16_round(x)
                pos = np.concatenate([np.arange(5), rng.integers(0, 131072, size=t - 5)]).astype(np.int64)
                y = ref_tensor.apply_rope(x, pos, ref_tensor.RopeParams(d, base))
                key = f"ar{n:02d}"
                arrays[f"{key}/x"], arrays[f"{key}/pos"], arrays[f"{key}/y"] = x, pos, y
                manifest[key] = {"head_dim": d, "base": base, "bf16_grid": grid, "tokens": t}
                n += 1
    for i, (t, h, d) in enumerate([(9, 8, 128), (3, 2, 16), (64, 8, 128)]):
        x = bf16_round(rng.normal(size=(t, h, d)).astype(F32))
        pos = rng.integers(0, 40000, size=t).astype(np.int64)
        y = ref_tensor.rotate_heads(x, pos, ref_tensor.RopeParams(d))
        key = f"rh{i:02d}"
        arrays[f"{key}/x"], arrays[f"{key}/pos"], arrays[f"{key}/y"] = x, pos, y
        manifest[key] = {"shape": [t, h, d]}
    n = 0
    for bits in (2, 4, 8):
        for R in (0, 128):
            h, d = 8, 128
            rope = ref_tensor.RopeParams(d)
            cache = ref_cache.CompressedLayerCache(h, d, bits, R)
            for k_pre, v, pos in rope_af_inputs(n, bits, R, h, d):
                # append_fused (model.py:176-178) with the projection result given
                cache.append_tokens(ref_tensor.rotate_heads(k_pre, pos, rope), v)
            blob = ref_cache.serialize_cache(cache)
            manifest[f"af{n:02d}"] = {"bits": bits, "R": R, "chunks": list(ROPE_AF_CHUNKS), "bytes": len(blob),
                                      "sha256": hashlib.sha256(blob).hexdigest()}
            n += 1
    np.savez_compressed(os.path.join(HERE, "rope.npz"), **arrays)
    with open(os.path.join(HERE, "rope_manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_rope.py", "reference": REF_SRC,
                   "numpy": np.__version__, "cases": manifest}, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(manifest)} cases")


if __name__ == "__main__":
    main()
