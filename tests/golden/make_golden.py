"""Generate golden vectors for the TaDA hot path from the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``tadakv`` read-only from /root/reference/pkg/src, runs it on seeded
inputs, and writes ``tests/golden/golden.npz`` + ``tests/golden/manifest.json``.
The fixtures are committed; nothing at test/bench time reads /root/reference.

Cases (each key prefix in golden.npz is ``<case-id>/``):

* ``q*``  quantize_tensor / dequantize_tensor on (t, H, D) deviations of many
  widths and group sizes, incl. constants, exact ramps, .5 ties, wide scale mix.
* ``mc*`` mean_center on f32 and bf16-gridded activations.
* ``kv*`` CompressedLayerCache append schedules -> TADAKV1 bytes (serialize_cache).
* ``at*`` attend_streaming / attend_naive outputs over those caches.
* ``c1*`` BASELINE config 1: H=8, D=128, T=512, 4-bit, bf16-gridded N(0,1),
  seed 1001, R in {0, 128}, Hq in {8, 32}; blob sha256 + attention outputs.
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

from tadakv import attention as ref_attn  # noqa: E402
from tadakv import cache as ref_cache  # noqa: E402
from tadakv import quant as ref_quant  # noqa: E402
from tadakv.analysis import shared_outlier_activations  # noqa: E402

sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..")))
from golden_io import c1_inputs, kv_inputs, sha  # noqa: E402  (seeded generators, no reference logic)
from oracle.tada_oracle import bf16_round  # noqa: E402

F32 = np.float32


def u8(b: bytes) -> np.ndarray:
    return np.frombuffer(b, dtype=np.uint8).copy()


def quant_inputs():
    rng = np.random.default_rng(7001)
    cases = []
    for bits in (2, 4, 8, 16):
        for (t, h, d) in [(3, 2, 1), (4, 3, 3), (5, 2, 5), (2, 2, 7), (6, 4, 16), (3, 2, 33), (9, 8, 128), (2, 2, 256)]:
            cases.append((bits, rng.normal(size=(t, h, d)).astype(F32), "normal"))
        mix = rng.choice([0.01, 1.0, 50.0], size=(64, 1, 1))
        cases.append((bits, (rng.normal(size=(64, 1, 16)) * mix).astype(F32), "scale-mix"))
        cases.append((bits, np.full((2, 3, 8), -3.5, F32), "constant"))
        cases.append((bits, np.zeros((3, 2, 8), F32), "zeros"))
        # .5 ties: values on a 1/8 grid with span chosen so (x-min)/scale hits k+0.5
        lv = (1 << min(bits, 8)) - 1
        base = rng.integers(-8, 8, size=(16, 2, 1)).astype(F32)
        grid = rng.integers(0, 2 * lv + 1, size=(16, 2, 32)).astype(F32) * F32(0.5)
        grid[:, :, 0] = 0
        grid[:, :, 1] = lv
        cases.append((bits, base + grid, "ties"))
        cases.append((bits, bf16_round(rng.normal(size=(12, 8, 128)).astype(F32)), "bf16-grid"))
        cases.append((bits, shared_outlier_activations(rng, tokens=16, heads=8, head_dim=128), "outlier"))
    return cases


def main():
    arrays: dict[str, np.ndarray] = {}
    manifest: dict[str, dict] = {}

    # ---- quantizer
    for i, (bits, dev, kind) in enumerate(quant_inputs()):
        key = f"q{i:03d}"
        q = ref_quant.quantize_tensor(dev, bits)
        arrays[f"{key}/input"] = dev
        arrays[f"{key}/codes"] = u8(q.codes)
        arrays[f"{key}/scales"] = q.scales
        arrays[f"{key}/mins"] = q.mins
        arrays[f"{key}/deq"] = ref_quant.dequantize_tensor(q)
        manifest[key] = {"kind": kind, "bits": bits, "shape": list(dev.shape)}

    # ---- mean_center
    rng = np.random.default_rng(7002)
    for i, (t, h, d, grid) in enumerate([(5, 1, 8, False), (7, 2, 16, False), (4, 3, 16, False), (6, 5, 32, False),
                                         (16, 8, 128, False), (16, 8, 128, True), (3, 7, 64, True)]):
        key = f"mc{i:02d}"
        x = rng.normal(size=(t, h, d)).astype(F32)
        if grid:
            x = bf16_round(x)
        m, dv = ref_cache.mean_center(x)
        arrays[f"{key}/input"] = x
        arrays[f"{key}/mean"] = m
        arrays[f"{key}/dev"] = dv
        manifest[key] = {"shape": [t, h, d], "bf16_grid": grid}

    # ---- cache append schedules + attention
    rng = np.random.default_rng(7003)
    specs = []
    for bits in (2, 4, 8, 16):
        for (hq, h, d, R) in [(4, 2, 16, 4), (8, 2, 16, 0), (6, 3, 8, 3), (4, 4, 4, 5), (32, 8, 128, 128), (16, 8, 64, 16)]:
            specs.append((bits, hq, h, d, R))
    for i, (bits, hq, h, d, R) in enumerate(specs):
        key = f"kv{i:02d}"
        cache = ref_cache.CompressedLayerCache(h, d, bits, R)
        hi = 2 * max(R, 4) + 3 if d < 128 else R + 40
        sched = [int(x) for x in rng.integers(0, hi, size=5 if d < 128 else 3)]
        seed = 9000 + i
        k, v, q = kv_inputs(seed, sched, hq, h, d)
        for a, b in zip(np.split(k, np.cumsum(sched)[:-1]), np.split(v, np.cumsum(sched)[:-1])):
            cache.append_tokens(a, b)
        total = sum(sched)
        blob = ref_cache.serialize_cache(cache)
        if len(blob) < 300_000:
            arrays[f"{key}/blob"] = u8(blob)
        manifest[key] = {"bits": bits, "hq": hq, "h": h, "d": d, "R": R, "schedule": sched, "seed": seed,
                         "input_sha256": sha(k, v, q), "blob_sha256": hashlib.sha256(blob).hexdigest(),
                         "blob_len": len(blob)}
        if total:
            cfg = ref_cache.ModelConfig(1, hq, h, d, R, ref_cache.RopeParams(d), ref_cache.PrecisionPlan((bits,)))
            arrays[f"{key}/q"] = q
            arrays[f"{key}/attn_stream64"] = ref_attn.attend_streaming(q, cache, cfg, ref_attn.BlockSpec(64)).output
            arrays[f"{key}/attn_stream3"] = ref_attn.attend_streaming(q, cache, cfg, ref_attn.BlockSpec(3)).output
            arrays[f"{key}/attn_naive"] = ref_attn.attend_naive(q, cache, cfg).output

    # ---- BASELINE config 1
    for hq in (8, 32):
        for R in (0, 128):
            key = f"c1_hq{hq}_r{R}"
            k, v, q = c1_inputs(hq)
            cache = ref_cache.CompressedLayerCache(8, 128, 4, R)
            cache.append_tokens(k, v)
            blob = ref_cache.serialize_cache(cache)
            cfg = ref_cache.ModelConfig(1, hq, 8, 128, R, ref_cache.RopeParams(128), ref_cache.PrecisionPlan((4,)))
            arrays[f"{key}/attn_stream64"] = ref_attn.attend_streaming(q, cache, cfg).output
            arrays[f"{key}/k_scales"] = cache.k_dev.scales[:4096]
            manifest[key] = {
                "seed": 1001, "hq": hq, "R": R, "bits": 4,
                "input_sha256": sha(k, v, q),
                "blob_sha256": hashlib.sha256(blob).hexdigest(),
                "blob_len": len(blob),
            }

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "tadakv 0.1.0 (/root/reference/pkg)",
                   "numpy": np.__version__, "cases": manifest}, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(manifest)} cases")


if __name__ == "__main__":
    main()
