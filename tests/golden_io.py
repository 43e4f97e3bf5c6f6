"""Seeded input generators and loaders for the committed golden fixtures.

Shared by tests/golden/make_golden.py (which ran the reference on these inputs)
and the tests that replay them.  No reference logic lives here.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle.tada_oracle import bf16_round

F32 = np.float32
GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(*arrs) -> str:
    return hashlib.sha256(b"".join(np.ascontiguousarray(a).tobytes() for a in arrs)).hexdigest()


def kv_inputs(seed, sched, hq, h, d):
    """K, V (concatenated over the append schedule) and q for a kv* case."""
    rng = np.random.default_rng(seed)
    n = sum(sched)
    k = rng.normal(size=(n, h, d)).astype(F32)
    v = rng.normal(size=(n, h, d)).astype(F32)
    q = rng.normal(size=(hq, d)).astype(F32)
    return k, v, q


def c1_inputs(hq, seed=1001, tokens=512, heads=8, d=128):
    """BASELINE config 1 inputs: bf16-gridded N(0,1) K, V [512, 8, 128] and q [hq, 128]."""
    rng = np.random.default_rng(seed)
    k = bf16_round(rng.normal(size=(tokens, heads, d)).astype(F32))
    v = bf16_round(rng.normal(size=(tokens, heads, d)).astype(F32))
    q = bf16_round(rng.normal(size=(hq, d)).astype(F32))
    return k, v, q


def split_schedule(x, sched):
    return np.split(x, np.cumsum(sched)[:-1]) if len(sched) > 1 else [x]


_CACHE = {}


def load():
    """(arrays, manifest-cases) from tests/golden/golden.npz + manifest.json."""
    if "g" not in _CACHE:
        arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
        with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
            cases = json.load(f)["cases"]
        _CACHE["g"] = (arrays, cases)
    return _CACHE["g"]


def keys(prefix):
    _, cases = load()
    return sorted(k for k in cases if k.startswith(prefix))


# ---------------------------------------------------------------------- RoPE row (make_golden_rope.py)
ROPE_AF_CHUNKS = (130, 1, 1, 6)  # prefill (crosses R = 128), two decode steps, a chunk


def rope_af_inputs(case: int, bits: int, R: int, h=8, d=128):
    """Per chunk: (k_pre [n, h, d], v [n, h, d], positions), bf16-gridded, for af<case>.

    append_fused (model.py:167-183) is rotate_heads + (x_norm @ w_v) + append_tokens; the fixture feeds
    the value rows directly (the BLAS projection's summation order is host-specific)."""
    rng = np.random.default_rng(8100 + 7 * case + bits + R)
    out, start = [], 0
    for cnt in ROPE_AF_CHUNKS:
        k_pre = bf16_round(rng.normal(size=(cnt, h, d)).astype(F32))
        v = bf16_round(rng.normal(size=(cnt, h, d)).astype(F32))
        out.append((k_pre, v, np.arange(start, start + cnt, dtype=np.int64)))
        start += cnt
    return out


def load_rope():
    """(arrays, manifest-cases) from tests/golden/rope.npz + rope_manifest.json."""
    if "r" not in _CACHE:
        arrays = dict(np.load(os.path.join(GOLDEN_DIR, "rope.npz")))
        with open(os.path.join(GOLDEN_DIR, "rope_manifest.json")) as f:
            cases = json.load(f)["cases"]
        _CACHE["r"] = (arrays, cases)
    return _CACHE["r"]
