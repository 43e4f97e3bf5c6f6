"""Golden outputs of the reference toy decoder, generated from ``tadakv`` itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_decoder.py

Writes ``tests/golden/decoder.npz`` + ``tests/golden/decoder_manifest.json``.  For each case a seeded
``random_model`` (model.py:89-150) runs ``generate`` (model.py:292-330) on a fixed prompt; stored are the
greedy tokens, the prompt's prefill logits and the sha256 of every weight array (the tests regenerate
the weights with oracle.tada_oracle.toy_weights and check those hashes first).

Cases: AC3 (test_acceptance.py:129-143: 4 layers, 8 q / 2 kv heads, D=16, all-residual R=256, 2-bit
plan) and compressed decoding with R=4 at widths 2 and 4 and a mixed plan, plus a wider GQA model
(Hq=16, H=8, D=128) that exercises the fused RoPE append, and 4 / 16 KV-head models (Qwen2-style and MHA).
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

from tadakv import cache as ref_cache  # noqa: E402
from tadakv import model as ref_model  # noqa: E402
from tadakv import tensor as ref_tensor  # noqa: E402

CASES = [
    # name, layers, hq, h, d, vocab, seed, prompt, max_new, plan, R
    ("ac3", 4, 8, 2, 16, 256, 2024, [11, 47, 3], 64, [2, 2, 2, 2], 256),
    ("r4b2", 4, 8, 2, 16, 256, 2024, [11, 47, 3], 40, [2, 2, 2, 2], 4),
    ("r4b4", 4, 8, 2, 16, 256, 7, [5, 9, 200, 31, 77], 40, [4, 4, 4, 4], 4),
    ("mixed", 4, 8, 2, 16, 256, 11, [1, 2, 3, 4, 5, 6, 7, 8, 9], 32, [8, 4, 2, 4], 8),
    ("wide", 2, 16, 8, 128, 512, 3, [17, 400, 3, 99], 24, [4, 2], 16),
    # round 2: KV head counts other than 8 on the tensor-core path (Qwen2-style 4 KV / 28 q heads; 16-head MHA)
    ("qwen", 2, 28, 4, 128, 512, 5, [9, 300, 41, 7, 120], 24, [4, 2], 16),
    ("mha16", 2, 16, 16, 128, 512, 6, [2, 77, 301], 24, [2, 4], 16),
]


def main():
    arrays, manifest = {}, {}
    for name, layers, hq, h, d, vocab, seed, prompt, max_new, plan, R in CASES:
        cfg = ref_cache.ModelConfig(layers, hq, h, d, R, ref_tensor.RopeParams(d),
                                    ref_cache.PrecisionPlan(tuple(plan)))
        model = ref_model.random_model(cfg, vocab_size=vocab, seed=seed)
        tokens = ref_model.generate(model, prompt, max_new)
        logits = ref_model.reference_forward(model, prompt)
        arrays[f"{name}/tokens"] = np.asarray(tokens, dtype=np.int64)
        arrays[f"{name}/prefill_logits"] = logits.astype(np.float32)
        manifest[name] = {
            "layers": layers, "hq": hq, "h": h, "d": d, "vocab": vocab, "seed": seed, "prompt": prompt,
            "max_new": max_new, "plan": plan, "R": R,
            "weight_sha256": {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
                              for k, v in sorted(model.weights.items())},
        }
        if name == "ac3":
            manifest[name]["reference_generate_equal"] = tokens == ref_model.reference_generate(model, prompt, max_new)
    np.savez_compressed(os.path.join(HERE, "decoder.npz"), **arrays)
    with open(os.path.join(HERE, "decoder_manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_decoder.py", "reference": REF_SRC, "numpy": np.__version__,
                   "cases": manifest}, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(manifest)} cases")


if __name__ == "__main__":
    main()
