"""Golden precision-search results, generated from the REFERENCE ``tadakv.search``.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_search.py

Writes ``tests/golden/search.json``: for seeded toy models (weights regenerated in the tests by
oracle.tada_oracle.toy_weights, pinned by tests/golden/decoder_manifest.json-style hashes here too) and
synthetic calibration sets, the reference's ``score_plan`` of a few fixed plans, ``uncompressed_nll``,
and the full ``random_search`` report (report_to_json) with and without a memory budget.
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
from tadakv import search as ref_search  # noqa: E402
from tadakv import tensor as ref_tensor  # noqa: E402

CASES = [
    # name, layers, hq, h, d, vocab, seed, R, calib (n, length, seed), candidates, search seed, budget
    ("s4", 4, 8, 2, 16, 128, 31, 8, (3, 12, 5), 10, 1, None),
    ("s4b", 4, 8, 2, 16, 128, 31, 8, (3, 12, 5), 10, 1, 0.82),
    ("s6", 6, 8, 4, 16, 96, 77, 4, (2, 10, 9), 8, 3, None),
]


def main():
    out = {}
    for name, layers, hq, h, d, vocab, seed, R, (ncal, length, cseed), ncand, sseed, budget in CASES:
        cfg = ref_cache.ModelConfig(layers, hq, h, d, R, ref_tensor.RopeParams(d),
                                    ref_cache.PrecisionPlan.uniform(4, layers))
        model = ref_model.random_model(cfg, vocab_size=vocab, seed=seed)
        calib = ref_search.CalibrationSet.synthetic(vocab, ncal, length, cseed)
        plans = [ref_cache.PrecisionPlan.uniform(b, layers) for b in (2, 4, 8)]
        _, report = ref_search.random_search(
            ref_search.SearchConfig(num_candidates=ncand, seed=sseed, memory_budget=budget), calib, model)
        out[name] = {
            "model": {"layers": layers, "hq": hq, "h": h, "d": d, "vocab": vocab, "seed": seed, "R": R},
            "calib": [list(s) for s in calib.sequences],
            "search": {"num_candidates": ncand, "seed": sseed, "memory_budget": budget},
            "score_plan": {str(list(p.bits_per_layer)): ref_search.score_plan(p, calib, model) for p in plans},
            "uncompressed_nll": ref_search.uncompressed_nll(calib, model),
            "report": json.loads(ref_search.report_to_json(report)),
            "report_csv": ref_search.report_to_csv(report),
            "weight_sha256": {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
                              for k, v in sorted(model.weights.items())},
        }
    with open(os.path.join(HERE, "search.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_search.py", "reference": REF_SRC, "numpy": np.__version__,
                   "cases": out}, f, indent=1, sort_keys=True)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
