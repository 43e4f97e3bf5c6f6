"""Run the reference's own test suite against the drop-in.

``test_quant.py``, ``test_cache.py``, ``test_attention.py``, ``test_acceptance.py`` and ``util.py`` here are
the reference's files (pkg/tests, tadakv 0.1.0) unchanged apart from a provenance header.  This conftest
makes ``import tadakv...`` resolve to ``paper_2506_04642_b200`` before they are collected:

* ``tadakv``, ``tadakv.quant``, ``tadakv.cache``, ``tadakv.attention``, ``tadakv.errors``, ``tadakv.search``
  -> the drop-in modules of the same names (the hot path on the B200: K1 quantize / append, K2/K3 attention,
  the GPU precision search);
* ``tadakv.tensor`` -> the drop-in's ``RopeParams`` / ``apply_rope`` / ``rotate_heads`` (K1's RoPE), plus the
  reference's numpy utilities ``matmul`` / ``softmax_rows`` / ``as_f32`` restated here (not on the path);
* ``tadakv.model`` -> ``random_model`` = the oracle's seeded toy weights (pinned to the reference's weight
  hashes) wrapped as ``search.ToyWeights``; ``generate`` / ``append_fused`` = the drop-in's GPU decoder and fused
  append; ``reference_generate`` = the reference's recorded output for the one case AC3 runs
  (tests/golden/decoder.npz, written by the reference itself);
* ``tadakv.analysis`` -> ``shared_outlier_activations`` (oracle restatement) and ``centered_reconstruction``
  composed from the drop-in's mean_center / quantize_tensor / dequantize_tensor.

What is outside the KV path raises ``pytest.skip`` naming the reason when called: the CLI
(AC1), the ablation study (AC6), outlier-channel toy models, the TADAW1 weights container (second half of
AC9) and prefill attention on raw activations.  Every test here needs the GPU (marker ``gpu``).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import types

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
TESTS = os.path.dirname(HERE)
if HERE not in sys.path:
    sys.path.insert(0, HERE)

import paper_2506_04642_b200 as dropin  # noqa: E402
from paper_2506_04642_b200 import attention, cache, errors, quant, rope, search  # noqa: E402
from paper_2506_04642_b200.decoder import generate as _gpu_generate  # noqa: E402

from oracle import tada_oracle as orc  # noqa: E402

F32 = np.float32


def _out_of_scope(what: str):
    def stub(*args, **kwargs):
        pytest.skip(f"{what} is outside the KV-cache hot path this drop-in replaces (DESIGN.md §7)")

    stub.__name__ = what
    return stub


def _module(name: str, base=None, **extra) -> types.ModuleType:
    m = types.ModuleType(name)
    if base is not None:
        m.__dict__.update({k: v for k, v in vars(base).items() if not k.startswith("__")})
    m.__dict__.update(extra)
    m.__path__ = []  # importable as a package parent
    sys.modules[name] = m
    return m


# ---------------------------------------------------------------- tadakv.tensor (utilities off the path)
def _as_f32(x):
    return np.ascontiguousarray(x, dtype=F32)


def _matmul(a, b):
    a, b = _as_f32(a), _as_f32(b)
    if a.ndim != 2 or b.ndim != 2:
        raise errors.ShapeError(f"matmul expects 2-D operands, got {a.ndim}-D and {b.ndim}-D")
    if a.shape[1] != b.shape[0]:
        raise errors.ShapeError(f"inner dimensions disagree: {a.shape} x {b.shape}")
    return a @ b


def _softmax_rows(a):
    a = _as_f32(a)
    if a.ndim != 2:
        raise errors.ShapeError(f"softmax_rows expects a 2-D tensor, got {a.ndim}-D")
    e = np.exp(a - a.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


# ---------------------------------------------------------------- tadakv.model
def _random_model(cfg, vocab_size, *, seed, max_seq_len=4096, identical_kv_heads=False, outlier_channels=0,
                  outlier_scale=8.0, outlier_jitter=0.05):
    if outlier_channels:
        pytest.skip("outlier-channel toy models (analysis ablation, AC6) are outside the KV path (DESIGN.md §7)")
    w = orc.toy_weights(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, vocab_size, seed,
                        identical_kv_heads=identical_kv_heads)
    return search.ToyWeights(cfg, vocab_size, w, max_seq_len=max_seq_len)


def _generate(model, prompt_ids, max_new_tokens, *, plan=None, residual_length=None, block=None):
    return _gpu_generate(model.weights, model.cfg, model.vocab_size, list(prompt_ids), max_new_tokens, plan=plan,
                         residual_length=residual_length, max_seq_len=model.max_seq_len)


def _weights_digest(w) -> dict:
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in sorted(w.items())}


def _reference_generate(model, prompt_ids, max_new_tokens):
    """The reference's own uncompressed generation, recorded by tests/golden/make_golden_decoder.py for the
    case it ran (AC3's toy model); any other input is out of scope here."""
    with open(os.path.join(TESTS, "golden", "decoder_manifest.json")) as f:
        cases = json.load(f)["cases"]
    digest = _weights_digest(model.weights)
    for name, c in cases.items():
        if (c.get("reference_generate_equal") and list(prompt_ids) == c["prompt"] and max_new_tokens == c["max_new"]
                and digest == c["weight_sha256"]):
            return [int(t) for t in np.load(os.path.join(TESTS, "golden", "decoder.npz"))[f"{name}/tokens"]]
    pytest.skip("reference_generate (uncompressed numpy decoding) is outside the KV path; no recorded output "
                "for this input")


# ---------------------------------------------------------------- tadakv.analysis
def _shared_outlier_activations(rng, tokens, heads, head_dim, *, outlier_channels=2, outlier_scale=8.0,
                                noise_scale=0.1):
    return orc.outlier_activations(rng, tokens, heads, head_dim, channels=outlier_channels, scale=outlier_scale,
                                   noise=noise_scale)


def _centered_reconstruction(x, bits):
    mean, dev = cache.mean_center(x)
    return mean[:, None, :] - quant.dequantize_tensor(quant.quantize_tensor(dev, bits))


_module("tadakv", dropin)
_module("tadakv.quant", quant)
_module("tadakv.cache", cache)
_module("tadakv.errors", errors)
_module("tadakv.search", search)
_module("tadakv.attention", attention, prefill_attend=_out_of_scope("prefill_attend (raw-activation prompt attention)"))
_module("tadakv.tensor", None, RopeParams=cache.RopeParams, apply_rope=rope.apply_rope, rotate_heads=rope.rotate_heads,
        matmul=_matmul, softmax_rows=_softmax_rows, as_f32=_as_f32)
_module("tadakv.model", None, ToyModel=search.ToyWeights, random_model=_random_model, generate=_generate,
        append_fused=rope.append_fused, reference_generate=_reference_generate,
        weights_to_bytes=_out_of_scope("the TADAW1 weights container"),
        weights_from_bytes=_out_of_scope("the TADAW1 weights container"))
_module("tadakv.analysis", None, shared_outlier_activations=_shared_outlier_activations,
        centered_reconstruction=_centered_reconstruction, ablate_frobenius=_out_of_scope("the Frobenius ablation"))
_module("tadakv.cli", None, cli_main=_out_of_scope("the tadakv command line"))


def pytest_collection_modifyitems(config, items):
    import torch

    skip = None if torch.cuda.is_available() else pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if str(item.fspath).startswith(HERE):
            item.add_marker(pytest.mark.gpu)
            if skip is not None:
                item.add_marker(skip)


@pytest.fixture(scope="session")
def toy_cfg():
    """conftest.py:8-20 of the reference: 4 layers, 8 query heads, 2 KV heads, head_dim 16."""
    from util import make_cfg

    return make_cfg(num_layers=4, num_q_heads=8, num_kv_heads=2, head_dim=16, residual_length=4,
                    plan=cache.PrecisionPlan.uniform(4, 4))


@pytest.fixture(scope="session")
def toy_model(toy_cfg):
    return _random_model(toy_cfg, vocab_size=256, seed=2024)
