"""CPU tests: the C-ABI library loads and exports every symbol include/tadakv_b200.h declares,
host-only entry points answer correctly, and the Python host logic (configs, plans,
memory accounting, TADAKV1 parsing errors) mirrors the reference.  No GPU needed."""

import ctypes
import os
import re
import struct

import pytest

from paper_2506_04642_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tadakv_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tada_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.tada_abi_version() == 1


def test_host_only_entry_points():
    lib = _lib.load()
    assert lib.tada_bytes_per_group(128, 4) == 64
    assert lib.tada_bytes_per_group(5, 2) == 2
    assert lib.tada_bytes_per_group(33, 8) == 33
    assert lib.tada_bytes_per_group(16, 16) == 64
    assert lib.tada_bytes_per_group(16, 3) == -1
    lay = _lib.page_layout(64, 8, 128, 4)
    assert lay.group_bytes == 64
    offs = [lay.off_mean[0], lay.off_codes[0], lay.off_meta[0], lay.off_mean[1], lay.off_codes[1], lay.off_meta[1]]
    assert offs == sorted(offs) and all(o % 128 == 0 for o in offs)
    assert offs[1] - offs[0] >= 64 * 128 * 4 and offs[2] - offs[1] >= 64 * 8 * 64
    assert lay.page_bytes % 256 == 0 and lay.page_bytes >= offs[5] + 64 * 8 * 8
    with pytest.raises(_lib.ConfigError):
        _lib.page_layout(64, 8, 128, 3)
    # partial slots = splits + 1 (the residual rows get their own slot on the tensor-core path), doubled for
    # the padded q heads of a remapped group size, plus their staged q / outputs / lse
    def ws(b, hq, d, s):  # views of 8 KV heads x <= 8 padded q heads: <= 64 q rows per sequence
        return b * max(hq, 64) * (s + 1) * (d + 2) * 4 + b * 64 * (2 * d + 1) * 4 + 256
    assert lib.tada_decode_attn_workspace_bytes(16, 32, 128, 1) == ws(16, 32, 128, 1)
    assert lib.tada_decode_attn_workspace_bytes(16, 32, 128, 8) == ws(16, 32, 128, 8)
    assert 1 <= lib.tada_decode_attn_suggest_splits(16, 32768, 64) <= 4096
    # argument validation happens before any device work
    rc = lib.tada_quantize_groups(None, 0, 10, 16, 3, None, None, None, None, None)
    assert rc == 2 and b"bit width" in lib.tada_last_error()


def test_plan_and_config_validation():
    import paper_2506_04642_b200 as m

    plan = m.PrecisionPlan.uniform(4, 5)
    assert plan.bits_per_layer == (4, 4, 4, 4, 4) and plan.mean_bits == 4.0
    with pytest.raises(m.ConfigError):
        m.PrecisionPlan((4, 3))
    with pytest.raises(m.ConfigError):
        m.PrecisionPlan(())
    rope = m.RopeParams(16)
    with pytest.raises(m.ConfigError):
        m.ModelConfig(1, 6, 4, 16, 0, rope, m.PrecisionPlan((4,)))
    with pytest.raises(m.ConfigError):
        m.ModelConfig(3, 4, 2, 16, 0, rope, m.PrecisionPlan((4, 4)))
    with pytest.raises(m.ConfigError):
        m.ModelConfig(1, 2, 2, 16, 0, m.RopeParams(8), m.PrecisionPlan((4,)))
    with pytest.raises(m.ConfigError):
        m.BlockSpec(0)
    assert [m.kv_head_index(g, 8, 2) for g in range(8)] == [0, 0, 0, 0, 1, 1, 1, 1]


def test_memory_ratio_known_answers():
    """cache.py:216-239 via test_cache.py:211-251 and acceptance criterion 1."""
    import paper_2506_04642_b200 as m

    def cfg(hq, h, d, R, plan):
        return m.ModelConfig(len(plan), hq, h, d, R, m.RopeParams(d), m.PrecisionPlan(tuple(plan)))

    assert m.memory_ratio(cfg(32, 32, 128, 0, [4]), 1024) == 0.296875
    assert m.memory_ratio(cfg(32, 32, 128, 0, [4] * 24 + [2] * 8), 1024) == 0.265625
    assert m.memory_ratio(cfg(8, 8, 64, 0, [8]), 10) == 1 / 8 + 8 / 16 + 2 / 64
    assert m.memory_ratio(cfg(4, 4, 16, 8, [4]), 20, include_residual=True) == pytest.approx(
        (16 * (1 / 4 + 4 / 16 + 2 / 16) + 4) / 20)
    assert m.memory_ratio(cfg(4, 4, 16, 64, [4]), 20, include_residual=True) == 1.0
    assert m.memory_ratio(cfg(4, 4, 16, 64, [4]), 0) == 0.0
    # the BASELINE C2 plan: accounted 0.375, actual bytes 67,584 per context token per sequence
    c2 = cfg(32, 8, 128, 128, [8] * 2 + [4] * 22 + [2] * 8)
    assert m.memory_ratio(c2, 32768) == pytest.approx(0.375)
    assert sum(2 * m.actual_bytes_per_token(128, 8, b) for b in c2.plan.bits_per_layer) == 67584


def test_deserialize_rejects_malformed_without_gpu():
    """FormatError is raised while parsing, before any device state exists (cache.py:333-368)."""
    import paper_2506_04642_b200 as m

    hdr = b"TADAKV1" + struct.pack("<IIBIQQ", 2, 4, 4, 0, 1, 0)
    with pytest.raises(m.FormatError):
        m.deserialize_cache(b"NOTMAGI" + hdr[7:])
    with pytest.raises(m.FormatError):
        m.deserialize_cache(b"TADAKV9" + hdr[7:])
    with pytest.raises(m.FormatError):
        m.deserialize_cache(hdr)  # truncated
    bad_bits = b"TADAKV1" + struct.pack("<IIBIQQ", 2, 4, 3, 0, 0, 0)
    with pytest.raises(m.FormatError):
        m.deserialize_cache(bad_bits)


def test_quantized_deviation_validation():
    import numpy as np

    import paper_2506_04642_b200 as m

    with pytest.raises(m.FormatError):
        m.QuantizedDeviation(4, 2, 2, 8, b"\0" * 15, np.zeros(4, np.float32), np.zeros(4, np.float32))
    with pytest.raises(m.FormatError):
        m.QuantizedDeviation(4, 2, 2, 8, b"\0" * 16, np.zeros(3, np.float32), np.zeros(4, np.float32))
    rec = m.empty_deviation(2, 4, 16)
    assert rec.num_groups == 0 and rec.shape == (0, 4, 16)
    assert m.bytes_per_group(16, 16) == 64 and m.bytes_per_group(7, 2) == 2


def test_product_path_has_no_cpu_fallback():
    """Without CUDA every compute entry point raises BackendUnavailable instead of computing on the CPU."""
    import numpy as np
    import torch

    import paper_2506_04642_b200 as m

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_lib.BackendUnavailable):
        m.quantize_tensor(np.zeros((1, 1, 4), np.float32), 4)
    with pytest.raises(_lib.BackendUnavailable):
        m.CompressedLayerCache(2, 16, 4, 0)


def test_ctypes_layout_struct_size():
    # int32 x6 + int64 x7 = 24 + 56 = 80 bytes, no padding surprises
    assert ctypes.sizeof(_lib.PageLayout) == 80
