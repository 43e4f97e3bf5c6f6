"""GPU parity: quantizer / packer / mean-centering kernels vs reference golden vectors and the oracle.

Bar: codes bit-exact, scales bitwise, mins == (+0 == -0), dequantized values bitwise.
Mirrors pkg/tests/test_quant.py (hot-path subset) plus golden replays.
"""

import numpy as np
import pytest
import torch

import golden_io as gio
from oracle import tada_oracle as orc

pytestmark = pytest.mark.gpu

ARR, CASES = gio.load()


def tk():
    import paper_2506_04642_b200 as m

    return m


def bits_eq(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("key", gio.keys("q"))
def test_quantize_tensor_golden(key):
    dev = ARR[f"{key}/input"]
    q = tk().quantize_tensor(dev, CASES[key]["bits"])
    assert q.codes == ARR[f"{key}/codes"].tobytes()
    assert bits_eq(q.scales, ARR[f"{key}/scales"])
    assert np.array_equal(q.mins, ARR[f"{key}/mins"])
    assert bits_eq(tk().dequantize_tensor(q), ARR[f"{key}/deq"])


@pytest.mark.parametrize("key", gio.keys("q")[::5])
def test_quantize_tensor_device_inputs(key):
    """torch CUDA f32 input stays on device and gives the same bytes."""
    dev = torch.from_numpy(ARR[f"{key}/input"]).cuda()
    q = tk().quantize_tensor(dev, CASES[key]["bits"])
    assert q.on_device
    assert q.to_host().codes == ARR[f"{key}/codes"].tobytes()
    assert bits_eq(tk().dequantize_tensor(q).cpu().numpy(), ARR[f"{key}/deq"])


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_bf16_input_equals_f32_input(bits):
    rng = np.random.default_rng(bits)
    x = orc.bf16_round(rng.normal(size=(64, 8, 128)).astype(np.float32))
    a = tk().quantize_tensor(torch.from_numpy(x).cuda().to(torch.bfloat16), bits).to_host()
    b = orc.quantize(x, bits)
    assert a.codes == b.payload and bits_eq(a.scales, b.scales)


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("d", [16, 64, 128, 256])
def test_random_large_vs_oracle(bits, d):
    """Adversarial mixes: .5-tie grids, wide scale mix, outliers — 20k groups per case."""
    rng = np.random.default_rng(100 * bits + d)
    g = 20_000
    mix = rng.choice([1e-3, 1.0, 37.0, 1e4], size=(g, 1, 1))
    x = (rng.normal(size=(g, 1, d)) * mix).astype(np.float32)
    x[: g // 4] = np.round(x[: g // 4] * 8) / 8  # grid values -> many exact ties
    x = x.reshape(g // 4, 4, d)
    a = tk().quantize_tensor(x, bits)
    b = orc.quantize(x, bits)
    assert a.codes == b.payload
    assert bits_eq(a.scales, b.scales)
    assert np.array_equal(a.mins, b.mins)


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("group_size", [1, 3, 4, 5, 7, 16, 33])
def test_pack_unpack_bijective(bits, group_size):
    """test_quant.py:152-160 on the GPU kernels, checked against the oracle packer."""
    rng = np.random.default_rng(bits * 100 + group_size)
    codes = rng.integers(0, 2**bits, size=(25, group_size))
    packed = tk().pack_codes(codes, bits)
    assert packed == orc.pack(codes, bits)
    assert np.array_equal(tk().unpack_codes(packed, bits, 25, group_size), codes)
    sel = np.array([0, 7, 24, 3])
    assert np.array_equal(tk().unpack_codes(packed, bits, 25, group_size, groups=sel), codes[sel])


def test_quantize_group_known_answers():
    """test_quant.py:21-46."""
    codes, scale, vmin = tk().quantize_group(np.array([-1.0, 0.0, 1.0, 2.0], dtype=np.float32), 2)
    assert (vmin, scale, codes.tolist()) == (-1.0, 1.0, [0, 1, 2, 3])
    codes, scale, vmin = tk().quantize_group(np.arange(16, dtype=np.float32), 4)
    assert (vmin, scale, codes.tolist()) == (0.0, 1.0, list(range(16)))
    for bits in (2, 4, 8):
        codes, scale, vmin = tk().quantize_group(np.full(8, -3.5, dtype=np.float32), bits)
        assert scale == 0.0 and vmin == -3.5 and (codes == 0).all()


def test_errors():
    m = tk()
    with pytest.raises(m.DataError):
        m.quantize_group(np.array([1.0, np.nan], dtype=np.float32), 4)
    with pytest.raises(m.DataError):
        m.quantize_tensor(np.array([[[1.0, np.inf]]], dtype=np.float32), 16)
    with pytest.raises(m.ConfigError):
        m.quantize_group(np.ones(4, dtype=np.float32), 16)
    with pytest.raises(m.ConfigError):
        m.quantize_tensor(np.ones((1, 1, 4), dtype=np.float32), 3)
    with pytest.raises(m.ShapeError):
        m.quantize_tensor(np.zeros((3, 4), dtype=np.float32), 4)
    with pytest.raises(m.FormatError):
        m.unpack_codes(b"\x00\x00\x00", 2, 4, 16)
    with pytest.raises(m.ConfigError):
        m.pack_codes(np.zeros((1, 4), dtype=np.uint8), 16)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_round_trip_idempotent(bits):
    """test_quant.py:104-110: a second quantize/dequantize pass reproduces the first bit-exactly."""
    rng = np.random.default_rng(17)
    dev = rng.normal(size=(600, 2, 16)).astype(np.float32)
    first = tk().dequantize_tensor(tk().quantize_tensor(dev, bits))
    second = tk().dequantize_tensor(tk().quantize_tensor(first, bits))
    assert bits_eq(first, second)


def test_concat_and_group_selection():
    m = tk()
    rng = np.random.default_rng(41)
    a = rng.normal(size=(3, 2, 8)).astype(np.float32)
    b = rng.normal(size=(5, 2, 8)).astype(np.float32)
    joint = m.quantize_tensor(np.concatenate([a, b]), 4)
    split = m.concat_deviations(m.quantize_tensor(a, 4), m.quantize_tensor(b, 4))
    assert joint.codes == split.codes and bits_eq(joint.scales, split.scales)
    full = m.dequantize_tensor(joint).reshape(16, 8)
    picks = np.array([0, 5, 11, 15])
    assert bits_eq(m.dequantize_groups(joint, picks), full[picks])


@pytest.mark.parametrize("key", gio.keys("mc"))
def test_mean_center_golden(key):
    mean, dev = tk().mean_center(ARR[f"{key}/input"])
    assert bits_eq(mean, ARR[f"{key}/mean"])
    assert bits_eq(dev, ARR[f"{key}/dev"])


def test_mean_center_order_sensitive():
    """Sequential head-order fp64 sum (numpy reduces the head axis in order)."""
    x = np.zeros((2, 8, 8), dtype=np.float32)
    x[:, 0:4, 3] = np.array([1, 2**60, -(2**60), 1], dtype=np.float32)
    mean, _ = tk().mean_center(x)
    want, _ = orc.center(x)
    assert bits_eq(mean, want) and mean[0, 3] == 0.125
