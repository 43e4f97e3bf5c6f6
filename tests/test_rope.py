"""RoPE + compress row: apply_rope / rotate_heads / append_fused.

CPU: the oracle restatement (oracle/tada_oracle.py rope, rope_heads) against the reference's own outputs
(tests/golden/rope.npz, made by tests/golden/make_golden_rope.py from tadakv itself).
GPU: tada_apply_rope and K1's fused RoPE variant against the same fixtures, bit for bit; the fused
append against the composition rotate_heads + append_tokens (AC8, test_acceptance.py:272-305).
"""

import hashlib

import numpy as np
import pytest
import torch

from golden_io import load_rope, rope_af_inputs
from oracle import tada_oracle as orc


def _cases(prefix):
    _, cases = load_rope()
    return sorted(k for k in cases if k.startswith(prefix))


def _bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


# ---------------------------------------------------------------------- CPU: oracle pinned to the reference
@pytest.mark.parametrize("key", _cases("ar"))
def test_oracle_apply_rope_golden(key):
    arr, cases = load_rope()
    m = cases[key]
    assert _bits_equal(orc.rope(arr[f"{key}/x"], arr[f"{key}/pos"], m["head_dim"], m["base"]), arr[f"{key}/y"])


@pytest.mark.parametrize("key", _cases("rh"))
def test_oracle_rotate_heads_golden(key):
    arr, cases = load_rope()
    d = cases[key]["shape"][2]
    assert _bits_equal(orc.rope_heads(arr[f"{key}/x"], arr[f"{key}/pos"], d), arr[f"{key}/y"])


@pytest.mark.parametrize("key", _cases("af"))
def test_oracle_append_rope_golden(key):
    _, cases = load_rope()
    m = cases[key]
    st = orc.LayerState(8, 128, m["bits"], m["R"])
    for k_pre, v, pos in rope_af_inputs(int(key[2:]), m["bits"], m["R"]):
        orc.append(st, orc.rope_heads(k_pre, pos, 128), v)
    assert hashlib.sha256(orc.dump(st)).hexdigest() == m["sha256"]


def test_oracle_rope_table_matches_rows():
    tab = orc.rope_table(128, 10000.0, 300)
    x = np.random.default_rng(0).normal(size=(300, 128)).astype(np.float32)
    pos = np.arange(300)
    y = orc.rope(x, pos, 128)
    c, s = tab[..., 0], tab[..., 1]
    e, o = x[:, 0::2], x[:, 1::2]
    assert _bits_equal(y[:, 0::2], e * c - o * s) and _bits_equal(y[:, 1::2], e * s + o * c)


# ---------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("key", _cases("ar"))
def test_gpu_apply_rope_golden(key):
    import paper_2506_04642_b200 as tk

    arr, cases = load_rope()
    m = cases[key]
    got = tk.apply_rope(arr[f"{key}/x"], arr[f"{key}/pos"], tk.RopeParams(m["head_dim"], m["base"]))
    assert _bits_equal(got, arr[f"{key}/y"])


@pytest.mark.gpu
@pytest.mark.parametrize("key", _cases("rh"))
def test_gpu_rotate_heads_golden(key):
    import paper_2506_04642_b200 as tk

    arr, cases = load_rope()
    d = cases[key]["shape"][2]
    x = arr[f"{key}/x"]
    got = tk.rotate_heads(x, arr[f"{key}/pos"], tk.RopeParams(d))
    assert _bits_equal(got, arr[f"{key}/y"])
    # bf16 device input (the grid is bf16-exact) gives the same bits
    xt = torch.from_numpy(x).cuda().bfloat16()
    got_t = tk.rotate_heads(xt, torch.from_numpy(arr[f"{key}/pos"]), tk.RopeParams(d))
    assert _bits_equal(got_t.cpu().numpy(), arr[f"{key}/y"])


@pytest.mark.gpu
@pytest.mark.parametrize("key", _cases("af"))
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_gpu_append_rope_golden(key, dtype):
    """Fused K1 RoPE path: the TADAKV1 bytes equal the reference's rotate_heads + append_tokens."""
    import paper_2506_04642_b200 as tk

    _, cases = load_rope()
    m = cases[key]
    cache = tk.CompressedLayerCache(8, 128, m["bits"], m["R"])
    for k_pre, v, pos in rope_af_inputs(int(key[2:]), m["bits"], m["R"]):
        k_in, v_in = torch.from_numpy(k_pre).cuda(), torch.from_numpy(v).cuda()
        if dtype == "bf16":
            k_in, v_in = k_in.bfloat16(), v_in.bfloat16()
        tk.append_rope(cache, k_in, v_in, pos, tk.RopeParams(128))
    assert hashlib.sha256(tk.serialize_cache(cache)).hexdigest() == m["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("R", [0, 128])
def test_gpu_append_fused_equals_composition(bits, R):
    """AC8: append_fused == rotate_heads + the same projection + append_tokens, byte for byte."""
    import paper_2506_04642_b200 as tk

    rng = np.random.default_rng(90 + bits + R)
    rope = tk.RopeParams(128, 500000.0)
    fused, composed = tk.CompressedLayerCache(8, 128, bits, R), tk.CompressedLayerCache(8, 128, bits, R)
    start = 0
    for cnt in (200, 1, 1, 70):
        k_pre = orc.bf16_round(rng.normal(size=(cnt, 8, 128)).astype(np.float32))
        x_norm = rng.normal(size=(cnt, 64)).astype(np.float32)
        w_v = (rng.normal(size=(64, 1024)) * 0.1).astype(np.float32)
        pos = np.arange(start, start + cnt) + 1000
        if start % 2:  # device operands: the projection is a cuBLAS GEMM on both sides
            xd, wd = torch.from_numpy(x_norm).cuda(), torch.from_numpy(w_v).cuda()
            tk.append_fused(fused, k_pre, xd, wd, pos, rope)
            v = (xd @ wd).reshape(cnt, 8, 128)
        else:  # host operands: numpy's f32 matmul on both sides, exactly the reference's AC8 composition
            tk.append_fused(fused, k_pre, x_norm, w_v, pos, rope)
            v = (x_norm @ w_v).reshape(cnt, 8, 128)
        composed.append_tokens(tk.rotate_heads(k_pre, pos, rope), v)
        start += cnt
    assert tk.serialize_cache(fused) == tk.serialize_cache(composed)
    # the device projection agrees with numpy's to f32 rounding (different summation order)
    v_dev = (torch.from_numpy(x_norm).cuda() @ torch.from_numpy(w_v).cuda()).cpu().numpy()
    assert np.abs(v_dev - x_norm @ w_v).max() < 1e-4


@pytest.mark.gpu
def test_gpu_batched_append_rope_matches_per_sequence():
    """PagedKVCache.append_rope (batch 3, per-sequence positions) == three single-sequence caches."""
    import paper_2506_04642_b200 as tk
    from paper_2506_04642_b200.rope import _positions

    rng = np.random.default_rng(5)
    B, n, rope = 3, 150, tk.RopeParams(128)
    k = orc.bf16_round(rng.normal(size=(B, n, 8, 128)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(B, n, 8, 128)).astype(np.float32))
    pos = np.stack([np.arange(n) + 17 * b for b in range(B)])
    store = tk.PagedKVCache(1, 8, 128, [4], 128, batch=B)
    pd, top = _positions(pos, n, B)
    store.append_rope(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), pd, top, rope)
    for b in range(B):
        one = tk.CompressedLayerCache(8, 128, 4, 128)
        tk.append_rope(one, k[b], v[b], pos[b], rope)
        got = store.export(0, b)
        ref = one.store.export(0, 0)
        for name in ("k_mean", "v_mean", "residual_k", "residual_v"):
            assert torch.equal(got[name], ref[name]), name
        for name in ("k_dev", "v_dev"):
            assert torch.equal(got[name].device_tensors()[0], ref[name].device_tensors()[0]), name


@pytest.mark.gpu
def test_gpu_rope_errors_raise_before_mutation():
    import paper_2506_04642_b200 as tk

    cache = tk.CompressedLayerCache(8, 128, 4, 0)
    k = np.zeros((4, 8, 128), np.float32)
    with pytest.raises(tk.DataError):
        tk.append_rope(cache, k, k, [0, 1, -2, 3], tk.RopeParams(128))
    with pytest.raises(tk.DataError):
        tk.apply_rope(k[:, 0], np.array([0.5, 1, 2, 3]), tk.RopeParams(128))
    with pytest.raises(tk.ShapeError):
        tk.rotate_heads(k, [0, 1, 2], tk.RopeParams(128))
    with pytest.raises(tk.ShapeError):
        tk.apply_rope(k[:, 0, :64], [0, 1, 2, 3], tk.RopeParams(128))
    bad = k.copy()
    bad[1, 2, 3] = np.nan
    with pytest.raises(tk.DataError):
        tk.append_rope(cache, bad, k, [0, 1, 2, 3], tk.RopeParams(128))
    assert cache.total_tokens == 0
