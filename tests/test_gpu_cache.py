"""GPU parity of the compressed cache: K1 quantize-on-append into the paged layout.

Every cache is exported back to the reference layout and compared byte-for-byte
through TADAKV1 (serialize_cache) against the golden blobs the reference wrote,
or against the oracle.  Mirrors pkg/tests/test_cache.py (hot-path subset).
"""

import hashlib

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


def replay(key):
    c = CASES[key]
    k, v, q = gio.kv_inputs(c["seed"], c["schedule"], c["hq"], c["h"], c["d"])
    cache = tk().CompressedLayerCache(c["h"], c["d"], c["bits"], c["R"])
    for a, b in zip(gio.split_schedule(k, c["schedule"]), gio.split_schedule(v, c["schedule"])):
        cache.append_tokens(a, b)
    return cache, k, v, q


@pytest.mark.parametrize("key", gio.keys("kv"))
def test_append_schedule_blob_golden(key):
    cache, *_ = replay(key)
    blob = tk().serialize_cache(cache)
    assert len(blob) == CASES[key]["blob_len"]
    assert hashlib.sha256(blob).hexdigest() == CASES[key]["blob_sha256"]


@pytest.mark.parametrize("key", gio.keys("kv")[::3])
def test_deserialize_round_trip(key):
    cache, *_ = replay(key)
    blob = tk().serialize_cache(cache)
    restored = tk().deserialize_cache(blob)
    assert tk().serialize_cache(restored) == blob
    assert restored.total_tokens == cache.total_tokens


@pytest.mark.parametrize("key", gio.keys("c1"))
def test_config1_blob_golden(key):
    c = CASES[key]
    k, v, q = gio.c1_inputs(c["hq"])
    cache = tk().CompressedLayerCache(8, 128, 4, c["R"])
    cache.append_tokens(k, v)
    blob = tk().serialize_cache(cache)
    assert hashlib.sha256(blob).hexdigest() == c["blob_sha256"]
    # bf16 device input (production dtype) lands on the same bytes
    cache2 = tk().CompressedLayerCache(8, 128, 4, c["R"])
    cache2.append_tokens(torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16())
    assert tk().serialize_cache(cache2) == blob


def test_flush_trace_one_at_a_time():
    """test_cache.py:96-105."""
    cache = tk().CompressedLayerCache(2, 16, 4, 4)
    rng = np.random.default_rng(2)
    counts = []
    for _ in range(5):
        k = rng.normal(size=(1, 2, 16)).astype(np.float32)
        cache.append_tokens(k, k.copy())
        counts.append((cache.compressed_tokens, cache.r))
    assert counts == [(0, 1), (0, 2), (0, 3), (4, 0), (4, 1)]


@pytest.mark.parametrize("bits", [2, 4, 8, 16])
@pytest.mark.parametrize("R", [0, 3, 128])
def test_bulk_equals_incremental(bits, R):
    """test_cache.py:107-117, at decode granularity and the paper's R."""
    rng = np.random.default_rng(3 + bits)
    k = rng.normal(size=(300, 4, 32)).astype(np.float32)
    v = rng.normal(size=(300, 4, 32)).astype(np.float32)
    bulk = tk().CompressedLayerCache(4, 32, bits, R)
    bulk.append_tokens(k, v)
    step = tk().CompressedLayerCache(4, 32, bits, R)
    for t in range(0, 300, 7):
        step.append_tokens(k[t: t + 7], v[t: t + 7])
    ref = orc.LayerState(4, 32, bits, R)
    orc.append(ref, k, v)
    assert tk().serialize_cache(bulk) == tk().serialize_cache(step) == orc.dump(ref)


@pytest.mark.parametrize("bits", [2, 4, 8, 16])
def test_identical_heads_bit_exact(bits):
    """test_cache.py:159-173: identical heads reconstruct losslessly."""
    cache = tk().CompressedLayerCache(2, 16, bits, 3)
    rng = np.random.default_rng(6)
    k = np.repeat(rng.normal(size=(10, 1, 16)).astype(np.float32), 2, axis=1)
    v = np.repeat(rng.normal(size=(10, 1, 16)).astype(np.float32), 2, axis=1)
    cache.append_tokens(k, v)
    assert cache.compressed_tokens == 9
    for head in range(2):
        k_hat, v_hat = cache.reconstruct(head)
        assert np.array_equal(k_hat, k[:, head, :]) and np.array_equal(v_hat, v[:, head, :])


def test_outlier_regime_and_errors():
    m = tk()
    rng = np.random.default_rng(5)
    x = orc.outlier_activations(rng, 256, 8, 128)
    y = orc.outlier_activations(rng, 256, 8, 128)
    cache = m.CompressedLayerCache(8, 128, 2, 0)
    cache.append_tokens(x, y)
    ref = orc.LayerState(8, 128, 2, 0)
    orc.append(ref, x, y)
    assert m.serialize_cache(cache) == orc.dump(ref)
    with pytest.raises(m.ShapeError):
        cache.append_tokens(np.zeros((1, 3, 128), np.float32), np.zeros((1, 3, 128), np.float32))
    bad = x[:2].copy()
    bad[1, 3, 7] = np.nan
    before = m.serialize_cache(cache)
    with pytest.raises(m.DataError):
        cache.append_tokens(bad, bad)
    assert m.serialize_cache(cache) == before  # no mutation on error


@pytest.mark.parametrize("bits,R", [(4, 16), (2, 5), (8, 0)])
def test_nonfinite_flush_leaves_cache_unchanged(bits, R):
    """append_tokens with a non-finite row that K1 compresses raises DataError and restores the lengths and
    the residual rows the flush overwrote (no input pre-pass); the cache keeps working afterwards (oracle)."""
    m = tk()
    rng = np.random.default_rng(11 + bits)
    x = rng.standard_normal((3 * max(R, 1) + 3, 8, 128)).astype(np.float32)
    y = rng.standard_normal(x.shape).astype(np.float32)
    cache = m.CompressedLayerCache(8, 128, bits, R)
    ref = orc.LayerState(8, 128, bits, R)
    head = max(R - 2, 1)  # leaves a residual (R > 0) so the failing append's flush would overwrite it
    cache.append_tokens(x[:head], y[:head])
    orc.append(ref, x[:head], y[:head])
    before = m.serialize_cache(cache)
    for side in (0, 1):
        bad = [x[head:head + R + 4].copy(), y[head:head + R + 4].copy()]
        bad[side][1, 5, 9] = np.inf if side else np.nan
        with pytest.raises(m.DataError):
            cache.append_tokens(*bad)
        assert m.serialize_cache(cache) == before
        assert cache.total_tokens == head
    cache.append_tokens(x[head:], y[head:])
    orc.append(ref, x[head:], y[head:])
    assert m.serialize_cache(cache) == orc.dump(ref)


def test_nonfinite_residual_row_raises_at_its_flush():
    """Like the reference, a non-finite row that only enters the residual buffer is accepted; the append
    whose flush compresses it raises DataError and leaves the cache as it was before that append."""
    m = tk()
    rng = np.random.default_rng(3)
    x = rng.standard_normal((24, 8, 128)).astype(np.float32)
    x[2, 1, 3] = np.nan
    cache = m.CompressedLayerCache(8, 128, 4, 8)
    cache.append_tokens(x[:4], x[:4])  # 4 raw rows, one of them non-finite: no flush, no error
    assert cache.total_tokens == 4
    before = m.serialize_cache(cache)
    with pytest.raises(m.DataError):
        cache.append_tokens(x[4:12], x[4:12])  # flushes the first 8 rows
    assert m.serialize_cache(cache) == before


@pytest.mark.parametrize("plan", [(8, 4, 2, 16), (4, 4, 4, 4)])
def test_paged_multilayer_batched_vs_oracle(plan):
    """PagedKVCache: B sequences x L layers, shuffled pages, mixed widths; each (layer, seq) == oracle."""
    m = tk()
    B, H, D, R = 3, 8, 128, 16
    store = m.PagedKVCache(len(plan), H, D, plan, R, batch=B, page_tokens=16, max_tokens=200, shuffle_pages=True)
    rng = np.random.default_rng(11)
    chunks = [37, 1, 1, 60, 5]
    data = {}
    for layer in range(len(plan)):
        ks = orc.bf16_round(rng.normal(size=(B, sum(chunks), H, D)).astype(np.float32))
        vs = orc.bf16_round(rng.normal(size=(B, sum(chunks), H, D)).astype(np.float32))
        data[layer] = (ks, vs)
        off = 0
        for n in chunks:
            kt = torch.from_numpy(ks[:, off: off + n]).cuda().bfloat16()
            vt = torch.from_numpy(vs[:, off: off + n]).cuda().bfloat16()
            store.append(layer, kt, vt)
            off += n
    store.check_errors()
    for layer, bits in enumerate(plan):
        for b in range(B):
            ref = orc.LayerState(H, D, bits, R)
            orc.append(ref, data[layer][0][b], data[layer][1][b])
            ex = store.export(layer, b)
            kd = ex["k_dev"].to_host()
            assert kd.codes == ref.kdev.payload
            assert np.array_equal(ex["k_mean"].cpu().numpy(), ref.kmean)
            assert ex["v_dev"].to_host().codes == ref.vdev.payload
            assert np.array_equal(ex["residual_v"].cpu().numpy(), ref.rv)


def _k1_inputs(kind, B, T, H, D, rng):
    if kind == "normal":
        return orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))
    if kind == "ties":  # small integers: means on a 1/8 grid, many (x - min)/s exactly on .5
        return rng.integers(-8, 9, size=(B, T, H, D)).astype(np.float32)
    if kind == "outlier":  # shared outlier channels (analysis.py:37-57 regime)
        x = rng.normal(size=(B, T, H, D)).astype(np.float32) * 0.1
        x[..., :2] += 8.0 * rng.normal(size=(B, T, 1, 2)).astype(np.float32)
        return orc.bf16_round(x)
    if kind == "constant":  # zero-range groups -> scale 0, codes 0
        return orc.bf16_round(np.repeat(rng.normal(size=(B, T, H, 1)).astype(np.float32), D, axis=3))
    raise ValueError(kind)


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("kind", ["normal", "ties", "outlier", "constant"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_k1_fast_path_bit_exact(bits, kind, dtype):
    """K1 for head_dim 128 x 8 heads (the warp-per-token kernel): codes, scales, mins, means bit-exact."""
    m = tk()
    B, T, H, D = 2, 257, 8, 128
    rng = np.random.default_rng(hash((bits, kind)) % 2**32)
    k = _k1_inputs(kind, B, T, H, D, rng)
    v = _k1_inputs(kind, B, T, H, D, rng)
    store = m.PagedKVCache(1, H, D, (bits,), 0, batch=B, page_tokens=64, max_tokens=T, shuffle_pages=True)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    store.append(0, torch.from_numpy(k).cuda().to(tdt), torch.from_numpy(v).cuda().to(tdt))
    store.check_errors()
    for b in range(B):
        ref = orc.LayerState(H, D, bits, 0)
        orc.append(ref, k[b], v[b])
        ex = store.export(0, b)
        for side, rec, mean in (("k", ref.kdev, ref.kmean), ("v", ref.vdev, ref.vmean)):
            got = ex[f"{side}_dev"].to_host()
            assert got.codes == rec.payload
            assert np.array_equal(np.asarray(got.scales).view(np.uint32), rec.scales.view(np.uint32))
            assert np.array_equal(np.asarray(got.mins), rec.mins)
            assert np.array_equal(ex[f"{side}_mean"].cpu().numpy().view(np.uint32), mean.view(np.uint32))


def test_deserialize_untrusted_residual_header():
    """A TADAKV1 header with a huge residual_length must not allocate B*R*H*D floats up front, and a
    stream holding more raw rows than residual_length is accepted like the reference does; the next append
    flushes them exactly as the reference's append_tokens would (cache.py:171-180)."""
    import struct

    m = tk()
    rng = np.random.default_rng(3)
    H, D = 2, 16
    k = rng.normal(size=(9, H, D)).astype(np.float32)
    v = rng.normal(size=(9, H, D)).astype(np.float32)
    st = orc.LayerState(H, D, 4, 4)
    orc.append(st, k[:7], v[:7])  # C = 4, r = 3
    blob = orc.dump(st)
    hdr = len(orc.MAGIC)
    huge = blob[:hdr] + struct.pack("<IIBIQQ", H, D, 4, 0xFFFFFFFF, st.compressed, st.r) + blob[hdr + 29:]
    cache = m.deserialize_cache(huge)  # no 2^32-row residual allocation
    assert cache.total_tokens == 7 and m.serialize_cache(cache) == huge
    # r = 3 raw rows with residual_length 2: the reference keeps them; its next append flushes 4
    small = blob[:hdr] + struct.pack("<IIBIQQ", H, D, 4, 2, st.compressed, st.r) + blob[hdr + 29:]
    cache = m.deserialize_cache(small)
    ref = orc.load(small)
    cache.append_tokens(k[7:], v[7:])
    orc.append(ref, k[7:], v[7:])
    assert m.serialize_cache(cache) == orc.dump(ref)


@pytest.mark.parametrize("H,D", [(4, 256), (1, 64), (16, 128), (2, 32), (3, 96), (32, 128)])
@pytest.mark.parametrize("bits", [2, 4, 8, 16])
def test_append_other_geometries_bit_exact(H, D, bits):
    """K1 (the generic quant_append_kernel off H=8/D=128; the fast kernel there) at other head counts and head
    dims, bf16 and f32 inputs, with a residual flush: the TADAKV1 bytes equal the oracle's; decode attention
    (mode 0) is within 1e-5 of the oracle where it runs exact and 2e-3 on the tensor-core views."""
    import torch

    m = tk()
    rng = np.random.default_rng(1200 + H + D + bits)
    T, R, hq = 150, 16, 2 * H
    k = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    for dtype in (torch.bfloat16, torch.float32):
        cache = m.CompressedLayerCache(H, D, bits, R)
        cache.append_tokens(torch.from_numpy(k[:70]).cuda().to(dtype), torch.from_numpy(v[:70]).cuda().to(dtype))
        cache.append_tokens(torch.from_numpy(k[70:]).cuda().to(dtype), torch.from_numpy(v[70:]).cuda().to(dtype))
        st = orc.LayerState(H, D, bits, R)
        orc.append(st, k, v)
        assert m.serialize_cache(cache) == orc.dump(st), dtype
    q = orc.bf16_round(rng.normal(size=(hq, D)).astype(np.float32))
    want = orc.attend(q, st, hq)[0]
    out = cache.store.attend(0, torch.from_numpy(q).cuda().unsqueeze(0), out_dtype=torch.float32)[0].cpu().numpy()
    assert np.abs(out - want).max() <= 2e-3
    exact = m.attend_streaming(q, cache, m.ModelConfig(1, hq, H, D, R, m.RopeParams(D), m.PrecisionPlan((bits,)))).output
    assert np.abs(exact - want).max() <= 1e-5
