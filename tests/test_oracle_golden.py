"""Pin the CPU oracle (oracle/tada_oracle.py) to golden vectors produced by the reference.

CPU-only: these run in the build container and on the GPU box alike.
"""

import hashlib

import numpy as np
import pytest

import golden_io as gio
from oracle import tada_oracle as orc

ARR, CASES = gio.load()


def bits_eq(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("key", gio.keys("q"))
def test_quantizer_matches_reference(key):
    dev = ARR[f"{key}/input"]
    bits = CASES[key]["bits"]
    rec = orc.quantize(dev, bits)
    assert rec.payload == ARR[f"{key}/codes"].tobytes()
    assert bits_eq(rec.scales, ARR[f"{key}/scales"])
    assert np.array_equal(rec.mins, ARR[f"{key}/mins"])  # +0 == -0 (SURVEY §8a signed-zero note)
    assert bits_eq(orc.dequantize(rec), ARR[f"{key}/deq"])


@pytest.mark.parametrize("key", gio.keys("mc"))
def test_mean_center_matches_reference(key):
    mean, dev = orc.center(ARR[f"{key}/input"])
    assert bits_eq(mean, ARR[f"{key}/mean"])
    assert bits_eq(dev, ARR[f"{key}/dev"])


def _oracle_cache(key):
    c = CASES[key]
    k, v, q = gio.kv_inputs(c["seed"], c["schedule"], c["hq"], c["h"], c["d"])
    assert gio.sha(k, v, q) == c["input_sha256"]
    st = orc.LayerState(c["h"], c["d"], c["bits"], c["R"])
    for a, b in zip(gio.split_schedule(k, c["schedule"]), gio.split_schedule(v, c["schedule"])):
        orc.append(st, a, b)
    return st, q


@pytest.mark.parametrize("key", gio.keys("kv"))
def test_cache_blob_matches_reference(key):
    st, _ = _oracle_cache(key)
    blob = orc.dump(st)
    assert len(blob) == CASES[key]["blob_len"]
    assert hashlib.sha256(blob).hexdigest() == CASES[key]["blob_sha256"]
    if f"{key}/blob" in ARR:
        assert blob == ARR[f"{key}/blob"].tobytes()
    assert orc.dump(orc.load(blob)) == blob


@pytest.mark.parametrize("key", [k for k in gio.keys("kv") if sum(CASES[k]["schedule"]) > 0])
def test_attention_matches_reference(key):
    st, q = _oracle_cache(key)
    hq = CASES[key]["hq"]
    out64, _ = orc.attend(q, st, hq, block=64)
    out3, _ = orc.attend(q, st, hq, block=3)
    # BLAS accumulation order is unspecified, so attention is tolerance-pinned
    assert np.abs(out64 - ARR[f"{key}/attn_stream64"]).max() <= 1e-5
    assert np.abs(out3 - ARR[f"{key}/attn_stream3"]).max() <= 1e-5
    assert np.abs(orc.attend_full(q, st, hq) - ARR[f"{key}/attn_naive"]).max() <= 1e-5


@pytest.mark.parametrize("key", gio.keys("c1"))
def test_config1_matches_reference(key):
    c = CASES[key]
    k, v, q = gio.c1_inputs(c["hq"])
    assert gio.sha(k, v, q) == c["input_sha256"]
    st = orc.LayerState(8, 128, 4, c["R"])
    orc.append(st, k, v)
    blob = orc.dump(st)
    assert hashlib.sha256(blob).hexdigest() == c["blob_sha256"]
    out, _ = orc.attend(q, st, c["hq"])
    assert np.abs(out - ARR[f"{key}/attn_stream64"]).max() <= 1e-5


def test_tadakv1_rejects_corruption():
    st, _ = _oracle_cache("kv00")
    blob = orc.dump(st)
    for cut in range(0, len(blob), 41):
        with pytest.raises(orc.OracleError):
            orc.load(blob[:cut])
    with pytest.raises(orc.OracleError):
        orc.load(blob + b"\0")
    with pytest.raises(orc.OracleError):
        orc.load(b"TADAKV9" + blob[7:])


def test_accounted_ratio_known_answers():
    # cache.py:216-239; test_cache.py:211-251
    assert orc.accounted_ratio([4], 32, 128, 1024, 0) == 0.296875
    assert orc.accounted_ratio([4] * 24 + [2] * 8, 32, 128, 1024, 0) == 0.265625
    assert orc.accounted_ratio([8], 8, 64, 10, 0) == 1 / 8 + 8 / 16 + 2 / 64
    assert orc.accounted_ratio([4], 4, 64 // 4, 20, 64, include_residual=True) == 1.0
