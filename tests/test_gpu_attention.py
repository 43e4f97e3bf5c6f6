"""GPU parity of decode attention (K2 split-K + K3 combine) vs the reference.

Bars: exact kernels (f32 out) within 1e-5 of the reference's attend_streaming
(the reference's own streaming-vs-naive tolerance, test_acceptance.py:150-178);
the tensor-core kernels within the north_star's 2e-3 max-abs on randn-scale
activations, and within 2e-3 * max(1, |out|max) — a RELATIVE bar — in the outlier
regimes whose outputs exceed 1 (the f16 vmean; bf16 itself carries a
2e-3 half-ulp at |out| = 1).  Mirrors pkg/tests/test_attention.py (hot-path subset).
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


def cfg_for(hq, h, d, R, bits):
    m = tk()
    return m.ModelConfig(1, hq, h, d, R, m.RopeParams(d), m.PrecisionPlan((bits,)))


def replay(key):
    c = CASES[key]
    k, v, q = gio.kv_inputs(c["seed"], c["schedule"], c["hq"], c["h"], c["d"])
    cache = tk().CompressedLayerCache(c["h"], c["d"], c["bits"], c["R"])
    for a, b in zip(gio.split_schedule(k, c["schedule"]), gio.split_schedule(v, c["schedule"])):
        cache.append_tokens(a, b)
    return cache, q, cfg_for(c["hq"], c["h"], c["d"], c["R"], c["bits"])


@pytest.mark.parametrize("key", [k for k in gio.keys("kv") if sum(CASES[k]["schedule"]) > 0])
def test_attend_streaming_golden(key):
    cache, q, cfg = replay(key)
    out = tk().attend_streaming(q, cache, cfg).output
    assert np.abs(out - ARR[f"{key}/attn_stream64"]).max() <= 1e-5
    naive = tk().attend_naive(q, cache, cfg).output
    assert np.abs(naive - ARR[f"{key}/attn_naive"]).max() <= 1e-5


@pytest.mark.parametrize("key", gio.keys("c1"))
def test_config1_attention_golden(key):
    c = CASES[key]
    k, v, q = gio.c1_inputs(c["hq"])
    cache = tk().CompressedLayerCache(8, 128, 4, c["R"])
    cache.append_tokens(k, v)
    out = tk().attend_streaming(q, cache, cfg_for(c["hq"], 8, 128, c["R"], 4)).output
    assert np.abs(out - ARR[f"{key}/attn_stream64"]).max() <= 1e-5


def test_single_token_returns_value_and_empty_cache():
    m = tk()
    cfg = cfg_for(4, 2, 16, 4, 4)
    rng = np.random.default_rng(0)
    cache = m.CompressedLayerCache(2, 16, 4, 4)
    with pytest.raises(m.StateError):
        m.attend_streaming(np.zeros((4, 16), np.float32), cache, cfg)
    k = rng.normal(size=(1, 2, 16)).astype(np.float32)
    v = rng.normal(size=(1, 2, 16)).astype(np.float32)
    cache.append_tokens(k, v)
    out = m.attend_streaming(rng.normal(size=(4, 16)).astype(np.float32), cache, cfg).output
    for g in range(4):
        assert np.allclose(out[g], v[0, m.kv_head_index(g, 4, 2)], atol=1e-6)
    with pytest.raises(m.ShapeError):
        m.attend_streaming(np.zeros((3, 16), np.float32), cache, cfg)


def test_scores_normalized():
    m = tk()
    cfg = cfg_for(4, 2, 16, 4, 4)
    rng = np.random.default_rng(4)
    cache = m.CompressedLayerCache(2, 16, 4, 4)
    cache.append_tokens(rng.normal(size=(7, 2, 16)).astype(np.float32), rng.normal(size=(7, 2, 16)).astype(np.float32))
    out = m.attend_naive(rng.normal(size=(4, 16)).astype(np.float32), cache, cfg, return_scores=True)
    assert len(out.scores) == 4
    for row in out.scores:
        assert row.shape == (7,) and abs(float(row.sum()) - 1.0) < 1e-5


def _paged_case(B, H, hq, D, bits, T, R, seed, page_tokens=64, poison=False):
    m = tk()
    rng = np.random.default_rng(seed)
    k = orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))
    q = orc.bf16_round(rng.normal(size=(B, hq, D)).astype(np.float32))
    store = m.PagedKVCache(1, H, D, (bits,), R, batch=B, page_tokens=page_tokens, max_tokens=T + 1,
                           shuffle_pages=True, seed=seed)
    if poison:  # NaN bytes everywhere the append does not write (rows past the end of each sequence)
        for pool in store.pools:
            pool.fill_(0xFF)
    store.append(0, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16())
    want = []
    for b in range(B):
        st = orc.LayerState(H, D, bits, R)
        orc.append(st, k[b], v[b])
        want.append(orc.attend(q[b], st, hq)[0])
    return store, torch.from_numpy(q).cuda(), np.stack(want)


@pytest.mark.parametrize("bits", [2, 4, 8, 16])
@pytest.mark.parametrize("splits", [1, 3, 16])
def test_paged_batched_exact(bits, splits):
    store, q, want = _paged_case(B=3, H=8, hq=32, D=128, bits=bits, T=700, R=128, seed=bits)
    out = store.attend(0, q, num_splits=splits, mode=1)
    assert np.abs(out.cpu().numpy() - want).max() <= 1e-5


def _fast_or_skip(store, q, **kw):
    m = tk()
    try:
        return store.attend(0, q, mode=2, **kw)
    except m.ConfigError as e:  # geometry without a tensor-core instantiation (e.g. 8-bit x 64 q heads)
        pytest.skip(str(e))


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("hq", [8, 16, 24, 32, 40, 48, 56, 64])
def test_paged_batched_fast_bf16(bits, hq):
    """Every group size 1..8 on the tensor-core path: G in {3, 5, 6, 7} run zero-padded to the next
    instantiated group, 8-bit G > 4 in two passes (tada_attn.cu fast_map)."""
    store, q, want = _paged_case(B=4, H=8, hq=hq, D=128, bits=bits, T=1500, R=128, seed=10 + bits)
    out = _fast_or_skip(store, q.bfloat16(), out_dtype=torch.bfloat16)
    assert np.abs(out.float().cpu().numpy() - want).max() <= 2e-3
    out32 = _fast_or_skip(store, q, out_dtype=torch.float32)
    assert np.abs(out32.cpu().numpy() - want).max() <= 2e-3


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("T,splits", [(1000, 1), (1000, 7), (45, 1), (2080, 0), (17, 3)])
def test_fast_tails_and_splits(bits, T, splits):
    """Tail tiles (tokens past the sequence end inside a page), empty splits, single-tile caches."""
    store, q, want = _paged_case(B=2, H=8, hq=32, D=128, bits=bits, T=T, R=0, seed=100 + T + bits, poison=True)
    out = _fast_or_skip(store, q, out_dtype=torch.float32, num_splits=splits or None)
    assert np.abs(out.cpu().numpy() - want).max() <= 2e-3


def test_precision_ordering():
    """test_attention.py:158-176: median error vs the raw-K/V f64 oracle shrinks with width."""
    m = tk()
    errs = {b: [] for b in (2, 4, 8, 16)}
    for seed in range(20):
        rng = np.random.default_rng(seed)
        k = rng.normal(size=(12, 2, 16)).astype(np.float32)
        v = rng.normal(size=(12, 2, 16)).astype(np.float32)
        q = rng.normal(size=(4, 16)).astype(np.float32)
        exact = orc.attend_f64(q, k, v, 4)
        for b in errs:
            cache = m.CompressedLayerCache(2, 16, b, 0)
            cache.append_tokens(k, v)
            errs[b].append(float(np.linalg.norm(m.attend_naive(q, cache, cfg_for(4, 2, 16, 0, b)).output - exact)))
    med = [float(np.median(errs[b])) for b in (2, 4, 8, 16)]
    assert med[0] >= med[1] >= med[2] >= med[3]


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("hq", [32, 64])
@pytest.mark.parametrize("regime", ["shared", "head"])
def test_fast_outlier_regimes(bits, hq, regime):
    """Large means (analysis.py:37-57 shared outlier channels, x8) and head-specific outliers (one head's
    channel x40, so the mean and the deviations are both large): the f16 hi + lo mean terms and the
    16-bit fixed-point q keep the tensor-core kernels within 2e-3 of the reference (scaled by |out|max)."""
    m = tk()
    rng = np.random.default_rng(300 + bits + hq)
    B, T, H, D = 2, 900, 8, 128
    k = np.stack([orc.outlier_activations(rng, T, H, D) for _ in range(B)])
    v = np.stack([orc.outlier_activations(rng, T, H, D) for _ in range(B)])
    if regime == "head":
        k[:, :, 3, 17] *= 40.0
        v[:, :, 5, 90] *= 40.0
    k, v = orc.bf16_round(k.astype(np.float32)), orc.bf16_round(v.astype(np.float32))
    q = orc.bf16_round((rng.normal(size=(B, hq, D)) * 2.0).astype(np.float32))
    store = m.PagedKVCache(1, H, D, (bits,), 128, batch=B, page_tokens=64, max_tokens=T + 1, shuffle_pages=True)
    store.append(0, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16())
    want = []
    for b in range(B):
        st = orc.LayerState(H, D, bits, 128)
        orc.append(st, k[b], v[b])
        want.append(orc.attend(q[b], st, hq)[0])
    want = np.stack(want)
    out = _fast_or_skip(store, torch.from_numpy(q).cuda(), out_dtype=torch.float32)
    assert np.abs(out.cpu().numpy() - want).max() <= 2e-3 * max(1.0, float(np.abs(want).max()))


@pytest.mark.parametrize("bits,hq", [(4, 32), (2, 64), (8, 32), (4, 8)])
def test_append_attend_fused_equals_append_then_attend(bits, hq):
    """PagedKVCache.append_attend (K3 attends and stores the step's row) == append() + attend(), output bits
    and cache state, across decode steps that cross the residual flush (R = 8)."""
    m = tk()
    B, T, H, D, R = 3, 300, 8, 128, 8
    rng = np.random.default_rng(70 + bits + hq)
    k0 = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))).cuda().bfloat16()
    v0 = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))).cuda().bfloat16()
    a = m.PagedKVCache(1, H, D, (bits,), R, batch=B, page_tokens=64, max_tokens=T + 64)
    b = m.PagedKVCache(1, H, D, (bits,), R, batch=B, page_tokens=64, max_tokens=T + 64)
    a.append(0, k0, v0)
    b.append(0, k0, v0)
    for step in range(20):
        k = torch.from_numpy(rng.normal(size=(B, 1, H, D)).astype(np.float32)).cuda().bfloat16()
        v = torch.from_numpy(rng.normal(size=(B, 1, H, D)).astype(np.float32)).cuda().bfloat16()
        q = torch.from_numpy(rng.normal(size=(B, hq, D)).astype(np.float32)).cuda().bfloat16()
        want = (a.append(0, k, v), a.attend(0, q, out_dtype=torch.bfloat16, num_splits=5))[1]
        got = b.append_attend(0, q, k, v, out_dtype=torch.bfloat16, num_splits=5)
        assert torch.equal(got, want), step
        assert a.lengths(0, 0) == b.lengths(0, 0)
    r = a.lengths(0)[1]
    assert torch.equal(a.res_k[0][:, :r], b.res_k[0][:, :r]) and torch.equal(a.res_v[0][:, :r], b.res_v[0][:, :r])
    assert torch.equal(a.res_len[0], b.res_len[0]) and torch.equal(a.comp_len[0], b.comp_len[0])


@pytest.mark.parametrize("hq,mode", [(24, 1), (24, 2), (40, 1)])
def test_combine_other_group_sizes(hq, mode):
    """G = Hq/H outside {1, 2, 4, 8} (K3 combine_pair_kernel), with residual rows: exact path within the
    reference's 1e-5, tensor-core path (if the geometry has one) within 2e-3."""
    store, q, want = _paged_case(B=2, H=8, hq=hq, D=128, bits=4, T=700, R=128, seed=hq + mode)
    if mode == 1:
        out = store.attend(0, q, num_splits=5, mode=1)
        assert np.abs(out.cpu().numpy() - want).max() <= 1e-5
    else:
        out = _fast_or_skip(store, q, out_dtype=torch.float32)
        assert np.abs(out.cpu().numpy() - want).max() <= 2e-3


@pytest.mark.parametrize("R,T", [(200, 900), (200, 1000), (160, 159), (300, 1499)])
def test_long_residual_chunks(R, T):
    """residual_length > 128: K3 stages the residual rows through shared memory in chunks of 128
    (T % R rows stay raw: 100, 0 + 200 flush..., 159, 299)."""
    store, q, want = _paged_case(B=2, H=8, hq=32, D=128, bits=4, T=T, R=R, seed=R + T)
    out = store.attend(0, q, num_splits=4, mode=1)
    assert np.abs(out.cpu().numpy() - want).max() <= 1e-5
    out = _fast_or_skip(store, q, out_dtype=torch.float32)
    assert np.abs(out.cpu().numpy() - want).max() <= 2e-3


@pytest.mark.parametrize("hq", [8, 32, 64])
def test_fused_step_long_residual(hq):
    """Fused decode steps (K3 attends and stores the new row) across a residual that grows past one
    32-row round of a residual warp, against append-then-attend through the oracle."""
    m = tk()
    B, H, D, R, T = 2, 8, 128, 128, 640
    rng = np.random.default_rng(77 + hq)
    k = orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))
    store = m.PagedKVCache(1, H, D, (4,), R, batch=B, page_tokens=64, max_tokens=T + 80, shuffle_pages=True)
    store.append(0, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16())
    states = []
    for b in range(B):
        st = orc.LayerState(H, D, 4, R)
        orc.append(st, k[b], v[b])
        states.append(st)
    for step in range(70):
        kn = orc.bf16_round(rng.normal(size=(B, 1, H, D)).astype(np.float32))
        vn = orc.bf16_round(rng.normal(size=(B, 1, H, D)).astype(np.float32))
        q = orc.bf16_round(rng.normal(size=(B, hq, D)).astype(np.float32))
        out = store.append_attend(0, torch.from_numpy(q).cuda(), torch.from_numpy(kn).cuda().bfloat16(),
                                  torch.from_numpy(vn).cuda().bfloat16(), out_dtype=torch.float32)
        for b in range(B):
            orc.append(states[b], kn[b], vn[b])
        if step in (0, 31, 32, 69):
            want = np.stack([orc.attend(q[b], states[b], hq)[0] for b in range(B)])
            assert np.abs(out.cpu().numpy() - want).max() <= 2e-3, step


@pytest.mark.parametrize("bits", [2, 4])
@pytest.mark.parametrize("mag", [2000.0, 8000.0])
def test_fast_extreme_value_range(bits, mag):
    """A value channel at +-mag: group scales far above 256 (2-bit: ~5000).  P' = -p*vscale enters the
    PV code MMA as f16; unscaled it overflowed to inf (NaN output) at 2-bit +-8000 — the kernel stores
    it times 2^-8 and scales the code term back."""
    m = tk()
    rng = np.random.default_rng(5)
    B, T, H, D, hq = 2, 700, 8, 128, 32
    k = rng.normal(size=(B, T, H, D))
    v = rng.normal(size=(B, T, H, D))
    v[:, :, 3, 17] = rng.choice([-mag, mag], size=(B, T))
    k[:, :, 2, 5] = rng.choice([-mag, mag], size=(B, T)) * 0.01
    k, v = orc.bf16_round(k.astype(np.float32)), orc.bf16_round(v.astype(np.float32))
    q = orc.bf16_round(rng.normal(size=(B, hq, D)).astype(np.float32))
    store = m.PagedKVCache(1, H, D, (bits,), 128, batch=B, page_tokens=64, max_tokens=T + 1, shuffle_pages=True)
    store.append(0, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16())
    want = []
    for b in range(B):
        st = orc.LayerState(H, D, bits, 128)
        orc.append(st, k[b], v[b])
        want.append(orc.attend(q[b], st, hq)[0])
    want = np.stack(want)
    out = store.attend(0, torch.from_numpy(q).cuda(), mode=2, out_dtype=torch.float32).cpu().numpy()
    assert np.isfinite(out).all()
    assert np.abs(out - want).max() <= 2e-3 * max(1.0, float(np.abs(want).max()))


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("where", ["mean", "scale", "query"])
def test_auto_mode_beyond_f16_range(bits, where):
    """The tensor-core kernels stage q, the means and P' as f16 (|x| < 65504).  A 1e5-magnitude channel shared by
    all heads (a mean >= 2^15), a 1e6 channel on one head only (a group scale beyond the kernel's P' range), or a
    1e5 query element makes
    mode 0 attend that layer on K2's exact f32 path (K1 records the range; K2 checks q): the answer equals the
    exact kernel's and the oracle's, never inf/NaN."""
    m = tk()
    rng = np.random.default_rng(60 + bits + len(where))
    B, T, H, D, hq = 2, 700, 8, 128, 32
    k = rng.normal(size=(B, T, H, D))
    v = rng.normal(size=(B, T, H, D))
    q = rng.normal(size=(B, hq, D))
    if where == "mean":
        v[:, :, :, 17] += 1e5
        k[:, :, :, 40] -= 1e5
    elif where == "scale":  # one head's group range ~1.9e6: scale >= 2^15 at 2/4 bits, >= 2^8 at 8 bits
        v[:, :, 3, 17] = rng.choice([-1e6, 1e6], size=(B, T))
    else:
        q[:, :, 5] = 1e5 * rng.choice([-1.0, 1.0], size=(B, hq))
    k, v, q = (orc.bf16_round(x.astype(np.float32)) for x in (k, v, q))
    store = m.PagedKVCache(1, H, D, (bits,), 128, batch=B, page_tokens=64, max_tokens=T + 1, shuffle_pages=True)
    store.append(0, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    want = []
    for b in range(B):
        st = orc.LayerState(H, D, bits, 128)
        orc.append(st, k[b], v[b])
        want.append(orc.attend(q[b], st, hq)[0])
    want = np.stack(want)
    qd = torch.from_numpy(q).cuda()
    auto = store.attend(0, qd, mode=0, out_dtype=torch.float32).cpu().numpy()
    exact = store.attend(0, qd, mode=1, out_dtype=torch.float32).cpu().numpy()
    assert np.isfinite(auto).all()
    scale = max(1.0, float(np.abs(want).max()))
    assert np.abs(exact - want).max() <= 1e-5 * scale
    assert np.abs(auto - want).max() <= 1e-5 * scale
    rng_words = store.range[0].tolist()
    routed = rng_words[0] >= 15 or rng_words[1] >= (8 if bits == 8 else 15)
    assert routed == (where != "query"), rng_words
    # the fused decode step takes the same path
    kn = orc.bf16_round(rng.normal(size=(B, 1, H, D)).astype(np.float32))
    step = store.append_attend(0, qd, torch.from_numpy(kn).cuda(), torch.from_numpy(kn).cuda(), out_dtype=torch.float32)
    assert torch.isfinite(step).all()


@pytest.mark.parametrize("bits,hq", [(4, 24), (2, 40), (8, 48), (8, 64), (4, 128)])
def test_fast_mapped_lse_and_auto(bits, hq):
    """Remapped group sizes (padding / two passes / G = 16) through attend_lse and mode 0: outputs within 2e-3
    of the oracle, lse equal to the exact kernel's within 2e-3, mode 0 on the tensor-core path."""
    m = tk()
    store, q, want = _paged_case(B=3, H=8, hq=hq, D=128, bits=bits, T=700, R=128, seed=500 + bits + hq)
    out, lse = store.attend_lse(0, q, mode=2)
    assert np.abs(out.float().cpu().numpy() - want).max() <= 2e-3
    out1, lse1 = store.attend_lse(0, q, mode=1)
    assert np.abs(lse.cpu().numpy() - lse1.cpu().numpy()).max() <= 2e-3
    auto = store.attend(0, q.bfloat16(), out_dtype=torch.float32)
    assert np.abs(auto.cpu().numpy() - want).max() <= 2e-3
    assert m is not None


@pytest.mark.parametrize("bits,hq,H", [(4, 24, 8), (8, 40, 8), (8, 64, 8), (4, 32, 4), (4, 28, 4), (4, 32, 16),
                                       (2, 32, 32)])
def test_fused_step_mapped_geometry(bits, hq, H):
    """append_attend at remapped group sizes and head counts (fused steps over several q-head passes / 8-head
    views: every pass stores its heads' new rows, the last one advances the lengths) equals append() + attend()
    bit for bit across residual flushes."""
    m = tk()
    B, T, D, R = 2, 200, 128, 8
    rng = np.random.default_rng(90 + bits + hq)
    k0 = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))).cuda().bfloat16()
    v0 = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, T, H, D)).astype(np.float32))).cuda().bfloat16()
    a = m.PagedKVCache(1, H, D, (bits,), R, batch=B, page_tokens=64, max_tokens=T + 64)
    b = m.PagedKVCache(1, H, D, (bits,), R, batch=B, page_tokens=64, max_tokens=T + 64)
    a.append(0, k0, v0)
    b.append(0, k0, v0)
    for step in range(12):
        q = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, hq, D)).astype(np.float32))).cuda().bfloat16()
        k1 = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, 1, H, D)).astype(np.float32))).cuda().bfloat16()
        v1 = torch.from_numpy(orc.bf16_round(rng.normal(size=(B, 1, H, D)).astype(np.float32))).cuda().bfloat16()
        oa = a.append_attend(0, q, k1, v1, out_dtype=torch.float32)
        b.append(0, k1, v1)
        ob = b.attend(0, q, out_dtype=torch.float32)
        assert torch.equal(oa, ob), f"step {step}"
    assert a.lengths(0) == b.lengths(0)


@pytest.mark.parametrize("H,hq,D", [(8, 32, 128), (8, 8, 128), (8, 64, 128), (32, 32, 128), (16, 32, 128), (4, 32, 128),
                                    (2, 16, 128), (1, 8, 128), (32, 64, 128), (8, 24, 64), (4, 4, 64), (16, 48, 64),
                                    (8, 16, 256), (4, 16, 256), (8, 32, 32), (1, 4, 32), (8, 24, 128), (4, 28, 128),
                                    (8, 40, 128), (2, 12, 64)])
@pytest.mark.parametrize("bits", [2, 4, 8, 16])
def test_exact_kernel_geometries(H, hq, D, bits):
    """The exact f32 kernel (mode 1: attn_exact2_kernel for head_dim 32 / 64 / 128 / 256) at MHA, GQA and MQA shapes and
    every width, ragged tails and several splits: within the reference's 1e-5 streaming bar."""
    store, q, want = _paged_case(B=2, H=H, hq=hq, D=D, bits=bits, T=333, R=16, seed=700 + H + hq + D + bits,
                                 poison=True)
    for splits in (1, 5, 37):  # 37: splits of 16 tokens and empty ones
        out = store.attend(0, q, num_splits=splits, mode=1)
        assert np.abs(out.cpu().numpy() - want).max() <= 1e-5, f"splits {splits}"


@pytest.mark.gpu
@pytest.mark.parametrize("H,hq,D", [(1, 8, 128), (1, 4, 32), (3, 12, 128), (1, 16, 64)])
@pytest.mark.parametrize("bits", [2, 4, 8])
def test_exact_kernel_odd_lengths(H, hq, D, bits):
    """Odd compressed lengths (residual 7) with odd KV head counts: the exact kernel's flat tile staging copies the
    metas of a partial tile as 16-byte chunks plus one 8-byte tail."""
    store, q, want = _paged_case(B=2, H=H, hq=hq, D=D, bits=bits, T=333, R=7, seed=900 + H + hq + D + bits,
                                 poison=True)
    assert all(store.lengths(0, b)[0] % 2 == 1 for b in range(2)), store.lengths(0)
    for splits in (1, 5, 37):
        out = store.attend(0, q, num_splits=splits, mode=1)
        assert np.abs(out.cpu().numpy() - want).max() <= 1e-5, f"splits {splits}"


@pytest.mark.parametrize("where", ["mean", "scale"])
def test_imported_cache_range_words(where):
    """A TADAKV1 stream with a mean >= 2^15 (or a group scale >= 2^8) imported by deserialize_cache sets the
    layer's range words like K1 does, so mode 0 attends it on the exact path (finite, equal to the oracle)."""
    m = tk()
    rng = np.random.default_rng(81 + len(where))
    T, H, D, hq, bits = 300, 8, 128, 32, 8
    k = rng.normal(size=(T, H, D))
    v = rng.normal(size=(T, H, D))
    if where == "mean":
        v[:, :, 17] += 1e5
    else:
        v[:, 3, 17] = rng.choice([-1e6, 1e6], size=T)  # 8-bit group scale ~7e3 >= 2^8
    k, v = orc.bf16_round(k.astype(np.float32)), orc.bf16_round(v.astype(np.float32))
    st = orc.LayerState(H, D, bits, 128)
    orc.append(st, k, v)
    cache = m.deserialize_cache(orc.dump(st))
    words = cache.store.range[0].tolist()
    assert (words[0] >= 15) if where == "mean" else (words[1] >= 8), words
    q = orc.bf16_round(rng.normal(size=(hq, D)).astype(np.float32))
    want = orc.attend(q, st, hq)[0]
    out = cache.store.attend(0, torch.from_numpy(q).cuda().unsqueeze(0), mode=0, out_dtype=torch.float32)[0]
    out = out.cpu().numpy()
    assert np.isfinite(out).all()
    assert np.abs(out - want).max() <= 1e-5 * max(1.0, float(np.abs(want).max()))


@pytest.mark.parametrize("H,hq,bits", [(16, 16, 4), (32, 32, 4), (32, 32, 2), (16, 64, 2), (24, 48, 8), (32, 64, 8),
                                       (16, 48, 4), (4, 32, 4), (4, 28, 4), (4, 16, 2), (2, 16, 4), (6, 24, 4),
                                       (2, 8, 8), (4, 32, 8)])
def test_fast_head_group_views(H, hq, bits):
    """Layouts with 16 / 24 / 32 KV heads (Llama-2 multi-head attention) on the tensor-core path as views of 8 KV
    heads each, and an even count below 8 (Qwen2's 4 KV / 28 q heads, 2 KV heads) as one view whose missing heads read as
    zeros: outputs and lse within 2e-3 of the oracle / exact kernel; mode 0 takes this path; append_attend (a fused
    step over the views) stays finite."""
    m = tk()
    store, q, want = _paged_case(B=2, H=H, hq=hq, D=128, bits=bits, T=600, R=16, seed=900 + H + hq + bits)
    out, lse = store.attend_lse(0, q, mode=2)
    assert np.abs(out.float().cpu().numpy() - want).max() <= 2e-3
    many = store.attend(0, q, mode=2, num_splits=37, out_dtype=torch.float32)  # the staging fits the workspace
    assert np.abs(many.cpu().numpy() - want).max() <= 2e-3
    _, lse1 = store.attend_lse(0, q, mode=1)
    assert np.abs(lse.cpu().numpy() - lse1.cpu().numpy()).max() <= 2e-3
    auto = store.attend(0, q.bfloat16(), out_dtype=torch.float32)
    assert np.abs(auto.cpu().numpy() - want).max() <= 2e-3
    rng = np.random.default_rng(H + hq)
    k1 = torch.from_numpy(orc.bf16_round(rng.normal(size=(2, 1, H, 128)).astype(np.float32))).cuda().bfloat16()
    step = store.append_attend(0, q, k1, k1, out_dtype=torch.float32)
    assert torch.isfinite(step).all()
    assert m is not None


@pytest.mark.parametrize("H,hq,bits,page_tokens", [(4, 28, 4, 32), (16, 32, 2, 128), (8, 24, 8, 32), (2, 16, 4, 256)])
def test_views_and_padding_other_page_sizes(H, hq, bits, page_tokens):
    """The remapped tensor-core paths (8-head views, padded group sizes) with 32 / 128 / 256-token pages."""
    store, q, want = _paged_case(B=3, H=H, hq=hq, D=128, bits=bits, T=500, R=16, seed=1300 + H + hq + page_tokens,
                                 page_tokens=page_tokens)
    out = store.attend(0, q, mode=2, out_dtype=torch.float32)
    assert np.abs(out.cpu().numpy() - want).max() <= 2e-3
