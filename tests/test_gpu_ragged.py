"""Ragged batches and CUDA-graph decode steps (the reference keeps one cache per sequence, each with its
own length and flush state: cache.py:114-180).

* A batch of sequences at different lengths — ragged prefill (``lengths=``) and decode steps whose
  flushes happen at different steps per sequence — against one oracle state per sequence: the compressed
  state bit for bit (TADAKV1 fields) and every decode step's attention output (attention.py:103-151).
* One captured ``DecodeGraph`` step replayed across flushes equals the eager ``append_attend`` step bit
  for bit (outputs, lengths, cache state).
"""

import numpy as np
import pytest
import torch

from oracle import tada_oracle as orc

pytestmark = pytest.mark.gpu
H, D = 8, 128


def tk():
    import paper_2506_04642_b200 as m

    return m


def _rows(rng, *shape):
    return orc.bf16_round(rng.normal(size=shape).astype(np.float32))


def _check_state(store, layer, b, st):
    ex = store.export(layer, b)
    assert store.lengths(layer, b) == (st.compressed, st.r)
    assert np.array_equal(ex["k_mean"].cpu().numpy().view(np.uint32), st.kmean.view(np.uint32))
    assert np.array_equal(ex["v_mean"].cpu().numpy().view(np.uint32), st.vmean.view(np.uint32))
    for name, rec in (("k_dev", st.kdev), ("v_dev", st.vdev)):
        dev = ex[name].to_host()
        assert dev.codes == rec.payload, name
        assert np.array_equal(np.asarray(dev.scales).view(np.uint32), rec.scales.view(np.uint32)), name
    assert np.array_equal(ex["residual_k"].cpu().numpy(), st.rk)
    assert np.array_equal(ex["residual_v"].cpu().numpy(), st.rv)


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("R", [8, 0])
def test_ragged_prefill_and_decode_vs_per_sequence_oracle(bits, R):
    """B = 5 sequences with prompts of 13, 1, 30, 8 and 21 tokens, then 20 decode steps through
    append_attend (tensor-core K2/K3, every sequence flushing at its own steps when R = 8)."""
    m = tk()
    rng = np.random.default_rng(40 + bits + R)
    lens = [13, 1, 30, 8, 21]
    B, n, hq = len(lens), max(lens), 32
    k = _rows(rng, B, n, H, D)
    v = _rows(rng, B, n, H, D)
    store = m.PagedKVCache(1, H, D, (bits,), R, batch=B, page_tokens=64, max_tokens=n + 32, shuffle_pages=True)
    store.append(0, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16(), lengths=lens)
    states = []
    for b in range(B):
        st = orc.LayerState(H, D, bits, R)
        orc.append(st, k[b, :lens[b]], v[b, :lens[b]])
        states.append(st)
        _check_state(store, 0, b, st)
    for step in range(20):
        kn = _rows(rng, B, 1, H, D)
        vn = _rows(rng, B, 1, H, D)
        q = _rows(rng, B, hq, D)
        out = store.append_attend(0, torch.from_numpy(q).cuda(), torch.from_numpy(kn).cuda(),
                                  torch.from_numpy(vn).cuda(), out_dtype=torch.float32)
        for b in range(B):
            orc.append(states[b], kn[b], vn[b])
        want = np.stack([orc.attend(q[b], states[b], hq)[0] for b in range(B)])
        assert np.abs(out.cpu().numpy() - want).max() <= 2e-3, step
    store.check_errors()
    for b in range(B):
        _check_state(store, 0, b, states[b])
    # the exact kernel on the same ragged state (reference streaming bar)
    q = _rows(rng, B, hq, D)
    want = np.stack([orc.attend(q[b], states[b], hq)[0] for b in range(B)])
    got = store.attend(0, torch.from_numpy(q).cuda(), mode=1)
    assert np.abs(got.cpu().numpy() - want).max() <= 1e-5


def test_ragged_append_rope_equals_composition():
    """Ragged fused-RoPE appends (K1 rotates the compressed keys, the commit kernel the raw ones) leave the
    same bytes as rotating first (tada_apply_rope) and appending (append_fused == composition, AC8)."""
    m = tk()
    from paper_2506_04642_b200.rope import _positions, rope_table

    rng = np.random.default_rng(8)
    lens = [150, 3, 77, 128]
    B, n, rope = len(lens), max(lens), m.RopeParams(128)
    k = _rows(rng, B, n, H, D)
    v = _rows(rng, B, n, H, D)
    pos = np.stack([np.arange(n) + 11 * b for b in range(B)])
    a = m.PagedKVCache(1, H, D, (4,), 64, batch=B)
    b_ = m.PagedKVCache(1, H, D, (4,), 64, batch=B)
    pd, top = _positions(pos, n, B)
    kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    a.append_rope(0, kd, vd, pd, top, rope, lengths=lens)
    b_.append(0, b_._rotate(kd, pd, rope_table(rope, top)), vd, lengths=lens)
    # a second ragged chunk on top (residual rows of different counts flush at different points)
    lens2 = [40, 100, 0, 1]
    k2, v2 = _rows(rng, B, 100, H, D), _rows(rng, B, 100, H, D)
    pos2 = np.stack([np.arange(100) + lens[b] + 11 * b for b in range(B)])
    pd2, top2 = _positions(pos2, 100, B)
    a.append_rope(0, torch.from_numpy(k2).cuda(), torch.from_numpy(v2).cuda(), pd2, top2, rope, lengths=lens2)
    b_.append(0, b_._rotate(torch.from_numpy(k2).cuda(), pd2, rope_table(rope, top2)), torch.from_numpy(v2).cuda(),
              lengths=lens2)
    for s in range(B):
        assert a.lengths(0, s) == b_.lengths(0, s)
        ga, gb = a.export(0, s), b_.export(0, s)
        for name in ("k_mean", "v_mean", "residual_k", "residual_v"):
            assert torch.equal(ga[name], gb[name]), (s, name)
        for name in ("k_dev", "v_dev"):
            for x, y in zip(ga[name].device_tensors(), gb[name].device_tensors()):
                assert torch.equal(x, y), (s, name)


@pytest.mark.parametrize("hq,H,splits", [(32, 8, None), (64, 8, None), (28, 4, None), (32, 16, None), (24, 8, None),
                                          (32, 16, 4), (32, 32, 3)])
def test_decode_graph_replay_equals_eager(hq, H, splits):
    """A DecodeGraph captured once and replayed for 24 steps (two layers, plan (4, 2), R = 8: every sequence
    flushes during replays, at different steps) == the same steps run eagerly through append_attend; also for
    4 / 16 / 32 KV heads (8-head views) and a padded group size.  With explicit splits the 16 / 32-head views
    run as concurrent units on auxiliary streams (launch_fast_mapped), captured into the graph too."""
    m = tk()
    rng = np.random.default_rng(90 + hq + H)
    if splits:  # an eager call first, so the auxiliary streams exist before the capture
        warm = m.PagedKVCache(1, H, D, (4,), 8, batch=2, page_tokens=64, max_tokens=128)
        warm.append(0, torch.zeros(2, 40, H, D, device="cuda", dtype=torch.bfloat16),
                    torch.zeros(2, 40, H, D, device="cuda", dtype=torch.bfloat16))
        warm.attend(0, torch.zeros(2, hq, D, device="cuda", dtype=torch.bfloat16), num_splits=4)
    lens = [20, 5, 33, 12]
    B, n, L, R = len(lens), max(lens), 2, 8
    k = torch.from_numpy(_rows(rng, B, n, H, D)).cuda().bfloat16()
    v = torch.from_numpy(_rows(rng, B, n, H, D)).cuda().bfloat16()
    stores = [m.PagedKVCache(L, H, D, (4, 2), R, batch=B, page_tokens=64, max_tokens=n + 64) for _ in range(2)]
    for st in stores:
        for layer in range(L):
            st.append(layer, k, v, lengths=lens)
    eager, graphed = stores
    g = m.DecodeGraph(graphed, hq, num_splits={4: splits, 2: splits} if splits else None)
    for step in range(24):
        q = torch.from_numpy(_rows(rng, L, B, hq, D)).cuda().bfloat16()
        kn = torch.from_numpy(_rows(rng, L, B, 1, H, D)).cuda().bfloat16()
        vn = torch.from_numpy(_rows(rng, L, B, 1, H, D)).cuda().bfloat16()
        want = [eager.append_attend(i, q[i], kn[i], vn[i], out_dtype=torch.bfloat16, num_splits=g.splits[i])
                for i in range(L)]
        g.q.copy_(q)
        g.k.copy_(kn)
        g.v.copy_(vn)
        got = g.replay()
        for i in range(L):
            assert torch.equal(got[i], want[i]), (step, i)
    for i in range(L):
        assert torch.equal(eager.comp_len[i], graphed.comp_len[i]) and torch.equal(eager.res_len[i], graphed.res_len[i])
        for s in range(B):
            assert eager.lengths(i, s) == graphed.lengths(i, s)
            ea, ga = eager.export(i, s), graphed.export(i, s)
            for name in ("k_mean", "v_mean", "residual_k", "residual_v"):
                assert torch.equal(ea[name], ga[name]), (i, s, name)
