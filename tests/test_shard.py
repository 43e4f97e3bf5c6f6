"""Multi-GPU sharding: host logic on CPU (gloo, world_size 2) + the CUDA merge on one GPU.

* ShardPlan: batch-axis blocks and sequence-axis R-block interleaving.
* The union of the per-rank oracle caches equals the reference state (same compressed blocks,
  same residual rows), because quantization is per token and flushes move whole R-blocks
  (cache.py:98-111, 171-180).
* Partial (out, lse) pairs exchanged over a real process group merge to the single-rank answer.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tada_oracle as orc
from paper_2506_04642_b200.errors import ConfigError
from paper_2506_04642_b200.shard import ShardPlan, exchange_partials, gather_outputs


def test_plan_batch_axis_blocks():
    plans = [ShardPlan.make(4, r, 10, 128) for r in range(4)]
    assert all(p.axis == "batch" and p.parts == 1 for p in plans)
    ranges = [p.seq_range() for p in plans]
    assert ranges[0][0] == 0 and ranges[-1][1] == 10
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(3))
    assert sum(p.local_batch for p in plans) == 10
    assert plans[1].owned_spans(77, 5) == [(0, 5)]


def test_plan_sequence_axis_interleaves_blocks():
    world, batch, R = 8, 4, 128
    plans = [ShardPlan.make(world, r, batch, R) for r in range(world)]
    assert all(p.axis == "seq" and p.parts == 2 for p in plans)
    assert [p.seq_range()[0] for p in plans] == [0, 0, 1, 1, 2, 2, 3, 3]
    total = 1000
    owner = np.full(total, -1)
    for p in plans[:2]:
        for lo, hi in p.owned_spans(0, total):
            assert (owner[lo:hi] == -1).all()
            owner[lo:hi] = p.part
    assert (owner >= 0).all()
    assert all(owner[i] == (i // R) % 2 for i in range(total))
    # chunked appends route identically to one bulk append
    for p in plans[:2]:
        got, pos = [], 0
        for n in (1, 127, 3, 300, 1, 568):
            got += [(pos + lo, pos + hi) for lo, hi in p.owned_spans(pos, n)]
            pos += n
        flat = sorted(i for lo, hi in got for i in range(lo, hi))
        assert flat == [i for i in range(total) if owner[i] == p.part]
        assert p.local_tokens(total) == len(flat)


def test_plan_rejects_bad_geometry():
    with pytest.raises(ConfigError):
        ShardPlan.make(8, 0, 3, 128)
    with pytest.raises(ConfigError):
        ShardPlan.make(2, 2, 4, 128)


def _oracle_local_state(plan, k, v, schedule, bits, R):
    st = orc.LayerState(k.shape[1], k.shape[2], bits, R)
    pos = 0
    for n in schedule:
        for lo, hi in plan.owned_spans(pos, n):
            orc.append(st, k[pos + lo: pos + hi], v[pos + lo: pos + hi])
        pos += n
    return st


@pytest.mark.parametrize("R", [0, 16])
def test_union_of_rank_states_is_reference_state(R):
    rng = np.random.default_rng(7)
    H, D, T, bits = 2, 16, 150, 4
    k = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    schedule = [1, 40, 7, 60, 42]
    ref = orc.LayerState(H, D, bits, R)
    for a, n in zip(np.cumsum([0] + schedule[:-1]), schedule):
        orc.append(ref, k[a:a + n], v[a:a + n])
    plans = [ShardPlan.make(4, r, 2, R) for r in range(4)]  # 2 parts per sequence
    states = [_oracle_local_state(p, k, v, schedule, bits, R) for p in plans[:2]]
    blk = plans[0].block
    # reassemble the compressed rows in global token order
    comp_rows, res_rows = {}, {}
    for p, st in zip(plans[:2], states):
        toks = [i for lo, hi in p.owned_spans(0, T) for i in range(lo, hi)]
        for j in range(st.compressed):
            comp_rows[toks[j]] = (st, j)
        for j in range(st.r):
            res_rows[toks[st.compressed + j]] = (st, j)
    assert sorted(comp_rows) == list(range(ref.compressed))
    assert sorted(res_rows) == list(range(ref.compressed, T))
    gb = orc.group_nbytes(D, bits)
    for t, (st, j) in comp_rows.items():
        assert np.array_equal(st.kmean[j], ref.kmean[t])
        assert st.kdev.payload[j * H * gb:(j + 1) * H * gb] == ref.kdev.payload[t * H * gb:(t + 1) * H * gb]
        assert np.array_equal(st.vdev.scales[j * H:(j + 1) * H], ref.vdev.scales[t * H:(t + 1) * H])
    for t, (st, j) in res_rows.items():
        assert np.array_equal(st.rk[j], ref.rk[t - ref.compressed])
    assert blk == (R if R else 64)


def _gloo_worker(rank, world, port, q, k, v, schedule, bits, R, batch, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = ShardPlan.make(world, rank, batch, R)
        if plan.axis == "seq":
            st = _oracle_local_state(plan, k, v, schedule, bits, R)
            o, lse = orc.attend_lse(q, st, q.shape[0])
            o_parts, lse_parts = exchange_partials(torch.from_numpy(o), torch.from_numpy(lse), plan)
            merged = orc.merge_lse(o_parts[0].numpy(), lse_parts[0].numpy())
            result_q.put((rank, merged))
        else:
            a, b = plan.seq_range()
            local = torch.arange(a, b, dtype=torch.float32)[:, None].repeat(1, 3)
            full = gather_outputs(local, plan)
            result_q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


def _run_gloo(world, batch, R, port):
    rng = np.random.default_rng(11)
    H, D, Hq, T, bits = 2, 16, 4, 200, 4
    k = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    q = orc.bf16_round(rng.normal(size=(Hq, D)).astype(np.float32))
    schedule = [100, 1, 1, 98]
    ctx = mp.get_context("spawn")
    rq = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q, k, v, schedule, bits, R, batch, rq))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(rq.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res, (q, k, v, bits, R)


def test_gloo_sequence_axis_merge_matches_single_rank():
    res, (q, k, v, bits, R) = _run_gloo(world=2, batch=1, R=32, port=29611)
    ref = orc.LayerState(k.shape[1], k.shape[2], bits, R)
    orc.append(ref, k, v)
    want, _ = orc.attend(q, ref, q.shape[0])
    for rank in (0, 1):
        assert np.abs(res[rank] - want).max() <= 1e-5


def test_gloo_batch_axis_gather_ragged():
    res, _ = _run_gloo(world=2, batch=3, R=32, port=29612)
    for rank in (0, 1):
        assert res[rank][:, 0].tolist() == [0.0, 1.0, 2.0]


@pytest.mark.gpu
@pytest.mark.parametrize("R,mode", [(0, 1), (128, 1), (0, 2), (128, 2)])
def test_gpu_sequence_axis_two_ranks_on_one_device(R, mode):
    """Both ranks of a 2-way sequence split on one GPU; the CUDA merge equals the 1-rank oracle.  mode 1:
    the exact kernel (1e-5, the reference's streaming bar); mode 2: the tensor-core K2 + K3 that bench.py
    times, whose per-rank (out, lse) partials merge within the north_star's 2e-3."""
    import paper_2506_04642_b200 as tk
    from paper_2506_04642_b200.shard import merge_partials

    rng = np.random.default_rng(5)
    H, D, Hq, T, bits = 8, 128, 32, 700, 4
    k = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    v = orc.bf16_round(rng.normal(size=(T, H, D)).astype(np.float32))
    q = orc.bf16_round(rng.normal(size=(Hq, D)).astype(np.float32))
    ranks = [tk.ShardedKVCache(1, H, D, (bits,), R, batch=1, world=2, rank=r) for r in range(2)]
    kd = torch.from_numpy(k).cuda()[None]
    vd = torch.from_numpy(v).cuda()[None]
    pos = 0
    for n in (300, 1, 1, 398):
        for rk in ranks:
            rk.append(0, kd[:, pos:pos + n], vd[:, pos:pos + n])
        pos += n
    qd = torch.from_numpy(q).cuda()[None]
    parts = [rk.store.attend_lse(0, qd, mode=mode) for rk in ranks]
    o = torch.stack([p[0] for p in parts], dim=1)    # [1, 2, Hq, D]
    lse = torch.stack([p[1] for p in parts], dim=1)  # [1, 2, Hq]
    got = merge_partials(o, lse)[0].cpu().numpy()
    ref = orc.LayerState(H, D, bits, R)
    orc.append(ref, k, v)
    want, want_lse = orc.attend_lse(q, ref, Hq)
    assert np.abs(got - want).max() <= (1e-5 if mode == 1 else 2e-3)
    # each rank's lse matches the oracle on its own tokens
    for p, rk in zip(parts, ranks):
        st = _oracle_local_state(rk.plan, k, v, [300, 1, 1, 398], bits, R)
        _, l_r = orc.attend_lse(q, st, Hq)
        assert np.abs(p[1][0].cpu().numpy() - l_r).max() <= (1e-4 if mode == 1 else 2e-3)
