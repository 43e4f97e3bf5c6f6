"""Benchmark of the TaDA KV hot path on B200 (BASELINE.json metric / config 2).

Workload (``config.workload``): Llama-3-8B-shaped decode — 32 layers, 32 q / 8 kv
heads, head_dim 128, 32k context, batch 16 per GPU, searched-style per-layer
plan [8]*2 + [4]*22 + [2]*8, residual_length 128.  One STEP = one decode
token for every sequence through every layer: K1 append of the new token's K/V
(residual write; block flush every 128 steps) + K2/K3 split-K decode attention
over the compressed cache, then one NCCL all-gather of the step's attention
outputs when N > 1.  Multi-GPU: sequences are sharded by rank (weak scaling:
16 sequences per GPU), no collective inside the hot loop.

``value``  = decode tokens/s (whole job) with inputs resident in HBM.
``e2e``    = the same through the public API with pinned-host q / K / V copied in
             and attention outputs copied out every step.
``roofline`` = decode attention (K2+K3) algorithmic bytes / its CUDA-event time.
``quant_append`` = config 3's metric (prefill bulk quantize-append GB/s), measured
             while the 32k-token cache is built.
``cpu_baseline`` = the CPU oracle port (oracle/tada_oracle.py, numpy) timed on this
             host on a bounded sample, extrapolated to the same step.

``--impl reference`` times that CPU implementation alone on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn tokens/s + HBM GB/s vs roofline (Llama-3-8B, 32k ctx); quant-append GB/s"
# BASELINE.json configs that fit one GPU (per-GPU share for the weak-scaled ones).  2 is the headline.
CONFIGS = {
    2: dict(L=32, HQ=32, T=32768, B=16, plan=[8] * 2 + [4] * 22 + [2] * 8,
            workload="llama3-8b decode, 32 layers, 32q/8kv heads, head_dim 128, 32k ctx, batch 16/GPU, "
                     "plan [8]*2+[4]*22+[2]*8"),
    4: dict(L=32, HQ=32, T=131072, B=4, plan=[2] * 32,
            workload="llama3-8b long-context decode, 32 layers, 32q/8kv heads, head_dim 128, 128k ctx, batch 4/GPU, "
                     "uniform 2-bit"),
    5: dict(L=80, HQ=64, T=32768, B=16, plan=[4] * 80,
            workload="llama3-70b decode, 80 layers, 64q/8kv heads, head_dim 128, 32k ctx, batch 16/GPU "
                     "(128 at 8 GPUs), uniform 4-bit"),
}
H, D, R = 8, 128, 128
# --scaling strong: the global batch BASELINE.json quotes (config 5: 128 sequences, which fit only on 8 B200s)
STRONG_GLOBAL_BATCH = {2: 16, 4: 4, 5: 128}
L = HQ = T = B_PER_GPU = 0
PLAN: list = []
WORKLOAD = ""


def use_config(n: int) -> None:
    global L, HQ, T, B_PER_GPU, PLAN, WORKLOAD
    c = CONFIGS[n]
    L, HQ, T, B_PER_GPU, PLAN, WORKLOAD = c["L"], c["HQ"], c["T"], c["B"], list(c["plan"]), c["workload"]


use_config(2)


def tok_bytes(bits: int) -> int:
    """Algorithmic bytes per compressed context token per side: f32 mean + codes + f32 (scale, min)."""
    gb = D * 4 if bits == 16 else D * bits // 8
    return 4 * D + H * gb + 8 * H


def attn_alg_bytes(bits: int, batch: int, ctx_c: int, ctx_r: int) -> int:
    """One decode-attention launch (one layer, `batch` sequences): both sides + residual (bf16-accounted) + q/out."""
    return batch * (2 * ctx_c * tok_bytes(bits) + 2 * ctx_r * H * D * 2 + 2 * HQ * D * 2)


def attn_kernel_name(bits: int, hq: int) -> str:
    """The tensor-core decode kernel tada_decode_attn dispatches for this geometry (tada_attn.cu)."""
    if bits in (2, 4) and hq in (8, 16, 32, 64):
        return f"attn_v8_kernel<{bits},{hq}>"
    return f"attn_fast_kernel<{bits},{hq},{16 if bits != 8 else 32}>"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self, t_start=None, t_end=None):
        """Samples whose timestamp falls inside [t_start, t_end] (time.time() seconds) — the timed region."""
        import datetime

        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if ts is not None and t_start is not None and not (t_start - 0.06 <= ts <= t_end + 0.06):
                continue
            try:
                sm.append(float(parts[2]))
                mx = max(mx, float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        busy = [s for s in sm if s > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------ CPU oracle leg
_CPU = {}  # per worker process: the oracle LayerStates it built (one per plan width) and their append times


def _cpu_init(tokens: int, hq: int, widths: list) -> None:
    """Worker initializer (one host core): build one oracle (sequence, layer) cache per width with the
    reference's append_tokens policy (cache.py:154-180, R=128) at `tokens` tokens, timing each append —
    the CPU quantize-append baseline (config 3's metric)."""
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass
    from oracle import tada_oracle as orc

    rng = np.random.default_rng(1000 + os.getpid() % 1000)
    _CPU.update(states={}, append_s={}, hq=hq)
    for bits in widths:
        st = orc.LayerState(H, D, bits, R)
        k = orc.bf16_round(rng.normal(size=(tokens, H, D)).astype(np.float32))
        v = orc.bf16_round(rng.normal(size=(tokens, H, D)).astype(np.float32))
        t0 = time.perf_counter()
        orc.append(st, k, v)
        _CPU["append_s"][bits] = time.perf_counter() - t0
        _CPU["states"][bits] = st
    _CPU["q"] = orc.bf16_round(rng.normal(size=(hq, D)).astype(np.float32))


def _cpu_unit(_):
    """One sampled step's share of one worker: attend (attention.py:103-151, block 64) over its cache of
    each width once; returns the per-width unit times and the build-time append times."""
    from oracle import tada_oracle as orc

    times = {}
    for bits, st in _CPU["states"].items():
        t0 = time.perf_counter()
        orc.attend(_CPU["q"], st, _CPU["hq"], block=64)
        times[bits] = time.perf_counter() - t0
    return times, dict(_CPU["append_s"]), os.getpid()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class CpuOracle:
    """The CPU reference path (the numpy oracle port of tadakv, one process per host core) on a bounded
    sample of the configured workload.

    Setup (untimed): every worker appends `tokens` = min(T, 32768) tokens of bf16 K/V into one cache per
    plan width (timed per worker: the CPU quantize-append GB/s).  One STEP = every worker attends one
    (sequence, layer) unit of each width — workers x widths units, timed by the wall clock around the
    parallel map.  Decode tokens/s = workers / (time to attend one sequence through all L layers of the
    plan on one core), from the per-width median unit times (scaled linearly to T when T > tokens)."""

    def __init__(self, workers: int | None = None):
        self.workers = workers or min(os.cpu_count() or 1, 32)
        self.tokens = min(T, 32768)
        self.widths = sorted(set(PLAN), reverse=True)
        for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"  # inherited by the spawned workers before their numpy loads
        self.pool = mp.get_context("spawn").Pool(self.workers, initializer=_cpu_init,
                                                 initargs=(self.tokens, HQ, self.widths))
        self.unit = {b: [] for b in self.widths}
        self.append = {}
        self.step_s = []

    def step(self, timed: bool = True) -> float:
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_unit, range(self.workers), chunksize=1)
        dt = time.perf_counter() - t0
        for times, app, pid in res:
            self.append[pid] = app
            if timed:
                for b in self.widths:
                    self.unit[b].append(times[b])
        if timed:
            self.step_s.append(dt)
        return dt

    def close(self):
        self.pool.close()
        self.pool.join()

    def summary(self) -> dict:
        med = {b: statistics.median(self.unit[b]) * (T / self.tokens) for b in self.widths}
        seq_s = sum(med[b] for b in PLAN)  # one sequence through all L layers on one core
        tok_s = self.workers / seq_s
        alg = sum(attn_alg_bytes(b, 1, T, 0) for b in PLAN)  # per decoded token
        # quantize-append: bytes of config 3's accounting (bf16 K/V read + compressed write) per worker append
        app_bytes = {b: 2 * self.tokens * H * D * 2 + 2 * self.tokens * tok_bytes(b) for b in self.widths}
        app_s = {b: statistics.median([a[b] for a in self.append.values()]) for b in self.widths}
        append_gbs = self.workers * sum(app_bytes.values()) / sum(app_s.values()) / 1e9
        return {
            "tokens_per_s": tok_s, "alg_gbs": tok_s * alg / 1e9, "workers": self.workers,
            "unit_s": {str(b): med[b] for b in self.widths}, "steps_timed": len(self.step_s),
            "ms_per_step": 1e3 * statistics.median(self.step_s) if self.step_s else None,
            "append_gbs": append_gbs, "append_s_per_unit": {str(b): app_s[b] for b in self.widths},
            "cpu_model": cpu_model(),
            "sample": f"one step = {self.workers} processes (1 core each) x 1 (sequence, layer) attend per width "
                      f"{self.widths} at T={self.tokens}" + (f" (scaled x{T // self.tokens} to T={T})" if T != self.tokens else "")
                      + f"; tokens/s = {self.workers} / (sum over the {L} layers' per-width median unit times); "
                      f"append_gbs = {self.workers} workers x one {self.tokens}-token append_tokens per width",
        }


def parity_sample(store, outs, q_all, seq: int):
    """Checker (outside every timed region): the last timed step's bf16 output of one sampled sequence in
    the first layer of each width vs the CPU oracle's attend (attention.py:103-151) over that layer's
    exported compressed state — the same state the step attended (nothing was appended since).  Bar: the
    north_star's 2e-3 max-abs (|out| << 1 for these N(0, 1) inputs)."""
    from oracle import tada_oracle as orc

    rows = {}
    for bits in sorted(set(PLAN)):
        layer = PLAN.index(bits)
        ex = store.export(layer, seq)
        st = orc.LayerState(H, D, bits, R)
        st.kmean, st.vmean = ex["k_mean"].cpu().numpy(), ex["v_mean"].cpu().numpy()
        for name in ("k_dev", "v_dev"):
            d = ex[name].to_host()
            rec = orc.Deviation(bits, d.num_tokens, d.num_heads, d.group_size, d.codes, np.asarray(d.scales),
                                np.asarray(d.mins))
            setattr(st, "kdev" if name == "k_dev" else "vdev", rec)
        st.rk, st.rv = ex["residual_k"].cpu().numpy(), ex["residual_v"].cpu().numpy()
        q = q_all[layer][seq].float().cpu().numpy()
        want, _ = orc.attend(q, st, HQ)
        got = outs[layer][seq].float().cpu().numpy()
        rows[str(bits)] = {"layer": layer, "seq": seq, "tokens": st.compressed + st.r,
                           "max_abs": float(np.abs(got - want).max()), "out_absmax": float(np.abs(want).max())}
    worst = max(r["max_abs"] for r in rows.values())
    return {"max_abs": worst, "bar": 2e-3, "pass": worst <= 2e-3, "per_width": rows,
            "oracle": "oracle/tada_oracle.py attend over the exported state (bf16 output of the timed step)"}


def run_reference(args):
    """The reference arm: the CPU oracle port on this host's cores, K timed sampled steps after W warm-up
    steps (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cpu = CpuOracle()
    for _ in range(args.warmup):
        cpu.step(timed=False)
    for _ in range(args.steps):
        cpu.step()
    cpu.close()
    s = cpu.summary()
    v = s["tokens_per_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": s["steps_timed"], "warmup": args.warmup, "ms_per_step": s["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD + " (CPU oracle port, numpy)", "global_batch": B_PER_GPU, "seq_len": T,
                   "parallelism": f"{s['workers']} host processes"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": s["workers"], "kind": "port", "sample": s["sample"],
                         "cpu_model": s["cpu_model"], "append_gbs": s["append_gbs"], "alg_gbs": s["alg_gbs"]},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "hbm_gbs_equiv": s["alg_gbs"], "unit_s": s["unit_s"],
        "note": "ms_per_step is the wall time of one sampled step (see cpu_baseline.sample), not of a full decode step",
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2506_04642_b200 as tk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                "collective": "all_gather_into_tensor of the step's attention outputs (once per step, after the "
                              "last layer); no collective inside the per-layer hot loop"}
        print(f"[rank {rank}] NCCL communicator: {comm['nranks']} ranks, backend {comm['backend']}, "
              f"NCCL {comm['nccl_version']}", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    B = B_PER_GPU
    if args.scaling == "strong":  # the config's global batch split over the ranks
        global_b = STRONG_GLOBAL_BATCH.get(args.config, B_PER_GPU)
        if global_b % world:
            raise SystemExit(f"strong scaling: global batch {global_b} is not divisible by {world} GPUs")
        B = global_b // world
    need = B * (T + R) * sum(2 * tok_bytes(b) for b in PLAN)  # this rank's compressed cache bytes
    free = torch.cuda.mem_get_info(dev)[0]
    if need > 0.97 * free:
        raise SystemExit(f"config {args.config} x batch {B} per GPU needs ~{need / 1e9:.0f} GB of cache; "
                         f"{free / 1e9:.0f} GB free on this GPU ({args.scaling} scaling at {world} GPUs)")
    steps, warm = args.steps, args.warmup
    max_tokens = T + R + 2 * steps + warm + 16  # timed + e2e passes
    store = tk.PagedKVCache(L, H, D, PLAN, R, batch=B, page_tokens=64, max_tokens=max_tokens, shuffle_pages=True,
                            seed=rank)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1002 + rank)

    # ---- prefill: bulk quantize-append of 32k tokens into every layer (config 3's quant-append GB/s)
    # untimed warm-up of every width's append kernel (lazy module load, smem attributes) on a scratch cache
    widths = sorted(set(PLAN))
    scratch = tk.PagedKVCache(len(widths), H, D, widths, R, batch=B, page_tokens=64, max_tokens=2 * R + 64)
    for i in range(len(widths)):
        wk = torch.randn((B, 2 * R, H, D), generator=gen, device=dev).to(torch.bfloat16)
        scratch.append(i, wk, wk)
    torch.cuda.synchronize()
    del scratch
    qa_ms, qa_bytes = [], 0
    for layer in range(L):
        k = torch.randn((B, T, H, D), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)
        v = torch.randn((B, T, H, D), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        store.append(layer, k, v)
        e1.record()
        e1.synchronize()
        qa_ms.append(e0.elapsed_time(e1))
        qa_bytes += 2 * B * T * H * D * 2 + B * T * 2 * tok_bytes(PLAN[layer])
        del k, v
    store.check_errors()
    quant_append_gbs = qa_bytes / (sum(qa_ms) / 1e3) / 1e9

    # ---- per-step synthetic inputs (a few sets, cycled; the 35 GB cache is the traffic, >> L2)
    nsets = 4
    qs = [torch.randn((L, B, HQ, D), generator=gen, device=dev).to(torch.bfloat16) for _ in range(nsets)]
    ks = [torch.randn((L, B, 1, H, D), generator=gen, device=dev).to(torch.bfloat16) for _ in range(nsets)]
    vs = [torch.randn((L, B, 1, H, D), generator=gen, device=dev).to(torch.bfloat16) for _ in range(nsets)]
    outs = torch.empty((L, B, HQ, D), dtype=torch.bfloat16, device=dev)
    gathered = torch.empty((world, L, B, HQ, D), dtype=torch.bfloat16, device=dev) if world > 1 else None
    splits = {bits: store.suggest_splits(PLAN.index(bits), HQ) for bits in sorted(set(PLAN))}
    attn_events = []

    def step(i, q_in=None, k_in=None, v_in=None, record=False):
        s = i % nsets
        q_all = qs[s] if q_in is None else q_in
        k_all = ks[s] if k_in is None else k_in
        v_all = vs[s] if v_in is None else v_in
        group = None  # record=True: one event pair per run of consecutive same-width layers
        for layer in range(L):
            if record and (layer == 0 or PLAN[layer] != PLAN[layer - 1]):
                group = [torch.cuda.Event(enable_timing=True), None, 0, PLAN[layer], 0]
                group[0].record()
            # one decode step of the layer: append (residual row, or flush through K1) + K2/K3
            store.append_attend(layer, q_all[layer], k_all[layer], v_all[layer], out=outs[layer],
                                num_splits=splits[PLAN[layer]], mode=args.mode)
            if record:
                c, r = store.lengths(layer)
                group[2] += attn_alg_bytes(PLAN[layer], B, c, r)
                group[4] += 1
                if layer == L - 1 or PLAN[layer + 1] != PLAN[layer]:
                    group[1] = torch.cuda.Event(enable_timing=True)
                    group[1].record()
                    attn_events.append(tuple(group))
        if world > 1:
            dist.all_gather_into_tensor(gathered, outs)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(warm):
        step(i)
    barrier()
    from paper_2506_04642_b200._lib import launch_count

    launches_before = launch_count()
    with ClockSampler(local) as clk:
        time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        barrier()
        wall0 = time.time()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for i in range(steps):
            step(warm + i, record=True)  # one event pair per run of same-width layers (roofline per width)
        t1.record()
        barrier()
        wall1 = time.time()
        time.sleep(0.1)
    gpu_launches = launch_count() - launches_before
    ms = t0.elapsed_time(t1)
    parity = None
    if not args.no_parity:  # the timed step's output vs the oracle (untimed; before e2e changes the state)
        last = (warm + steps - 1) % nsets
        parity = parity_sample(store, outs, qs[last], seq=(5 + rank) % B)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # ---- e2e through the public API: pinned host q/K/V in, outputs out, every step.  As a serving loop
    # would, the copies run on their own streams and overlap compute: step i+1's q/K/V land (H2D stream)
    # while step i computes, and step i's outputs leave (D2H stream) while step i+1 computes; inputs and
    # outputs are double-buffered and ordered by one event per buffer and step (per-layer events on the
    # compute stream cost several us each).  Every byte is copied inside the timed region, every step.
    qh = [t.cpu().pin_memory() for t in qs[:2]]
    kh = [t.cpu().pin_memory() for t in ks[:2]]
    vh = [t.cpu().pin_memory() for t in vs[:2]]
    out_h = [torch.empty(outs.shape, dtype=outs.dtype).pin_memory() for _ in range(2)]
    q_d = [torch.empty_like(qs[0]) for _ in range(2)]
    k_d = [torch.empty_like(ks[0]) for _ in range(2)]
    v_d = [torch.empty_like(vs[0]) for _ in range(2)]
    outs2 = [outs, torch.empty_like(outs)]
    main = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]
    e2e_steps = max(3, steps)
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()

    def issue_h2d(j):
        bj = j % 2
        with torch.cuda.stream(h2d_s):
            if j >= 2:
                h2d_s.wait_event(comp_done[bj])  # step j-2 (same buffer) has finished reading it
            q_d[bj].copy_(qh[bj], non_blocking=True)
            k_d[bj].copy_(kh[bj], non_blocking=True)
            v_d[bj].copy_(vh[bj], non_blocking=True)
            h2d_done[bj].record(h2d_s)

    issue_h2d(0)
    for i in range(e2e_steps):
        bi = i % 2
        if i + 1 < e2e_steps:
            issue_h2d(i + 1)
        main.wait_event(h2d_done[bi])
        if i >= 2:
            main.wait_event(d2h_done[bi])  # step i-2's outputs (same buffer) have left
        for layer in range(L):
            store.append_attend(layer, q_d[bi][layer], k_d[bi][layer], v_d[bi][layer], out=outs2[bi][layer],
                                num_splits=splits[PLAN[layer]], mode=args.mode)
        if world > 1:
            dist.all_gather_into_tensor(gathered, outs2[bi])
        comp_done[bi].record(main)
        with torch.cuda.stream(d2h_s):
            d2h_s.wait_event(comp_done[bi])
            out_h[bi].copy_(outs2[bi], non_blocking=True)
            d2h_done[bi].record(d2h_s)
    main.wait_stream(d2h_s)
    main.wait_stream(h2d_s)
    t1.record()
    barrier()
    ms_per_step = ms / steps
    value = B * world * steps / (ms / 1e3)
    attn_ms = sum(e0.elapsed_time(e1) for e0, e1, _, _, _ in attn_events)
    attn_bytes = sum(b for _, _, b, _, _ in attn_events)
    step_bytes = attn_bytes / steps
    per_width = {}
    for bits in sorted(set(PLAN)):
        ev = [(e0.elapsed_time(e1), nb, n) for e0, e1, nb, wb, n in attn_events if wb == bits]
        per_width[str(bits)] = {"gbs": sum(nb for _, nb, _ in ev) / (sum(t for t, _, _ in ev) / 1e3) / 1e9,
                                "us_per_launch": 1e3 * sum(t for t, _, _ in ev) / sum(n for _, _, n in ev),
                                "layers": PLAN.count(bits)}
    dom = max(set(PLAN), key=PLAN.count)  # the dominant kernel: the 4-bit instantiation (22 of 32 layers)
    achieved = per_width[str(dom)]["gbs"]
    peak, peak_kind = peaks()

    e2e_ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = B * world * e2e_steps / (e2e_ms / 1e3)
    h2d = (qh[0].numel() + kh[0].numel() + vh[0].numel()) * 2
    d2h = out_h[0].numel() * 2
    store.check_errors()

    # dram bytes per launch of the dominant kernel from its ncu --set full capture (tools/make_profiles.py),
    # taken at B=16 x 32k compressed tokens: the same per-launch bytes as configs 2, 4 (4 x 128k) and 5
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(prof):
        try:
            for e in json.load(open(prof)).get("entries", []):
                if e["bits"] == dom and e["hq"] == HQ and B * T == 16 * 32768:
                    traffic, traffic_src = e["traffic_bytes_per_launch"], e["source"]
        except Exception:
            traffic = None

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            oracle_cpu = CpuOracle()
            oracle_cpu.step()
            oracle_cpu.close()
            c = oracle_cpu.summary()
            cpu = {"value": c["tokens_per_s"], "unit": "tokens/s", "cores": c["workers"], "kind": "port",
                   "sample": c["sample"], "alg_gbs": c["alg_gbs"], "append_gbs": c["append_gbs"],
                   "cpu_model": c["cpu_model"]}
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "u8 codes / f32 means+scales, bf16 q/out", "data": "synthetic (torch.randn bf16, seeded)",
            "config": {"workload": WORKLOAD, "global_batch": B * world, "seq_len": T, "layers": L,
                       "parallelism": f"seq-shard x{world}", "num_splits": {str(k): v for k, v in splits.items()}, "page_tokens": 64,
                       "kernel_mode": args.mode, "l2": "cache 35 GB/GPU >> 126 MB L2 (no flush needed)"},
            "hbm_gbs": step_bytes / (ms_per_step / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": f"decode attention K2+K3 (tada_decode_attn), {dom}-bit layers: {attn_kernel_name(dom, HQ)}"
                                   f" + combine_kv_kernel (K3)",
                         "alg_bytes_per_launch": attn_alg_bytes(dom, B, T, 1), "peak_source": peak_kind,
                         "frac_of_8tbs_spec": achieved / 8000.0, "per_width": per_width,
                         "all_layers_gbs": attn_bytes / (attn_ms / 1e3) / 1e9,
                         "alg_bytes_per_step": step_bytes, "attn_ms_per_step": attn_ms / steps,
                         # effective KV bytes streamed per decoded token (all layers, one sequence; step_bytes is this rank's), and the
                         # same as a fraction of a bf16 K/V cache's 2*H*D*2 bytes per token per layer
                         "kv_bytes_per_decoded_token": step_bytes / B,
                         "kv_bytes_vs_bf16": step_bytes / B / (L * T * 2 * H * D * 2)},
            "quant_append": {"value": quant_append_gbs, "unit": "GB/s", "frac": quant_append_gbs / peak,
                             "workload": f"prefill bulk quantize-append 32k tokens x batch {B} x 32 layers (config 3 "
                                         f"shape per sequence)", "ms_per_layer": statistics.median(qa_ms)},
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(wall0, wall1),
            "cpu_baseline": cpu,
            "parity": parity,
            "comm": comm if comm is None else dict(comm, bytes_per_step=int(gathered.numel()) * 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def self_launch(args) -> int:
    """--gpus N > 1 without a launcher: re-exec under torch.distributed.run, one rank per GPU (127.0.0.1
    rendezvous).  Fails (non-zero) when this box has fewer than N GPUs instead of running fewer ranks."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, this box has {have}", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", type=int, default=0, help="attention kernel: 0 auto, 1 exact generic, 2 tensor-core")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle leg")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-run oracle check of the timed step")
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE.json config (2 = headline; 4 = 128k 2-bit; 5 = 70B shape)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the config's batch per GPU; strong: the config's global batch split over the GPUs "
                         "(config 2: 16 sequences; config 5: 128)")
    args = ap.parse_args()
    use_config(args.config)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
