"""Where does the e2e loop lose time against the device-resident loop?  (bench.py config 2 shape)

python tools/e2e_probe.py   -> ms/step of: resident inputs | copy-stream loop without copies | with copies
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04642_b200 as tk  # noqa: E402

L, H, D, HQ, T, B, R = 32, 8, 128, 32, 32768, 16, 128
PLAN = [8] * 2 + [4] * 22 + [2] * 8


def main():
    dev = torch.device("cuda")
    steps = 10
    store = tk.PagedKVCache(L, H, D, PLAN, R, batch=B, page_tokens=64, max_tokens=T + R + 8 * steps + 16,
                            shuffle_pages=True)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for layer in range(L):
        k = torch.randn((B, T, H, D), generator=g, device=dev).to(torch.bfloat16)
        store.append(layer, k, k)
        del k
    qs = [torch.randn((L, B, HQ, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(2)]
    ks = [torch.randn((L, B, 1, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(2)]
    outs = [torch.empty((L, B, HQ, D), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    splits = {b: store.suggest_splits(PLAN.index(b), HQ) for b in set(PLAN)}

    def layers(q, k, out):
        for layer in range(L):
            store.append_attend(layer, q[layer], k[layer], k[layer], out=out[layer], num_splits=splits[PLAN[layer]])

    def timed(fn):
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        fn()
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / steps

    for i in range(3):
        layers(qs[i % 2], ks[i % 2], outs[i % 2])
    if os.environ.get("PROBE_DRIFT"):  # resident loop repeated: GPU ms/step and host enqueue ms/step
        import time

        for rep in range(6):
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for i in range(steps):
                layers(qs[i % 2], ks[i % 2], outs[i % 2])
            t1.record()
            h1 = time.perf_counter()
            torch.cuda.synchronize()
            import subprocess

            smi = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                                  "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
            print(f"rep {rep} residual ~{3 + rep * steps}..{3 + (rep + 1) * steps}: gpu {t0.elapsed_time(t1) / steps:.3f} "
                  f"ms/step, host enqueue {(h1 - h0) * 1e3 / steps:.3f} ms/step  [{smi}]", flush=True)
            if os.environ.get("PROBE_COOL"):
                time.sleep(float(os.environ["PROBE_COOL"]))
        return
    res = {"resident": timed(lambda: [layers(qs[i % 2], ks[i % 2], outs[i % 2]) for i in range(steps)])}

    main_s = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    qh = [t.cpu().pin_memory() for t in qs]
    kh = [t.cpu().pin_memory() for t in ks]
    oh = [torch.empty(outs[0].shape, dtype=outs[0].dtype).pin_memory() for _ in range(2)]
    qd = [torch.empty_like(qs[0]) for _ in range(2)]
    kd = [torch.empty_like(ks[0]) for _ in range(2)]
    ev = {n: [torch.cuda.Event() for _ in range(2)] for n in ("h2d", "comp", "d2h")}

    def loop(copy_in, copy_out):
        def h2d(j):
            bj = j % 2
            with torch.cuda.stream(h2d_s):
                if j >= 2:
                    h2d_s.wait_event(ev["comp"][bj])
                if copy_in:
                    qd[bj].copy_(qh[bj], non_blocking=True)
                    kd[bj].copy_(kh[bj], non_blocking=True)
                ev["h2d"][bj].record(h2d_s)

        h2d(0)
        for i in range(steps):
            bi = i % 2
            if i + 1 < steps:
                h2d(i + 1)
            main_s.wait_event(ev["h2d"][bi])
            if i >= 2:
                main_s.wait_event(ev["d2h"][bi])
            layers(qd[bi], kd[bi], outs[bi])
            ev["comp"][bi].record(main_s)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev["comp"][bi])
                if copy_out:
                    oh[bi].copy_(outs[bi], non_blocking=True)
                ev["d2h"][bi].record(d2h_s)
        main_s.wait_stream(d2h_s)
        main_s.wait_stream(h2d_s)

    for name, ci, co in (("events only", False, False), ("h2d only", True, False), ("d2h only", False, True),
                         ("h2d + d2h", True, True)):
        res[name] = timed(lambda: loop(ci, co))
    res["resident again"] = timed(lambda: [layers(qs[i % 2], ks[i % 2], outs[i % 2]) for i in range(steps)])
    for k, v in res.items():
        print(f"{k:16s} {v:.3f} ms/step  {B / v * 1e3:.1f} tok/s")


if __name__ == "__main__":
    main()
