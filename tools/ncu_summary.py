"""One-screen summary of an ncu --set full report: headline metrics, stall reasons, SASS opcode mix.
Usage: python tools/ncu_summary.py report.ncu-rep [tiles]   (tiles: divide instruction counts per tile)"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 0
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    for k in ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
              "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
              "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "launch__grid_size"]:
        if k in d:
            print(f"{k:70s} {d[k]:>14s} {u.get(k, '')}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v.replace('.', '').isdigit()}
    tot = sum(st.values()) or 1
    print("stalls:", " ".join(f"{k}={100*v/tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    agg, hdr, n_all = collections.Counter(), None, 0.0
    for r in csv.reader(io.StringIO(sass)):
        if "Instructions Executed" in r and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            row = dict(zip(hdr, r))
            try:
                n = float(row["Instructions Executed"] or 0)
            except ValueError:
                continue
            toks = row["Source"].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            agg[op.split(".")[0]] += n
            n_all += n
    div = tiles or 1
    print(f"SASS instructions {n_all:.0f}" + (f" = {n_all/tiles:.0f}/tile" if tiles else ""))
    print("  ".join(f"{op}:{n/div:.0f}" for op, n in agg.most_common(24)))


if __name__ == "__main__":
    main()
