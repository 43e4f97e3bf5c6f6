"""Copy the judged evidence from gpurun_out/ (scratch) into profiles/ (tracked).

python tools/make_profiles.py <tag>
  gpurun_out/attn_b<bits>_h<hq>.ncu-rep (4:32, 2:32, 4:64)
                            -> profiles/<tag>_attn4_ncu.txt / <tag>_attn_b2_h32_ncu.txt / <tag>_attn_b4_h64_ncu.txt
                               (headline metrics, stalls, opcode mix, hot lines)
                               profiles/attn_traffic.json   (dram bytes per launch per instantiation, read by bench.py)
  gpurun_out/launches.csv   -> profiles/<tag>_launches.csv + profiles/<tag>_launches.txt
  gpurun_out/bench.log      -> profiles/<tag>_bench.json (the bench line)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def run(*cmd):
    return subprocess.run([sys.executable, *cmd], capture_output=True, text=True, cwd=ROOT).stdout


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    entries = []
    for bits, hq in ((4, 32), (2, 32), (4, 64)):
        rep = os.path.join(OUT, f"attn_b{bits}_h{hq}.ncu-rep")
        if not os.path.exists(rep) and (bits, hq) == (4, 32):
            rep = os.path.join(OUT, "attn4.ncu-rep")  # older single-capture sessions
        if not os.path.exists(rep):
            continue
        name = "attn4" if (bits, hq) == (4, 32) else f"attn_b{bits}_h{hq}"
        tiles = 16 * 32768 // 16  # 16-token tiles of attn_v8_kernel<bits,hq> at B=16, T=32768
        txt = run("tools/ncu_summary.py", rep, str(tiles))
        txt += "\n--- per source line (top 40 by instructions + stalls)\n"
        txt += run("tools/ncu_lines.py", rep, "paper_2506_04642_b200/csrc/tada_attn_v8.cu", "40", str(tiles))
        open(os.path.join(PROF, f"{tag}_{name}_ncu.txt"), "w").write(
            "ncu --set full --clock-control none --import-source on -k regex:attn_v8 -s 3 -c 1 "
            f"python tools/attn_bench.py --bits {bits} --hq {hq} (B=16, T=32768, Hq={hq}, H=8, D=128)\n\n" + txt)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        d = dict(zip(rows[0], rows[2]))
        unit = dict(zip(rows[0], rows[1]))

        def nbytes(k):
            v = float(d[k])
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit[k]]

        gb = 128 * bits // 8
        entries.append({"kernel": f"attn_v8_kernel<{bits},{hq}>", "bits": bits, "hq": hq,
                        "traffic_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
                        "shape": f"B=16, T=32768 compressed, Hq={hq}, H=8, D=128, {bits}-bit",
                        "alg_bytes_per_launch": 16 * (32768 * 2 * (4 * 128 + 8 * gb + 64) + 2 * hq * 128 * 2),
                        "source": f"profiles/{tag}_{name}_ncu.txt"})
    if entries:
        json.dump({"entries": entries}, open(os.path.join(PROF, "attn_traffic.json"), "w"), indent=1)
    k1 = os.path.join(OUT, "k1.ncu-rep")
    if os.path.exists(k1):
        open(os.path.join(PROF, f"{tag}_k1_ncu.txt"), "w").write(
            "ncu --set full -k regex:quant_append -s 2 -c 1 python tools/k1_bench.py --bits 4 (B=8, T=32768, H=8, D=128)"
            "\n('tile' = one token, both sides)\n\n" + run("tools/ncu_summary.py", k1, str(8 * 32768)))
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches.csv"))
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write(
            "ncu --metrics gpu__time_duration.sum --clock-control none (2 decode steps of bench.py, after prefill "
            "and warm-up; cold-cache serialised launches: compare shares)\n" + run("tools/launch_summary.py", lc))
    bl = os.path.join(OUT, "bench.log")
    if os.path.exists(bl):
        for ln in open(bl):
            if ln.startswith("{"):
                open(os.path.join(PROF, f"{tag}_bench.json"), "w").write(ln)


if __name__ == "__main__":
    main()
