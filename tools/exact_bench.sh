#!/usr/bin/env bash
# Decode-attention speed of the exact f32 kernel (mode 1) and the auto path (mode 0) on several geometries.
mkdir -p gpurun_out; : > gpurun_out/exact.log
run() { timeout 300 python tools/attn_bench.py "$@" --iters 5 --reps 3 >> gpurun_out/exact.log 2>&1; }
run --bits 4 --hq 32 --mode 1
run --bits 2 --hq 32 --mode 1
run --bits 8 --hq 32 --mode 1
run --bits 4 --hq 32 --heads 32 --mode 1 --batch 4
run --bits 4 --hq 32 --heads 32 --mode 0 --batch 4
run --bits 4 --hq 24 --mode 0
run --bits 4 --hq 8 --heads 8 --dim 64 --mode 0
run --bits 8 --hq 64 --mode 0
run --bits 4 --hq 32 --heads 16 --mode 0 --batch 8
run --bits 4 --hq 32 --heads 4 --mode 0
run --bits 4 --hq 28 --heads 4 --mode 0
run --bits 4 --hq 16 --heads 8 --dim 256 --mode 1
run --bits 4 --hq 32 --batch 1 --mode 1
run --bits 4 --hq 16 --heads 16 --dim 64 --mode 1 --batch 8
