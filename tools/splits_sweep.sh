#!/usr/bin/env bash
# Split-count sweep of the decode kernels at config 2's shape (B=16, T=32k): gpurun_out/splits.log
mkdir -p gpurun_out; : > gpurun_out/splits.log
for rep in 1 2; do
for cfg in "--bits 4 --hq 32" "--bits 2 --hq 32" "--bits 8 --hq 32" "--bits 4 --hq 64"; do
  for s in ${SPLITS:-9 18 27 37 55 74}; do
    timeout 120 python tools/attn_bench.py $cfg --splits $s >> gpurun_out/splits.log 2>&1
  done
done
done
