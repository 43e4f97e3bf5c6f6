#!/usr/bin/env bash
# A/B of whole bench.py steps (config 2): the default build against VARIANTS, alternating, -> gpurun_out/ab_bench.log
mkdir -p gpurun_out; : > gpurun_out/ab_bench.log
for rep in 1 2 3; do
  for v in "" ${VARIANTS:-}; do
    echo "lib=$v" >> gpurun_out/ab_bench.log
    TADA_LIB_PATH=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/ab_bench.log
  done
done
