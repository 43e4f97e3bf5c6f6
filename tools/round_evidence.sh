#!/usr/bin/env bash
# One gpurun session that refreshes the round's evidence: GPU tests, smoke, bench lines for configs
# 2 (headline), 4 (128k 2-bit) and 5 (70B shape), the ncu launch list and the dominant-kernel captures.
#   gpurun --timeout 2400 -- 'bash tools/round_evidence.sh'
set -u
mkdir -p gpurun_out
bash tools/gpu_session.sh tests
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/bench_c4.log 2>&1
timeout 1200 python bench.py --config 5 --steps 6 --warmup 3 > gpurun_out/bench_c5.log 2>&1
bash tools/gpu_session.sh ncu
bash tools/gpu_session.sh prof
bash tools/gpu_session.sh profk1
