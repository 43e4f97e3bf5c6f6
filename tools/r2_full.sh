#!/usr/bin/env bash
# Round-2 evidence pass: GPU tests, smoke, bench (configs 2, 4, 5 and the reference arm), launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
if [[ -n "${FULL:-}" ]]; then
timeout 600 python bench.py --config 4 --steps 10 --no-cpu > gpurun_out/bench_c4.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --config 5 --steps 10 --no-cpu > gpurun_out/bench_c5.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-parity > gpurun_out/ncu_bench.log 2>&1
