#!/usr/bin/env bash
# One gpurun session: GPU tests, smoke, micro-benches, bench line, ncu launch list.
# Usage (from this container):
#   gpurun --timeout 1500 -- 'bash tools/gpu_session.sh [tests|bench|ncu|all]'
# Everything lands in gpurun_out/; each step has its own timeout so one hang cannot eat the call.
set -u
what=${1:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
if [[ ! -f paper_2506_04642_b200/libtadakv_b200.so ]]; then make -j8 > gpurun_out/make.log 2>&1; fi

if [[ $what == tests || $what == all ]]; then
  timeout 900 python -m pytest tests -m gpu -q -rA --timeout 120 --durations 25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [[ $what == micro || $what == all ]]; then
  : > gpurun_out/micro.log
  for bits in 2 4 8; do
    for mode in ${MODES:-2}; do
      timeout 300 python tools/attn_bench.py --bits $bits --mode $mode >> gpurun_out/micro.log 2>&1
    done
  done
fi
if [[ $what == bench || $what == all ]]; then
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
if [[ $what == prof || $what == all ]]; then
  # the dominant kernel of each bench config: 4-bit Hq=32 (config 2), 2-bit Hq=32 (config 4), 4-bit Hq=64 (config 5)
  : > gpurun_out/prof.log
  for cfg in ${PROF_CFGS:-4:32 2:32 4:64}; do
    bits=${cfg%%:*}; hq=${cfg#*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:${PROF_KERNEL:-attn_v8} -s 3 -c 1 \
      -o gpurun_out/attn_b${bits}_h${hq} -f python tools/attn_bench.py --bits $bits --hq $hq --iters 2 >> gpurun_out/prof.log 2>&1
    echo "prof $cfg rc=$?" >> gpurun_out/prof.log
  done
  cp gpurun_out/attn_b4_h32.ncu-rep gpurun_out/attn4.ncu-rep 2>/dev/null
fi
if [[ $what == ncu || $what == all ]]; then
  # skip prefill (2 launches/layer) + 3 warm-up steps (3 launches/layer/step), list 2 steps
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'attn|combine|residual|lengths|quant' \
    -s 352 -c 192 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
fi
if [[ $what == profk1 || $what == all ]]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_append -s 2 -c 1 \
    -o gpurun_out/k1 -f python tools/k1_bench.py --bits 4 > gpurun_out/profk1.log 2>&1
  echo "profk1 rc=$?" >> gpurun_out/profk1.log
fi
