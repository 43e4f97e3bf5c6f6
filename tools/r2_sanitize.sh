#!/usr/bin/env bash
# compute-sanitizer pass over the round-2 kernels (tools/sanitize_case.py shapes) -> gpurun_out/san.log
mkdir -p gpurun_out; : > gpurun_out/san.log
CS=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $1 $2" >> gpurun_out/san.log; timeout 600 $CS --tool $1 --print-limit 5 python tools/sanitize_case.py $2 >> gpurun_out/san.log 2>&1; }
for tool in memcheck racecheck; do
  run $tool "--bits 4 --hq 32"
  run $tool "--bits 2 --hq 64"
  run $tool "--bits 8 --hq 32"
  run $tool "--bits 4 --hq 24"
  run $tool "--bits 8 --hq 64"
  run $tool "--bits 4 --hq 32 --mode 1"
  run $tool "--bits 2 --hq 32 --heads 32 --mode 1"
  run $tool "--bits 8 --hq 16 --heads 16 --dim 64 --mode 1"
  run $tool "--bits 16 --hq 24 --heads 4 --dim 64 --mode 1"
  run $tool "--bits 4 --hq 8 --heads 1 --mode 1 --tokens 301 --residual 5"
  run $tool "--bits 2 --hq 12 --heads 3 --mode 1 --tokens 299 --residual 7"
done
run synccheck "--bits 4 --hq 32"
run synccheck "--bits 4 --hq 32 --mode 1"
run initcheck "--bits 4 --hq 24"
run initcheck "--bits 4 --hq 8 --heads 1 --mode 1 --tokens 301 --residual 5"
