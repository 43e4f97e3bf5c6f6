mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not ref_suite" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
: > gpurun_out/ab.log
for rep in 1 2; do for v in "" xv/old.so; do
 for cfg in "--bits 4 --hq 32" "--bits 2 --hq 32" "--bits 8 --hq 32" "--bits 4 --hq 32 --heads 32 --batch 4" "--bits 4 --hq 8 --dim 64 --mode 0" "--bits 4 --hq 32 --batch 1"; do
  echo "lib=$v" >> gpurun_out/ab.log
  TADA_LIB_PATH=$v timeout 300 python tools/attn_bench.py --mode 1 $cfg >> gpurun_out/ab.log 2>&1
 done; done; done
