#!/usr/bin/env bash
# A/B of decode-attention builds: tests on the default build, then attn_bench per (bits:hq) for each lib.
#   CFGS="2:32 4:32" VARIANTS="variants/classic/libtadakv_b200.so" bash tools/ab_attn.sh
mkdir -p gpurun_out
if [[ -z "${NOTEST:-}" ]]; then
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_headline_parity.py tests/test_gpu_ragged.py -q -x > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
fi
: > gpurun_out/ab.log
for rep in 1 2; do
for v in "" ${VARIANTS:-}; do
  for cfg in ${CFGS:-2:32 4:32}; do
    bits=${cfg%%:*}; hq=${cfg#*:}
    echo "lib=$v" >> gpurun_out/ab.log
    TADA_LIB_PATH=$v timeout 300 python tools/attn_bench.py --bits $bits --hq $hq >> gpurun_out/ab.log 2>&1
  done
done
done
