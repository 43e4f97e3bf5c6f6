#!/usr/bin/env bash
# A/B of K1 builds: K1 parity tests on the default build, then tools/k1_bench.py per width for each lib.
#   VARIANTS="variants/x/libtadakv_b200.so" bash tools/ab_k1.sh
mkdir -p gpurun_out
if [[ -z "${NOTEST:-}" ]]; then
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_cache.py tests/test_rope.py tests/test_gpu_ragged.py -q -x -m gpu > gpurun_out/tk1.log 2>&1; echo "rc=$?" >> gpurun_out/tk1.log
fi
: > gpurun_out/abk1.log
for rep in 1 2; do
for v in "" ${VARIANTS:-}; do
  for bits in ${BITS:-4 2 8}; do
    echo "lib=$v" >> gpurun_out/abk1.log
    TADA_LIB_PATH=$v timeout 300 python tools/k1_bench.py --bits $bits ${K1ARGS:-} >> gpurun_out/abk1.log 2>&1
  done
done
done
