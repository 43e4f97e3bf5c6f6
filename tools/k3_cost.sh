mkdir -p gpurun_out; : > gpurun_out/k3.log
for bits in 4 2; do for T in 32768 32868; do for dg in 0 3; do
 echo "bits=$bits T=$T diag=$dg" >> gpurun_out/k3.log
 TADA_ATTN_DIAG=$dg python tools/attn_bench.py --bits $bits --hq 32 --tokens $T >> gpurun_out/k3.log 2>&1
done; done; done
