mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.json 2>&1 || exit 1
for spec in "big_diag 30 diag" "factor_dmma_small_kernel 10 small48" "bwd_small 7 bwdsmall" "big_assemble 4 asm" "big_trsm 4 trsm"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip $2 -c 1 -f -o gpurun_out/ncu_$3 $B > gpurun_out/ncu_$3.log 2>&1
done
ls -la gpurun_out
