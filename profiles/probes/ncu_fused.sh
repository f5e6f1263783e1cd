# ncu --set full of the shared-memory fused-front kernels and the Schur kernel at c3
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
$B > gpurun_out/plain_fu.json 2>&1 || exit 1
for spec in "front_kernel<.int.96 4 f96" "front_kernel<.int.128 5 f128" "front_kernel<.int.64 6 f64" "schur_update_kernel 11 schur"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -f -o gpurun_out/ncu_$3 $B > gpurun_out/ncu_$3.log 2>&1
  python profiles/ncu_summary.py gpurun_out/ncu_$3.ncu-rep "$3 (c3)" > gpurun_out/ncu_$3.txt 2>&1
done
ls -la gpurun_out/*.txt
