# Full ncu captures of single launches (run after the plain command succeeded).
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.json 2>&1 || exit 1
for spec in "schur_update_kernel 6 schur" "front_kernel<.int.48 2 f48" "front_kernel<.int.128 4 f128" "bwd_small_kernel 7 bwdsmall"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -f -o gpurun_out/ncu_$3 $B > gpurun_out/ncu_$3.log 2>&1
done
