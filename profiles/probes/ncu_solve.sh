# ncu --set full of the warp-per-front solve kernels at c3
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
$B > gpurun_out/plain_so.json 2>&1 || exit 1
for spec in "bwd_small_tma 29 bwdsmall" "fwd_small_tma 10 fwdsmall" "fwd_top 3 fwdtop"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -f -o gpurun_out/ncu_$3 $B > gpurun_out/ncu_$3.log 2>&1
  python profiles/ncu_summary.py gpurun_out/ncu_$3.ncu-rep "$3 (c3)" > gpurun_out/ncu_$3.txt 2>&1
done
