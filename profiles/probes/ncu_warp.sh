# ncu --set full of the warp-front kernels and the shared-memory m<=48 kernel at c3
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
KH_WARP_CLASSES=3 $B > gpurun_out/plain_wf.json 2>&1 || exit 1
for spec in "warp_front_kernel<.int.6 7 wf6" "warp_front_kernel<.int.4 5 wf4"; do
  set -- $spec
  KH_WARP_CLASSES=3 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -f -o gpurun_out/ncu_$3 $B > gpurun_out/ncu_$3.log 2>&1
  python profiles/ncu_summary.py gpurun_out/ncu_$3.ncu-rep "$3 (c3)" > gpurun_out/ncu_$3.txt 2>&1
done
ls -la gpurun_out/*.txt
