# Round-1 closing measurement after the bulk write-out: GPU tests, c3 bench
# line (CPU baseline, e2e, per-level roofline), launch list with DRAM bytes.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r1e_gpu_tests.txt 2>&1
python bench.py > gpurun_out/r1e_bench_c3.log 2>&1; tail -1 gpurun_out/r1e_bench_c3.log > gpurun_out/r1e_bench_c3.json
bash profiles/launch_list_dram.sh r1e
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:front_kernel<.int.48" --launch-skip 14 -c 1 -f -o gpurun_out/ncu_r1e_f48 $B > gpurun_out/ncu_r1e_f48.log 2>&1
python profiles/ncu_summary.py gpurun_out/ncu_r1e_f48.ncu-rep "f48 (c3, $B)" > gpurun_out/r1e_ncu_f48.txt 2>&1
