# Round-1 closing measurements after the warp-count tuning: GPU tests, bench lines (c3 with
# the CPU baseline, c3 reference arm, c5, c4), launch list with DRAM bytes
# (traffic.json), ncu --set full captures + summaries of the top kernels at
# their largest launches. Run from the repo root on the box.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/r1f_box_gpu.txt
python -m pytest tests -m gpu -q > gpurun_out/r1f_gpu_tests.txt 2>&1
python bench.py > gpurun_out/r1f_bench_c3.log 2>&1; tail -1 gpurun_out/r1f_bench_c3.log > gpurun_out/r1f_bench_c3.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1f_ref.log 2>&1; tail -1 gpurun_out/r1f_ref.log > gpurun_out/r1f_bench_c3_reference_arm.json
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r1f_bench_c5.log 2>&1; tail -1 gpurun_out/r1f_bench_c5.log > gpurun_out/r1f_bench_c5.json
bash profiles/launch_list_dram.sh r1f
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
for spec in "schur_update_kernel 13 schur" "front_kernel<.int.48 14 f48" "front_kernel<.int.32 12 f32" "bwd_small_kernel 29 bwdsmall" "big_assemble_kernel 12 asm" "dgemm_kernel 8 dgemm"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -f -o gpurun_out/ncu_r1f_$3 $B > gpurun_out/ncu_r1f_$3.log 2>&1
  python profiles/ncu_summary.py gpurun_out/ncu_r1f_$3.ncu-rep "$3 (c3, $B)" > gpurun_out/r1f_ncu_$3.txt 2>&1
done
timeout 1500 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1f_bench_c4.log 2>&1; tail -1 gpurun_out/r1f_bench_c4.log > gpurun_out/r1f_bench_c4.json
ls -la gpurun_out
