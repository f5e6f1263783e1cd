# Round-2 measurements on one B200 (run from the repo root on the box):
# GPU tests, bench lines (c3 with the CPU baseline, the reference arm, c1, c2,
# c4, c5), launch list with DRAM bytes (traffic.json), ncu --set full of the
# top kernels. usage: bash profiles/capture_r2.sh <tag>
T=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${T}_box_gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/${T}_box_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.txt 2>&1
python bench.py > gpurun_out/${T}_bench_c3.log 2>&1; tail -n 1 gpurun_out/${T}_bench_c3.log > gpurun_out/${T}_bench_c3.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.log 2>&1; tail -n 1 gpurun_out/${T}_ref.log > gpurun_out/${T}_bench_c3_reference_arm.json
for c in c1 c2 c5; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.log 2>&1; tail -n 1 gpurun_out/${T}_bench_$c.log > gpurun_out/${T}_bench_$c.json
done
timeout 1500 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_bench_c4.log 2>&1; tail -n 1 gpurun_out/${T}_bench_c4.log > gpurun_out/${T}_bench_c4.json
# launch list of the default configuration (two shift lanes: every launch covers half the shifts)
bash profiles/launch_list_dram.sh $T
# per-level breakdown, per-launch solve table and the ncu captures with one lane
# (whole-batch launches, levels not interleaved)
export KH_LANES=1 KH_SOLVE_LANES=1
cp profiles/traffic.json gpurun_out/traffic_keep.json
bash profiles/launch_list_dram.sh ${T}_1lane
cp gpurun_out/traffic_keep.json profiles/traffic.json
python profiles/level_breakdown.py gpurun_out/launches_dram_${T}_1lane.csv > gpurun_out/${T}_level_breakdown.txt 2>&1
python profiles/solve_launches.py gpurun_out/launches_dram_${T}_1lane.csv > gpurun_out/${T}_solve_launches.md 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
for spec in "schur_update_kernel 11 schur" "warp_front_kernel<.int.6 7 wf6" "warp_front_kernel<.int.5 7 wf5" "warp_front_kernel<.int.4 5 wf4" "front_kernel<.int.96 4 f96" "pivot_warp_kernel 12 pivot" "panel_trsm_kernel 12 ptrsm" "bwd_small_tma_kernel 66 bwdsmall" "fwd_stream_kernel 5 fwdstream" "dgemm_kernel 8 dgemm"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -f -o gpurun_out/ncu_${T}_$3 $B > gpurun_out/ncu_${T}_$3.log 2>&1
  python profiles/ncu_summary.py gpurun_out/ncu_${T}_$3.ncu-rep "$3 (c3, $B)" > gpurun_out/${T}_ncu_$3.txt 2>&1
  python profiles/ncu_lines.py gpurun_out/ncu_${T}_$3.ncu-rep "" 25 >> gpurun_out/${T}_ncu_$3.txt 2>&1
done
ls -la gpurun_out | grep $T
