# Launch list of one bench step (after the same command ran cleanly without ncu).
# usage: bash profiles/launch_list.sh <tag>
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
$B > gpurun_out/plain_$1.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(?!at::|cutlass|cublas|void at::|void cutlass)' \
    --csv --log-file gpurun_out/launches_$1.csv $B > gpurun_out/ncu_$1.log 2>&1
python profiles/summarize.py gpurun_out/launches_$1.csv gpurun_out/launches_$1.md
