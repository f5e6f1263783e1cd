# Launch list with DRAM bytes per launch (one bench step after warm-up);
# writes profiles/traffic.json for bench.py's roofline.traffic.
# usage: bash profiles/launch_list_dram.sh <tag>
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-levels"
$B > gpurun_out/plain_$1.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_dram_$1.csv $B > gpurun_out/ncu_dram_$1.log 2>&1
python profiles/summarize.py gpurun_out/launches_dram_$1.csv gpurun_out/launches_dram_$1.md \
    --traffic profiles/traffic.json c3 2
cp profiles/traffic.json gpurun_out/traffic.json
