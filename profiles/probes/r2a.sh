T=r2a
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${T}_box_gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/${T}_box_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_gpu_tests.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1; tail -1 gpurun_out/${T}_bench_c3.log > gpurun_out/${T}_bench_c3.json
bash profiles/launch_list_dram.sh $T
