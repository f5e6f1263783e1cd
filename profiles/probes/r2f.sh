T=${1:-r2f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -n 2 gpurun_out/${T}_gpu_tests.txt
python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1; tail -n 1 gpurun_out/${T}_bench_c3.log > gpurun_out/${T}_bench_c3.json
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_c3.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
