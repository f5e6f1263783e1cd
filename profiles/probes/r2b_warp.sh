# warp-front kernel: kernel parity tests, then c3 bench A/B (KH_WARP_CLASSES)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/wf_tests.txt 2>&1
tail -1 gpurun_out/wf_tests.txt
for wc in ${WCS:-0 1 2 3}; do
  KH_WARP_CLASSES=$wc timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/wf_bench_$wc.log 2>&1
  tail -1 gpurun_out/wf_bench_$wc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$wc', round(d['ms_per_step'],2), round(r['ms_per_step'],2), round(r['frac'],3), [round(l['ms'],3) for l in r['levels']])"
done
