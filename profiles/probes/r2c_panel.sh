# two-launch panel path for large fronts: kernel tests (both paths), c3 bench A/B (KH_PANEL_INV)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pi_tests.txt 2>&1
tail -1 gpurun_out/pi_tests.txt
KH_WARP_CLASSES=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k superlu > gpurun_out/pi_tests0.txt 2>&1
tail -1 gpurun_out/pi_tests0.txt
for v in 1; do
  KH_PANEL_INV=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pi_bench_$v.log 2>&1
  tail -1 gpurun_out/pi_bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_step'],2), round(r['ms_per_step'],2), round(r['frac'],3), [round(l['ms'],3) for l in r['levels']])"
done
