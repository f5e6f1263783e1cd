# split solves of the m > 64 fronts: kernel tests (both paths), c3 bench A/B (KH_SPLIT_SOLVE)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/ss_tests.txt 2>&1; tail -n 1 gpurun_out/ss_tests.txt
KH_SPLIT_SOLVE=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "superlu or wide" > gpurun_out/ss_tests0.txt 2>&1; tail -n 1 gpurun_out/ss_tests0.txt
bash profiles/probes/ab_env.sh "KH_SPLIT_SOLVE=1" "KH_SPLIT_SOLVE=0"
for v in 1 0; do KH_SPLIT_SOLVE=$v python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v solves', d['kernels']['refinement_solves'])"; done
