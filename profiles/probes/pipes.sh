# bench at 1, 2, 4 shift pipelines (engine.FDEngine pipes)
for np in 1 2 4; do
  KH_PIPES=$np python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bp.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1]);print('pipes', sys.argv[1], d['ms_per_step'], d['roofline']['ms_per_step'], d['residual'])" $np
done
