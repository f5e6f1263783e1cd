# bench A/B over an environment switch: bash profiles/probes/ab_env.sh VAR "v1 v2 ..."
for v in $2; do
  env $1=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(sys.argv[1], d['ms_per_step'], d['roofline']['ms_per_step'], d['residual'])" "$1=$v"
done
