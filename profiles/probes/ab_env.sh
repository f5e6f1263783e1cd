# A/B of env knobs on the c3 bench: bash profiles/probes/ab_env.sh "VAR=a VAR2=b" "VAR=c" ...
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  tail -n 1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', round(d['ms_per_step'],2), round(r['ms_per_step'],2), round(r['frac'],3), [round(l['ms'],3) for l in r['levels']])" || tail -n 3 gpurun_out/ab.log
done
