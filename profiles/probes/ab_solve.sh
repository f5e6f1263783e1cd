# A/B of env knobs on the c3 solve time: bash profiles/probes/ab_solve.sh "VAR=a" "VAR=b" ...
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-levels > gpurun_out/ab.log 2>&1
  tail -n 1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['refinement_solves']; print('$cfg', 'step', round(d['ms_per_step'],2), 'solve', round(k['ms_per_step'],3), round(k['frac'],3), 'res', d['residual'])" || tail -n 3 gpurun_out/ab.log
done
