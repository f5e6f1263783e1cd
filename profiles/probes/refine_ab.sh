# Richardson vs FD-preconditioned GMRES refinement on c3, c5, c4
for cfg in c3 c5 c4; do
  for m in richardson gmres; do
    KH_REFINE=$m timeout 900 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-levels > gpurun_out/ra.log 2>&1
    python -c "import json,sys;d=json.loads(open('gpurun_out/ra.log').read().strip().splitlines()[-1]);print(sys.argv[1], sys.argv[2], round(d['ms_per_step'],1), d['refine_steps'], '%.2e'%d['residual'])" $cfg $m
  done
done
