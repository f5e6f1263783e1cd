# A/B of library builds: bench line (c3 by default) per .so given as arguments
# (the in-tree library when the argument is "main").
# usage: bash profiles/probes/ab_libs.sh [--config cN] main build_variants/lib_x.so ...
CFG=""
if [ "$1" = "--config" ]; then CFG="--config $2"; shift 2; fi
for f in "$@"; do
  if [ "$f" = "main" ]; then unset KHB200_LIB; else export KHB200_LIB=$PWD/$f; fi
  python bench.py $CFG --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[1], 'step', round(d['ms_per_step'],3), 'factor', round(r['ms_per_step'],3), 'frac', round(r['frac'],4), 'res', d['residual'], 'steps', d['refine_steps'])" $f || tail -20 gpurun_out/ab.log
done
unset KHB200_LIB
