# bench at several nested-dissection leaf sizes (the front-size distribution)
for L in ${LEAVES:-16 24 32 40 48}; do
  python bench.py --no-cpu-baseline --no-e2e --no-levels --leaf-size $L > gpurun_out/ls.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ls.log').read().strip().splitlines()[-1]);r=d['roofline'];print('leaf', sys.argv[1], d['ms_per_step'], r['ms_per_step'], r['flops_per_shift'], d['residual'])" $L
done
