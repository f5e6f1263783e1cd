for f in build_variants/lib_*.so; do
  KHB200_LIB=$PWD/$f timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bv.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/bv.log').read().strip().splitlines()[-1]);print(sys.argv[1], d['ms_per_step'], d['roofline']['ms_per_step'], d['residual'])" $f 2>/dev/null || { echo "$f FAILED"; grep -iE "error|Error" gpurun_out/bv.log | tail -3; }
done
