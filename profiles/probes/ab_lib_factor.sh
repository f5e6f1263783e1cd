# A/B of library builds (build_variants/libkh_<name>.so; "default" = the in-tree library) on the c3 factorization
for v in "$@"; do
  if [ "$v" = default ]; then unset KHB200_LIB; else export KHB200_LIB=$PWD/build_variants/libkh_$v.so; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  tail -n 1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_step'],2), round(r['ms_per_step'],2), round(r['frac'],3), [round(l['ms'],3) for l in r['levels']], d['residual'])" || tail -n 3 gpurun_out/ab.log
done
