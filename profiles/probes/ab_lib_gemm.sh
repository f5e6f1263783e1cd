# A/B of library builds (build_variants/libkh_<name>.so; "default" = the in-tree library) on the c3 transform GEMMs
for v in "$@"; do
  if [ "$v" = default ]; then unset KHB200_LIB; else export KHB200_LIB=$PWD/build_variants/libkh_$v.so; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-levels > gpurun_out/ab.log 2>&1
  tail -n 1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['transform_gemms']; print('$v', 'step', round(d['ms_per_step'],2), 'gemm', round(k['ms_per_step'],3), round(k['frac'],3), 'res', d['residual'])" || tail -n 3 gpurun_out/ab.log
done
