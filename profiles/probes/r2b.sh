mkdir -p gpurun_out
python profiles/probes/ddcheck.py > gpurun_out/r2b_ddcheck.txt 2>&1
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/r2b_gpu_tests.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -rA > gpurun_out/r2b_fullsize.txt 2>&1
timeout 900 python profiles/probes/scaling_predict.py c3 c4 > gpurun_out/r2b_scaling.txt 2>&1
