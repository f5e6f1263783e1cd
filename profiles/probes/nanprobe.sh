KH_POISON=1 KH_SMALL_MAX=0 python profiles/probes/nan_factors.py 64 2>&1 | tail -10
KH_POISON=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
