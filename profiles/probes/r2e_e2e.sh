# e2e pipeline: GPU FD tests, e2e phases at c3
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fd.py tests/test_reference_objects.py tests/test_gpu_configs.py -x -q > gpurun_out/e2e_tests.txt 2>&1; tail -n 2 gpurun_out/e2e_tests.txt
python profiles/probes/e2e_phases.py c3 2>&1 | tail -3
