python -m pytest tests/test_gpu.py -m gpu -x -q -k "variants or unknown_option" > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
