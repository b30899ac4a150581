python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python tools/exp_xt.py > gpurun_out/xt.log 2>&1
