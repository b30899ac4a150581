python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/exp_rank_share.py 4 32768 > gpurun_out/rank_share.log 2>&1
