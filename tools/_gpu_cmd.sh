python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
EIGMOD_B200_OPTS=fpre_min_kp=1 python -m pytest tests/test_stress.py -m gpu -x -q > gpurun_out/gpu_stress_all.log 2>&1; tail -1 gpurun_out/gpu_stress_all.log
python tools/exp_fpre.py 2>&1 | grep -v "Warn\|_warn" | grep "fpre=" | head -2 > gpurun_out/share.log
