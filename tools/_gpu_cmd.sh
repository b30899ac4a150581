EIGMOD_B200_OPTS=fpre_min_kp=1 python -m pytest tests/test_stress.py -m gpu -x -q > gpurun_out/gpu_stress_all.log 2>&1; tail -1 gpurun_out/gpu_stress_all.log
EIGMOD_B200_OPTS=sweep_poles=0 python -m pytest tests/test_stress.py tests/test_locate.py -m gpu -x -q > gpurun_out/gpu_stress_old.log 2>&1; tail -1 gpurun_out/gpu_stress_old.log
python tools/exp_rank_kernels.py 8 3 > gpurun_out/rk.log 2>&1
python tools/exp_fpre.py 2>&1 | grep -v "Warn\|_warn" | head -8 >> gpurun_out/rk.log
