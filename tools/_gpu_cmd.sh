python tools/exp_solver_share.py 2>&1 | head -4 > gpurun_out/share.log
python tools/exp_fpre.py 2>&1 | grep -v "Warn\|_warn" | head -8 >> gpurun_out/share.log
