set -e
python tools/profile_case.py --n 8192 > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_8192.csv python tools/profile_case.py --n 8192 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dmma_gemm_nt_tma -c 1 -o gpurun_out/prof_gemm_tma python tools/profile_case.py --n 8192 > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:solve_roots_kernel -c 1 -o gpurun_out/prof_solve2 python tools/profile_case.py --n 8192 > gpurun_out/ncu_solve.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xt_tile_kernel -c 1 -o gpurun_out/prof_xt2 python tools/profile_case.py --n 8192 > gpurun_out/ncu_xt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:transform_partial -c 1 -o gpurun_out/prof_tf python tools/profile_case.py --n 8192 > gpurun_out/ncu_tf.log 2>&1
