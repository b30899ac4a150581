set -e
python tools/profile_case.py --n 8192 > gpurun_out/prof_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:solve_roots_kernel -c 1 -o gpurun_out/prof_solve python tools/profile_case.py --n 8192 > gpurun_out/ncu_solve.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xt_kernel -c 1 -o gpurun_out/prof_xt python tools/profile_case.py --n 8192 > gpurun_out/ncu_xt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dmma_gemm -c 1 -o gpurun_out/prof_gemm python tools/profile_case.py --n 8192 > gpurun_out/ncu_gemm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_case.py --n 8192 > gpurun_out/ncu_launch.log 2>&1
