python tools/profile_case.py --n 32768 > gpurun_out/pc.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"solve_roots_kernel|count_sweep_kernel|group_weights_kernel|fpresolve_kernel" -c 5 -o gpurun_out/k3_32k_v13 -f python tools/profile_case.py --n 32768 > gpurun_out/ncu_k3_v13.log 2>&1
echo "ncu rc=$?"
