python bench.py > gpurun_out/bench_v13.json 2> gpurun_out/bench_v13.err
tail -c 300 gpurun_out/bench_v13.err
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:eigb --csv --log-file gpurun_out/launches_v13.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_v13.log 2>&1
echo "ncu rc=$?"
python tools/exp_rank_share.py 4 32768 > gpurun_out/rank_share.log 2>&1
python tools/exp_solver_share.py 2>&1 | head -4 > gpurun_out/share.log
