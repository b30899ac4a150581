python bench.py > gpurun_out/bench_v14.json 2> gpurun_out/bench_v14.err
tail -c 300 gpurun_out/bench_v14.err
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:eigb --csv --log-file gpurun_out/launches_v14.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_v14.log 2>&1
echo "ncu rc=$?"
python tools/exp_rank_share.py 4 32768 > gpurun_out/rank_share.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
