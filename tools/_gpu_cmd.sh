python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_v12.json 2> gpurun_out/bench_v12.err
tail -c 300 gpurun_out/bench_v12.err
python bench.py --impl reference > gpurun_out/bench_ref_v12.json 2> gpurun_out/bench_ref_v12.err; tail -c 300 gpurun_out/bench_ref_v12.err
