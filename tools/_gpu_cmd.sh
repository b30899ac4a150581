python bench.py > gpurun_out/bench_v15.json 2> gpurun_out/bench_v15.err
tail -c 300 gpurun_out/bench_v15.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
