mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench_default.log | cut -c1-1500
