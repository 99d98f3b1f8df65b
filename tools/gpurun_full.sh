# the whole -m gpu suite, smoke(), the default bench line, and the sensitivity runs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_full.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log; tail -3 gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_full.log; tail -2 gpurun_out/smoke_full.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 1200 python tools/sensitivity.py --out gpurun_out/sensitivity.json > gpurun_out/sensitivity.log 2>&1; echo "sens rc=$?"
