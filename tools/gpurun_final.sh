# the whole -m gpu suite, smoke(), the default bench line, the fuzz parity run
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_final.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_final.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_final.log; tail -3 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log; tail -2 gpurun_out/smoke_final.log
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_final.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['serial']['value'],d['roofline']['frac'],d['clocks'])"
timeout 900 python tools/fuzz_parity.py 200 13 > gpurun_out/fuzz_final.txt 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/fuzz_final.txt
