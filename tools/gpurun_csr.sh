python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_csr.log 2>&1
timeout 900 python -m pytest tests/test_gpu_csr_prep.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "csr or road or config3 or error or prep or singular" > gpurun_out/pytest_csr.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_csr.log; tail -3 gpurun_out/pytest_csr.log
timeout 900 python bench.py --config config3 --steps 5 --warmup 3 --no-two-level --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d['e2e']), json.dumps(d['roofline']['kernels']))"
