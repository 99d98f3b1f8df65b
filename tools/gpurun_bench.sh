python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_b.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-two-level --e2e-steps 5 > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err; echo "rc=$?"; tail -2 gpurun_out/bench_pipe.err
python -c "import json;d=json.load(open('gpurun_out/bench_pipe.json'));print(d['value'],d['ms_per_step'],json.dumps(d['e2e'])[:1200])"
