python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_b.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "rc=$?"; tail -2 gpurun_out/bench_final.err
python -c "import json;d=json.load(open('gpurun_out/bench_final.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['serial']['value'],d['roofline']['frac'],d['clocks'],d['cpu_baseline']['value'])"
timeout 900 python bench.py --no-cpu-baseline --no-two-level --config config3 > gpurun_out/bench_config3.json 2> gpurun_out/bench_config3.err; echo "rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_config3.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['serial']['value'],d['roofline']['frac'])"
