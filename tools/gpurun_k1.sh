python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
echo "== no prefetch"; python tools/kbench.py --config config4 --solves 2
echo "== prefetch"; IRLS_K1_PREFETCH=1 python tools/kbench.py --config config4 --solves 2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-two-level > gpurun_out/bench_k1.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_k1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernels'])"
