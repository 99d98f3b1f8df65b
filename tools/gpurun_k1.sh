python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "512" 2>&1 | tail -1
for V in T N T N; do echo "== $V"; if [ $V = N ]; then export IRLS_K1_NOTMA=1; else unset IRLS_K1_NOTMA; fi; timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K1"; done
unset IRLS_K1_NOTMA
timeout 300 python -m pytest tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --no-two-level > gpurun_out/bench_k1.json 2> gpurun_out/bench_k1.err; python -c "import json;d=json.load(open('gpurun_out/bench_k1.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'])"
