python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
for K in 0 2 3; do echo "== IRLS_K1=$K"; IRLS_K1=$K python tools/kbench.py --config config4 --solves 1 | grep -E "K1|solve"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -2
IRLS_K1=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "512" 2>&1 | tail -2
