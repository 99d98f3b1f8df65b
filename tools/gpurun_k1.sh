python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
for V in 0 1 0 1; do echo "== NOORD=$V"; if [ $V = 1 ]; then export IRLS_K1_NOORD=1; else unset IRLS_K1_NOORD; fi; timeout 300 python tools/kbench.py --config config4 --solves 1 | grep -E "K1|solve"; done
unset IRLS_K1_NOORD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4" 2>&1 | tail -1
