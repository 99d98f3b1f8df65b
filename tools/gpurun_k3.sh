python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k3.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "512" 2>&1 | tail -1
for V in T N T N; do echo "== $V"; if [ $V = N ]; then export IRLS_K3_NOTMA=1; else unset IRLS_K3_NOTMA; fi; timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K3|solve"; done
unset IRLS_K3_NOTMA
timeout 300 python -m pytest tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4" 2>&1 | tail -1
