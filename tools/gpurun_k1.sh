python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "512" 2>&1 | tail -1
for V in F B N F B N; do echo "== $V"; unset IRLS_K1_NOTMA IRLS_K1_BAR; if [ $V = N ]; then export IRLS_K1_NOTMA=1; fi; if [ $V = B ]; then export IRLS_K1_BAR=1; fi; timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K1"; done
unset IRLS_K1_NOTMA IRLS_K1_BAR
timeout 300 python -m pytest tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4" 2>&1 | tail -1
