python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
IRLS_K1_ZP=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "512" 2>&1 | tail -1
for V in 0 4 8 16 32 0 8 16; do echo "== zp $V"; IRLS_K1_ZP=$V timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K1"; done
IRLS_K1_ZP=8 timeout 300 python -m pytest tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -1
IRLS_K1_ZP=8 timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4" 2>&1 | tail -1
