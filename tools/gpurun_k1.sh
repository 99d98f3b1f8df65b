python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
for V in 0 2 3 0 2 3; do echo "== split $V"; IRLS_K1_SPLIT=$V timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K1"; done
IRLS_K1_SPLIT=3 timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4_golden_solve" 2>&1 | tail -1
