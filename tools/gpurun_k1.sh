python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
for V in P N P N P N; do echo "== $V"; unset IRLS_K1_NOPF; if [ $V = N ]; then export IRLS_K1_NOPF=1; fi; timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K1"; done
unset IRLS_K1_NOPF
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "512" 2>&1 | tail -1
