python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k3.log 2>&1
for V in 0 1 2 3 0; do echo "== IRLS_K1S_V=$V"; IRLS_K1S_V=$V python tools/kbench.py --config config3 --solves 1 | grep -E "K1|K3"; done
for V in 1 3; do IRLS_K1S_V=$V timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "road or csr or random" 2>&1 | tail -1; done
