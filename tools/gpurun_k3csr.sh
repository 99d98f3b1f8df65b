python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k3.log 2>&1
python tools/kbench.py --config config3 --solves 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "road or csr or random" 2>&1 | tail -2
