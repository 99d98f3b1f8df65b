python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
for ZP in 4 8 16 32; do echo "== ZP=$ZP"; IRLS_K1_ZP=$ZP python tools/kbench.py --config config4 --solves 1 | grep -E "K1|solve"; done
echo "== no z-march"; IRLS_K1_NOZM=1 python tools/kbench.py --config config4 --solves 1 | grep -E "K1|solve"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vgroup.py -x -q -k "512" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config4" 2>&1 | tail -2
