python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sweep_bb.py tests/test_gpu_parity.py tests/test_gpu_two_level.py tests/test_gpu_vgroup.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config2 or config4_golden_solve" 2>&1 | tail -2
python tools/sweep_time.py --config 4
