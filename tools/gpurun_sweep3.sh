python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sweep_bb.py -x -q 2>&1 | tail -5
python tools/sweep_time.py --config 3
python tools/sweep_time.py --config 4
