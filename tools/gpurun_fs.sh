python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fs.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
