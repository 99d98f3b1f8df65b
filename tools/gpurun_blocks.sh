python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_blocks.py -x -q --durations=10 > gpurun_out/pytest_blocks.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_blocks.log
tail -5 gpurun_out/pytest_blocks.log
timeout 900 python tools/block_quality.py --config 3 --blocks 0,16,64,256 --out gpurun_out/blocks_c3.json > gpurun_out/blocks_c3.log 2>&1
tail -6 gpurun_out/blocks_c3.log
