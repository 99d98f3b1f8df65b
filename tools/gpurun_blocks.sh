python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_blk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_blocks.py -x -q > gpurun_out/pytest_blocks.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_blocks.log
tail -2 gpurun_out/pytest_blocks.log
timeout 900 python tools/block_quality.py --config 3 --blocks 0,8,16,64 --reps 2 --out gpurun_out/blocks_c3.json > gpurun_out/blocks_c3.log 2>&1
tail -6 gpurun_out/blocks_c3.log
for B in 16 64; do
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/blk${B}_launches.csv python tools/profile_step.py --config config3 --T 10 --loop-mode 1 --block-size $B > gpurun_out/blk${B}_prof.log 2>&1
python tools/launch_summary.py gpurun_out/blk${B}_launches.csv | head -6
done
