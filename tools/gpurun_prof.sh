# launch lists (host loop: every kernel visible to ncu) + full captures of the top kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_prof.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_level.py tests/test_gpu_blocks.py -x -q > gpurun_out/pytest_prof.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_prof.log; tail -2 gpurun_out/pytest_prof.log
python tools/sweep_time.py --config 4 > gpurun_out/sweep_c4.json 2>&1; cat gpurun_out/sweep_c4.json
for B in 16 64; do
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/blk${B}_launches.csv python tools/profile_step.py --config config3 --T 10 --loop-mode 1 --block-size $B > gpurun_out/blk${B}_prof.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_block_factor|k_block_solve_iter" -c 2 -o gpurun_out/blk64_full python tools/profile_step.py --config config3 --T 2 --loop-mode 1 --block-size 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_onesweep|k_scan_argmin|k_sweep_prep" -c 3 -o gpurun_out/sweep_full python tools/sweep_time.py --config 4 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sweep|k_onesweep|k_scan|k_p0|k_final|k_side" --csv --log-file gpurun_out/sweep_launches.csv python tools/sweep_time.py --config 4 --reps 1 > /dev/null 2>&1
echo done
