python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_level.py tests/test_gpu_edge_cases.py tests/test_gpu_vgroup.py tests/test_gpu_fullsize.py -x -q -k "not every_step" > gpurun_out/pytest_sweep.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_sweep.log
tail -3 gpurun_out/pytest_sweep.log
python tools/sweep_time.py --config 4 > gpurun_out/sweep_c4.json 2>&1
python tools/sweep_time.py --config 3 > gpurun_out/sweep_c3.json 2>&1
cat gpurun_out/sweep_c4.json gpurun_out/sweep_c3.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sweep|k_onesweep|k_delta|k_tile|k_final|k_side" --csv --log-file gpurun_out/sweep_launches.csv python tools/sweep_time.py --config 4 --reps 1 > /dev/null 2>&1
echo "ncu rc=$?"
