python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sweep_bb.py -x -q 2>&1 | tail -15
python tools/sweep_time.py --config 4
IRLS_SWEEP_FULL=1 python tools/sweep_time.py --config 4
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sweep|k_onesweep|k_scan|k_p0|k_final|k_side|k_bb" --csv --log-file gpurun_out/sweep_launches.csv python tools/sweep_time.py --config 4 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/sweep_launches.csv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_level.py tests/test_gpu_fullsize.py -x -q -k "sweep or tie or config1 or random or blob or two or golden_solve or config2" 2>&1 | tail -2
