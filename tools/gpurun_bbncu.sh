python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_bb.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_bb_pass|k_bb_extract|k_side_cross_x|k_bb_cdelta" -c 4 -o gpurun_out/bb_pass python tools/sweep_time.py --config 4 --reps 1 > gpurun_out/bbncu.log 2>&1
tail -3 gpurun_out/bbncu.log
