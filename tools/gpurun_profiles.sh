# end-of-round-2 profiles: launch lists (host loop: every kernel visible) and full captures of the top kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02f_launches_c4.csv python tools/profile_step.py --config config4 --T 50 --loop-mode 1 > gpurun_out/r02f_prof_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02f_launches_c3.csv python tools/profile_step.py --config config3 --T 50 --loop-mode 1 > gpurun_out/r02f_prof_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pair_pspmv|k_pair_axpy|k_pair_fused" -s 3 -c 3 -o gpurun_out/r02f_full_c4 python tools/profile_step.py --config config4 --T 2 --loop-mode 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sellp_pspmv|k_sellp_assemble" -s 2 -c 2 -o gpurun_out/r02f_full_c3 python tools/profile_step.py --config config3 --T 2 --loop-mode 1 > /dev/null 2>&1
echo done
