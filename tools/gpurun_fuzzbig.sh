python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fz.log 2>&1
timeout 2400 python tools/fuzz_parity.py 600 21 > gpurun_out/fuzz_600.txt 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/fuzz_600.txt
timeout 2400 python tools/fuzz_sweep_bb.py 100 8 > gpurun_out/fuzz_sweep_bb_100.txt 2>&1; echo "bb rc=$?"; tail -2 gpurun_out/fuzz_sweep_bb_100.txt
