python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fz.log 2>&1
timeout 2400 python tools/fuzz_sweep_bb.py 40 5 > gpurun_out/fuzz_sweep_bb.txt 2>&1; echo "rc=$?"; tail -8 gpurun_out/fuzz_sweep_bb.txt
