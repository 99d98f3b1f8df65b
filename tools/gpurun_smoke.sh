python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/smoke_ncu.log
python tools/launch_summary.py gpurun_out/smoke_launches.csv | head -40
