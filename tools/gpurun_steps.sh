python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s.log 2>&1
timeout 300 python tools/step_breakdown.py
