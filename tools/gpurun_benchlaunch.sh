python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_bl.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --loop-mode 1 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-two-level --no-fixed-point-exit > gpurun_out/r02_bench_ncu.json 2> gpurun_out/r02_bench_ncu.err
echo "rc=$?"
python tools/launch_summary.py gpurun_out/r02_bench_launches.csv | head -30
