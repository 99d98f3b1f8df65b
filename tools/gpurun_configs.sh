python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_cfg.log 2>&1
timeout 1500 python bench.py --config config3 --no-cpu-baseline --no-two-level > gpurun_out/bench_config3.json 2> gpurun_out/bench_config3.err; echo "bench c3 rc=$?"
timeout 1500 python tools/bench_configs.py --configs 1,2,3,4,5 --out gpurun_out/configs_r02.json > gpurun_out/configs_r02.log 2>&1; echo "configs rc=$?"
tail -8 gpurun_out/configs_r02.log
