python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_pair_fused" -c 1 -o gpurun_out/k1_tma python tools/kbench.py --config config4 --solves 1 > gpurun_out/k1ncu.log 2>&1
IRLS_K1_NOTMA=1 ncu --set full --import-source on --clock-control none -k regex:"k_pair_fused" -c 1 -o gpurun_out/k1_notma python tools/kbench.py --config config4 --solves 1 >> gpurun_out/k1ncu.log 2>&1
tail -2 gpurun_out/k1ncu.log
