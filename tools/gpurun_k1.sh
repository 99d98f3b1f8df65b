python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1
for V in 8 16 32 12 8 16 32 12 64; do echo "== zp $V"; IRLS_K1_ZP=$V timeout 120 python tools/kbench.py --config config4 --solves 1 | grep -E "K1"; done
