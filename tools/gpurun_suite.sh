#!/bin/bash
# One gpurun call: build, the -m gpu suite, smoke(), a short bench line.
# usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpurun_suite.sh TAG'
TAG=${1:-run}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/pytest_$TAG.log gpurun_out/smoke_$TAG.log
