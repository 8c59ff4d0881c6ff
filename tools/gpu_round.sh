#!/bin/bash
# One gpurun call: GPU tests, smoke, the default bench line (and optional extra commands).
# usage: tools/gpu_round.sh <tag> [pytest-args...]
tag=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -v --timeout 240 --timeout-method thread --durations 30 "$@" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
fi
tail -40 gpurun_out/${tag}_pytest.log | grep -v PASSED; tail -2 gpurun_out/${tag}_smoke.log; tail -2 gpurun_out/${tag}_bench.err
