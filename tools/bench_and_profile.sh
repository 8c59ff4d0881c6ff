#!/bin/bash
# full bench line + the r02b profile set (launch lists, ncu --set full summaries)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/bp_smi.txt 2>&1
timeout 1000 python bench.py > gpurun_out/bp_bench.json 2> gpurun_out/bp_bench.err; echo "bench rc=$?" >> gpurun_out/bp_bench.err
TAG=${TAG:-r02c} timeout 2400 bash tools/profile_round.sh > gpurun_out/bp_prof.log 2>&1
mkdir -p gpurun_out/prof
PROF_DIR=gpurun_out/prof python tools/summarize_ncu.py ${TAG:-r02c} > gpurun_out/bp_summ.log 2>&1
mkdir -p /tmp/reps; mv gpurun_out/*.ncu-rep /tmp/reps/ 2>/dev/null
cp /tmp/reps/${TAG:-r02c}_full_csrnet.ncu-rep gpurun_out/ 2>/dev/null
tail -3 gpurun_out/bp_bench.err; tail -5 gpurun_out/bp_summ.log; ls gpurun_out/prof
