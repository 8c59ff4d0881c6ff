#!/bin/bash
mkdir -p gpurun_out
for spec in "resnet18 2" "resnet18 0" "resnet18_s2 2" "resnet18_s2 1" "resnet18 3"; do
  set -- $spec
  timeout 300 python tools/launch_trace.py $1 $2 6 > gpurun_out/x2_trace_${1}_${2}.log 2>&1
  FLUSH=1 timeout 300 python tools/launch_trace.py $1 $2 6 > gpurun_out/x2_traceF_${1}_${2}.log 2>&1
done
tail -n 12 gpurun_out/x2_trace*.log
