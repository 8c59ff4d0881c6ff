#!/bin/bash
# Run ON THE GPU BOX (via gpurun).  Produces, under gpurun_out/:
#   <tag>_launches_<cfg>.csv : ncu launch list (gpu__time_duration.sum, --clock-control none) of the
#                              bench command itself (cold-cache, serialised: compare SHARES)
#   <tag>_full_<cfg>.ncu-rep : ncu --set full of every libollie kernel of one step of <cfg>
set -u
TAG=${TAG:-r01}
mkdir -p gpurun_out
for cfg in ${CFGS:-resnet18 csrnet fsrcnn}; do
  # record the autotuned plans of a normal (un-profiled) run, then replay them under ncu: timing
  # inside ncu is meaningless, so without this the profiled runs would pick other plans
  export OLLIE_TUNE_FILE=gpurun_out/${TAG}_tune_${cfg}.txt
  rm -f $OLLIE_TUNE_FILE
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-cudnn > gpurun_out/${TAG}_tune_${cfg}.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
      --log-file gpurun_out/${TAG}_launches_${cfg}.csv \
      python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-cudnn --no-graph \
      > gpurun_out/${TAG}_launches_${cfg}.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"fused_conv|merged_gemm|rowstream_conv|tap_fold|offset_add|selective_add|eop_" -s ${SKIP:-0} -c ${COUNT:-12} \
      -o gpurun_out/${TAG}_full_${cfg} python tools/run_layer.py --config $cfg --iters 1 \
      > gpurun_out/${TAG}_full_${cfg}.log 2>&1
  echo "$cfg done"
  unset OLLIE_TUNE_FILE
done
