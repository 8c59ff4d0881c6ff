#!/bin/bash
mkdir -p gpurun_out
for form in ysum direct; do RS_FORM=$form timeout 200 python tools/rs_trace2.py fsrcnn:2 > gpurun_out/x5_rs_$form.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:rowstream -c 1 \
   -o gpurun_out/x5_map python tools/run_layer.py --config fsrcnn --layer 2 --iters 1 > gpurun_out/x5_map.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:tap_fold -c 1 \
   -o gpurun_out/x5_fold python tools/run_layer.py --config fsrcnn --layer 0 --iters 1 > gpurun_out/x5_fold.log 2>&1
tail -30 gpurun_out/x5_rs_*.log
