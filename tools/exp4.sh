#!/bin/bash
mkdir -p gpurun_out
for li in 0 2; do
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:fused_conv -c 1 \
   -o gpurun_out/x4_r18l$li python tools/run_layer.py --config resnet18 --layer $li --iters 1 > gpurun_out/x4_r18l$li.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:fused_conv -c 1 \
   -o gpurun_out/x4_s2l2 python tools/run_layer.py --config resnet18_s2 --layer 2 --iters 1 > gpurun_out/x4_s2l2.log 2>&1
ls -la gpurun_out/x4*
