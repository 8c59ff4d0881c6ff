#!/bin/bash
# Run ON THE GPU BOX: ncu --set full of single configured layers (one launch each).
# usage: tools/ncu_layers.sh <tag> <config> <layer-index>...
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
for li in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"fused_conv|merged_gemm|offset_add|selective_add|eop_" -c ${COUNT:-2} \
      -o gpurun_out/${tag}_${cfg}_L${li} python tools/run_layer.py --config $cfg --layer $li --iters 1 \
      > gpurun_out/${tag}_${cfg}_L${li}.log 2>&1
  echo "$cfg L$li rc=$?"
done
