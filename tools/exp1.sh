#!/bin/bash
mkdir -p gpurun_out
OLLIE_EOP_ROWS=1 timeout 300 python tools/write_bw.py > gpurun_out/x1_bw_rows1.log 2>&1
OLLIE_EOP_ROWS=0 timeout 300 python tools/write_bw.py > gpurun_out/x1_bw_rows0.log 2>&1
G8S=0,1 TOP=14 timeout 900 python tools/force_sweep.py csrnet 0 > gpurun_out/x1_sweep_csrnet.log 2>&1
for li in 0 1 2 3; do TOP=4 timeout 300 python tools/force_sweep.py resnet18 $li > gpurun_out/x1_sweep_r18_$li.log 2>&1; done
tail -n 30 gpurun_out/x1_*.log
