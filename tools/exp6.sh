#!/bin/bash
mkdir -p gpurun_out
for form in ysum direct; do RS_FORM=$form timeout 200 python tools/rs_trace2.py 16 > gpurun_out/x6_rs_$form.log 2>&1; done
RS_FORM=direct OLLIE_RS_DBG=8 timeout 200 python tools/rs_trace2.py 16 > gpurun_out/x6_rs_direct_dbg8.log 2>&1
RS_FORM=ysum OLLIE_RS_DBG=4 timeout 200 python tools/rs_trace2.py 16 > gpurun_out/x6_rs_ysum_dbg4.log 2>&1
true
