#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_g2bmm.py -q -x > gpurun_out/x10_pytest.log 2>&1
tail -3 gpurun_out/x10_pytest.log
timeout 300 python tools/time_g2bmm.py > gpurun_out/x10_g2.log 2>&1; tail -8 gpurun_out/x10_g2.log
