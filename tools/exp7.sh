#!/bin/bash
mkdir -p gpurun_out
RS_FORM=ysum OLLIE_RS_DBG=4 timeout 200 python tools/rs_trace2.py 16 > gpurun_out/x7_rs_ysum_dbg4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_rowstream.py tests/test_gpu_fullsize.py tests/test_gpu_stack.py -q -x > gpurun_out/x7_pytest.log 2>&1
timeout 600 python bench.py --config fsrcnn --no-suite --no-cpu-baseline --steps 5 > gpurun_out/x7_fsrcnn.json 2> gpurun_out/x7_fsrcnn.err
tail -3 gpurun_out/x7_pytest.log
python - <<'PY'
import json
d=json.loads(open('gpurun_out/x7_fsrcnn.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'])
for l in d['layers']: print("%-28s %7.1f %7.1f"%(l['layer'], l['ours_us'], l['ours_warm_us']))
PY
