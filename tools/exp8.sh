#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tapfold.py tests/test_gpu_stack.py tests/test_gpu_fullsize.py -q -x > gpurun_out/x8_pytest.log 2>&1
timeout 600 python bench.py --config fsrcnn --no-suite --no-cpu-baseline --steps 5 > gpurun_out/x8_fsrcnn.json 2> gpurun_out/x8_fsrcnn.err
tail -3 gpurun_out/x8_pytest.log
python - <<'PY'
import json
d=json.loads(open('gpurun_out/x8_fsrcnn.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'])
for l in d['layers']: print("%-28s %7.1f %7.1f %s"%(l['layer'], l['ours_us'], l['ours_warm_us'], l.get('launches')))
PY
