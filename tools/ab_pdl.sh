#!/bin/bash
for p in 1 0 1 0; do
  OLLIE_PDL=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-cudnn 2>/dev/null | tail -1 > /tmp/b.json
  python -c "import json; d=json.load(open('/tmp/b.json')); print('PDL=$p', round(d['value'],1), 'TF/s', round(d['ms_per_step']*1e3,1), 'us/step')"
done
