#!/bin/bash
# A/B/A/B of prebuilt libraries in abso/ on one box (kernel ms from bench.py)
for round in 1 2; do
for v in "$@"; do
  STROM_SO=abso/$v.so python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-gn --no-sharded --no-fullspace > gpurun_out/b_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_$v.json')); print('$v', 'kernel_ms', round(d['roofline']['kernel_ms_avg'],4), 'frac', round(d['roofline']['frac'],4))"
done
done
