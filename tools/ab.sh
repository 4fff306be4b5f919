#!/bin/bash
# quick A/B: parity tests + bench kernel time (used from gpurun)
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json; d=json.load(open('gpurun_out/b.json')); print('VALUE', d['value'], 'kernel_ms', d['roofline']['kernel_ms_avg'], 'frac', round(d['roofline']['frac'],4))"
