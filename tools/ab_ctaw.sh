# K1 (config 2) with 1/2/3/4 warps per CTA (STROM_MMA_WARPS)
for w in 1 2 3 4; do
  STROM_MMA_WARPS=$w python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/w.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/w.json')); print('warps/CTA $w kernel_ms', round(d['roofline']['kernel_ms_avg'],4), 'step_ms', round(d['ms_per_step'],4))"
done
