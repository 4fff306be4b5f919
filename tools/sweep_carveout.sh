# K1 shared-memory carveout sweep (config 2 kernel ms, cfg3 pass)
for c in 0 75 80 86 90 100; do
  E=""; [ $c != 0 ] && E="STROM_MMA_CARVEOUT=$c"
  env $E python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c.json')); print('carveout=$c kernel_ms', round(d['roofline']['kernel_ms_avg'],4))"
  env $E python tools/ab_cfg3.py 2>&1 | grep "P=64" | sed "s/^/carveout=$c /"
done
