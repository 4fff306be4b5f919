# blocks-per-SM cap sweep: cfg2 bench kernel, cfg3 derivs pass, cfg4 LP rows, cfg5 LM (128 candidates)
for b in 0 3 4 5; do
  E=""; [ $b != 0 ] && E="STROM_MMA_BPS=$b"
  env $E python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/s.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s.json')); print('BPS=$b cfg2 kernel_ms', round(d['roofline']['kernel_ms_avg'],4))"
  env $E python tools/ab_cfg3.py 2>&1 | grep us | sed "s/^/BPS=$b /"
  env $E python tools/bench_configs.py --only 4,5 --cfg4-snapshots 16 --cfg5-candidates 256 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); k = list(d)[0]; v = d[k]
    print('BPS=$b', k, {a: round(b, 2) for a, b in v.items() if a in ('pass_ms', 'rom_solves_per_s', 'lm_wall_s', 'indicator_wall_s')})"
done
