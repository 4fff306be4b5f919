# A/B of prebuilt libraries on the k_u > 16 configs: cfg3 derivs pass, cfg4 LP rows (16 snapshots), cfg5 LM + indicator (256)
for v in "$@"; do
  STROM_SO=abso/$v.so python tools/ab_cfg3.py 2>&1 | grep us | sed "s/^/$v /"
  STROM_SO=abso/$v.so python tools/bench_configs.py --only 4,5 --cfg4-snapshots 16 --cfg5-candidates 256 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); k = list(d)[0]; v = d[k]
    print('$v', k, {a: round(b, 2) for a, b in v.items() if a in ('pass_ms', 'rom_solves_per_s', 'lm_wall_s', 'indicator_wall_s')})"
done
