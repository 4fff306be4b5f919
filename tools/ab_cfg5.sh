for i in 1 2; do for v in base w2; do
STROM_SO=abso/$v.so python tools/bench_configs.py --only 5 --cfg5-candidates 256 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); k = list(d)[0]; v = d[k]
    print('$v', k, {a: round(b, 3) for a, b in v.items() if a in ('rom_solves_per_s', 'lm_wall_s', 'indicator_wall_s')})"
done; done
