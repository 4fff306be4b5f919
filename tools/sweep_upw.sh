for u in 0 74 89 111 148; do
  if [ $u = 0 ]; then python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s.json 2>/dev/null; else STROM_MMA_UPW=$u python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s.json 2>/dev/null; fi
  python -c "import json; d=json.load(open('gpurun_out/s.json')); print('cfg2 UPW=$u kernel_ms', round(d['roofline']['kernel_ms_avg'],4))"
done
for u in 40 48 56 64; do STROM_MMA_UPW=$u python tools/ab_cfg3.py 2>&1 | grep "P=64"; done
