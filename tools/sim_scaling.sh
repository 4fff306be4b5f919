# per-rank kernel time of an N-GPU cfg2 job (rank 0's element range on one GPU)
for n in 1 2 4 8; do
  BENCH_SIM_WORLD=$n python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-gn --no-sharded --no-fullspace > gpurun_out/sim.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sim.json')); r=d['roofline']; print('N=$n rank-share kernel_ms', round(r['kernel_ms_avg'],4), 'step_ms', round(d['ms_per_step'],4), 'frac', round(r['frac'],3))"
done
