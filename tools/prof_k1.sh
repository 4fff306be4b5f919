#!/bin/bash
# one ncu --set full capture of K1 (config-2 bench) into gpurun_out/prof_k1.ncu-rep
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gn --no-sharded --no-fullspace > gpurun_out/bench_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^derivs_mma -s 2 -c 1 -o gpurun_out/prof_k1 -f \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gn --no-sharded --no-fullspace > gpurun_out/ncu_k1.log 2>&1
echo "ncu rc=$?"
