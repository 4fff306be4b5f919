# round-end GPU session (part 2): launch list + ncu --set full of K1 (kept) and K2 (raw csv only:
# gpurun copies back at most 64 MiB)
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gn --no-sharded --no-fullspace > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gn --no-sharded --no-fullspace > gpurun_out/ncu_launch.log 2>&1
bash tools/prof_k1.sh > gpurun_out/prof_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^value_mma -s 3 -c 1 -o /tmp/prof_k2 -f \
    python tools/prof_value.py > gpurun_out/ncu_k2.log 2>&1 && \
ncu -i /tmp/prof_k2.ncu-rep --page raw --csv > gpurun_out/prof_k2_raw.csv 2>/dev/null
# K1 register-budget A/B: 168 registers (6 CTAs/SM) vs 144 (7 CTAs/SM)
[ -f abso/r144.so ] && bash tools/ab2.sh base r144 > gpurun_out/ab_r144.log 2>&1
