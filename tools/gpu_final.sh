# round-end GPU session: tests, bench lines (both arms), N>1 functional run, launch list, ncu captures
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bench_full.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# the N > 1 code path, functionally, with two ranks on the one device (gloo host collectives)
BENCH_ONE_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --gn-steps 3 --cfg-steps 1 \
  > gpurun_out/bench_2rank_1dev.json 2> gpurun_out/bench_2rank_1dev.err
bash tools/sim_scaling.sh > gpurun_out/sim_scaling.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gn --no-sharded > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gn --no-sharded > gpurun_out/ncu_launch.log 2>&1
bash tools/prof_k1.sh > gpurun_out/prof_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^value_mma -s 3 -c 1 -o gpurun_out/prof_k2 -f \
    python tools/prof_value.py > gpurun_out/ncu_k2.log 2>&1
