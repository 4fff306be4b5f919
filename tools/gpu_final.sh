# round-end GPU session (part 1): tests, bench lines (both arms), N>1 path on one device, scaling estimate
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bench_full.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# the N > 1 code path, functionally, with two ranks on the one device (gloo host collectives)
BENCH_ONE_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --gn-steps 3 --cfg-steps 1 \
  > gpurun_out/bench_2rank_1dev.json 2> gpurun_out/bench_2rank_1dev.err
bash tools/sim_scaling.sh > gpurun_out/sim_scaling.txt 2>&1
