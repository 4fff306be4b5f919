mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --steps 50 --no-cpu-baseline --no-sharded --no-fullspace > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python bench.py --steps 50 --no-cpu-baseline --no-sharded --no-fullspace --no-gn --no-graph > gpurun_out/bench_eager.json 2> gpurun_out/bench_eager.err
BENCH_SIM_WORLD=8 python bench.py --steps 50 --no-cpu-baseline --no-sharded --no-fullspace --no-gn > gpurun_out/bench_sim8.json 2>&1
rm -f gpurun_out/ab_lm.log; bash tools/ab_lm.sh base w2 w5 w8
