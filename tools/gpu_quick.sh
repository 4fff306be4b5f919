# quick GPU session: probe, parity tests, short bench (no CPU baselines)
mkdir -p gpurun_out
./tools/graph_cond_probe > gpurun_out/probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/probe.log
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --steps 50 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
