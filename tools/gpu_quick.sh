# quick GPU session: parity tests, diagnostics, short bench (no CPU baselines)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/diag_cfg45.py 4 64 > gpurun_out/diag4.log 2>&1
python tools/diag_cfg45.py 5 256 > gpurun_out/diag5.log 2>&1
python bench.py --steps 50 --no-cpu-baseline --no-sharded > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
