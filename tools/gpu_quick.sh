# quick GPU session: parity tests + LM kernel launch list (graph kernel nodes)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/prof_lm.py 3 > gpurun_out/prof_lm3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lm3_launches.csv python tools/prof_lm.py 3 > gpurun_out/ncu_lm3.log 2>&1
python tools/diag_cfg45.py 4 64 > gpurun_out/diag4.log 2>&1
