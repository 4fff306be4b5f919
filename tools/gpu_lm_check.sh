mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lm.py tests/test_gpu_config_goldens.py tests/test_gpu_dropin.py tests/test_gpu_configs.py tests/test_gpu_greedy_train.py -q > gpurun_out/pytest_lm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lm.log
timeout 600 python tools/prof_lm.py 3 > gpurun_out/prof_lm3.log 2>&1
timeout 600 python tools/prof_lm.py 3 >> gpurun_out/prof_lm3.log 2>&1
