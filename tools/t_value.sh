python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/bench_configs.py --only 3,5 --cfg5-iters 10 2>&1 | tail -2
