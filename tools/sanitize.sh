# compute-sanitizer on small K1 / K2 / LM cases (one tool per invocation), logs in gpurun_out/
# usage: bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
tool=${1:-memcheck}
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "euler_square_q6 or strip or degenerate or sector" \
  > gpurun_out/sanitize_$tool.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$tool.log
