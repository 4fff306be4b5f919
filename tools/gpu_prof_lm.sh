mkdir -p gpurun_out
python tools/prof_lm.py 3 > gpurun_out/prof_lm3.log 2>&1
python tools/prof_lm.py 5 > gpurun_out/prof_lm5.log 2>&1
bash tools/sanitize.sh memcheck
