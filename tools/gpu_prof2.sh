# profiles: K2 (cfg5 indicator) full ncu capture, LM kernel breakdown (cfg3 with slip wall)
mkdir -p gpurun_out
python tools/prof_value.py > gpurun_out/prof_value.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^value_mma -s 3 -c 1 -o gpurun_out/prof_k2 -f \
    python tools/prof_value.py > gpurun_out/ncu_k2.log 2>&1
python tools/prof_lm.py 3 > gpurun_out/prof_lm3.log 2>&1
python tools/prof_lm.py 5 > gpurun_out/prof_lm5.log 2>&1
