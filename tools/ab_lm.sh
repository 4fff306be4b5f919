# A/B of LM scheduling knobs on config 3 (GN solves/s): builds variants into separate .so files
# usage (GPU box): bash tools/ab_lm.sh   -> gpurun_out/ab_lm.log
mkdir -p gpurun_out
for v in base b8 t32 b8t32; do
  echo "== $v" >> gpurun_out/ab_lm.log
  STROM_SO=$PWD/paper_2305_15661_b200/_strom_$v.so python tools/prof_lm.py 3 >> gpurun_out/ab_lm.log 2>&1
  STROM_SO=$PWD/paper_2305_15661_b200/_strom_$v.so python tools/prof_lm.py 3 >> gpurun_out/ab_lm.log 2>&1
done
