# A/B of LM scheduling variants on config 3 (GN batch wall time, graph statistics)
# usage (GPU box): bash tools/ab_lm.sh base w2 w5 ...  (libraries paper_2305_15661_b200/_strom_<v>.so)
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab_lm.log
  STROM_SO=$PWD/paper_2305_15661_b200/_strom_$v.so python tools/prof_lm.py 3 >> gpurun_out/ab_lm.log 2>&1
  STROM_SO=$PWD/paper_2305_15661_b200/_strom_$v.so python tools/prof_lm.py 3 >> gpurun_out/ab_lm.log 2>&1
done
