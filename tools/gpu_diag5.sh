mkdir -p gpurun_out
for k in 1e-3 1e-2 1e-1 1; do python tools/diag_cfg45.py 5 128 $k >> gpurun_out/diag5_kappa.log 2>&1; done
