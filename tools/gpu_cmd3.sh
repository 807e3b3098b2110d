# cfg timings: tc path vs SIMT GEMM path
for c in 2 3 4; do
  timeout 120 python tools/run_cfg.py $c 2>&1 | tail -1
  NYS_K2_SIMT=1 timeout 120 python tools/run_cfg.py $c 2>&1 | tail -1
done
