# tcgen05 K2: gpu tests, then cfg timings with the tc path vs the SIMT GEMM path
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for c in 2 1 3 4; do
  timeout 120 python tools/run_cfg.py $c 2>&1 | tail -2
  NYS_K2_SIMT=1 timeout 120 python tools/run_cfg.py $c 2>&1 | tail -1
done
