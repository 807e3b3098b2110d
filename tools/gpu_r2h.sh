NYS_DBG_K2=16 timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep K2TF | head -4
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_formed_M" 2>&1 | grep -E "^E |Error" | head -20
