set -x
./tools/microbench/fir_tc 2>&1 | tail -8
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cholesky" 2>&1 | grep -E "Error|error|assert|^E " | head -20
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2e.json 2>&1; tail -c 2000 gpurun_out/bench_r2e.json
