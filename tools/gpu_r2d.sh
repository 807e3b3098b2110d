set -x
./tools/microbench/fir_tc 2>&1 | tail -6
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 600 python tools/refine_sweep.py 3 0.25:1e-3 > gpurun_out/sweep_cfg3c.jsonl 2>&1; cat gpurun_out/sweep_cfg3c.jsonl
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2d.json 2>&1; tail -c 2000 gpurun_out/bench_r2d.json
