set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 600 python tools/refine_sweep.py 3 0:0 0.25:1e-3 0.5:1e-3 > gpurun_out/sweep_cfg3b.jsonl 2>&1; cat gpurun_out/sweep_cfg3b.jsonl
timeout 300 python bench.py --steps 10 --warmup 3 --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>&1; tail -c 1500 gpurun_out/bench_cfg3.json
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2c.json 2>&1; tail -c 2500 gpurun_out/bench_r2c.json
