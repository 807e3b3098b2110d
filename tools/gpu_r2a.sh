set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python tools/refine_sweep.py 3 > gpurun_out/sweep_cfg3.jsonl 2> gpurun_out/sweep_cfg3.err; tail -3 gpurun_out/sweep_cfg3.err
cat gpurun_out/sweep_cfg3.jsonl
timeout 600 python tools/refine_sweep.py 2 0:0 1e-2:1e-3 > gpurun_out/sweep_cfg2.jsonl 2> gpurun_out/sweep_cfg2.err; tail -3 gpurun_out/sweep_cfg2.err
cat gpurun_out/sweep_cfg2.jsonl
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-rows 16 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -c 2500 gpurun_out/bench_r2a.json; tail -3 gpurun_out/bench_r2a.err
