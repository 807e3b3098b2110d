timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2g.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_r2g.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['stage_ms'], d.get('e2e_reference_types'))"
