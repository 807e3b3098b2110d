timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['stage_ms'])"
timeout 300 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'],d['value'],d['ms_per_step'],d['roofline']['kernel_ms'])"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
